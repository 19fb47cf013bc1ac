"""Multi-GPU engine: destination-interval sharding with streamed source blocks.

SURVEY.md §8(e), replacing the reference's ring-streaming simulator
 with real collectives over NVLink/NVSwitch:

* vertices are first re-encoded with ``reencode_balance`` for
  P = world intervals, so every rank owns about |V|/world vertices AND about |E|/world
  edge endpoints (R-MAT concentrates edges on low ids; without it rank 0 would own
  most in-edges);
* the 2D grid uses P = world intervals; rank r owns destination interval D_r (and,
  since layer outputs are indexed like inputs, source interval S_r = D_r of the next
  layer), the CSC chunks C_{i,r} of its column and the CSR chunks C_{r,j} of its row;
* forward, per layer: every source-feature block (h_i for GCN, [h_i | P_i] for G-GCN)
  is broadcast by its owner (NCCL, posted asynchronously in ascending i) into one [V, F]
  landing buffer; then ONE fused gather over the rank's whole column C_{*,r} (a pass index
  over global ids, each row's in-edges in ascending source: the 1-GPU P = 1 pass over the
  re-encoded graph, bit for bit) -- the default, ``ShardIndex(column=True)``: at 8 ranks the
  per-chunk launches below ran 2.5x under one launch's per-edge rate, because every chunk
  launch ends on its longest row (profiles/r02_dist_proxy.jsonl).  With ``column=False`` the
  gather over C_{i,r} waits only for block i, overlapping the transfer of the later blocks,
  and accumulates into A_r in ascending i (the 1-GPU chunked run with P = world, bitwise);
  then ApplyVertex on the local rows;
* loss: softmax-CE over local rows normalised by the global |V|, loss all-reduced;
* backward: dW_r = a_r^T dz_r all-reduced; GCN streams the dA blocks and runs the CSR
  dual over the rank's row C_{r,*} (or per chunk C_{r,j}, ascending j) with the ReLU mask of
  the layer below fused; G-GCN
  takes dQ = dA (.) S with S summed by the forward (GGCN_FWD_S), streams the [dA | Q]
  blocks and runs pass B (CSR, dP and the take_rows part of dh) over them.
NVSwitch gives every GPU full bandwidth to every peer, so the reference's fat-tree /
ring ordering (built to avoid shared PCIe links) reduces to per-block broadcasts.

Compute is behind a small backend interface so the host-side logic (sharding,
ordering, collectives) runs in CPU tests with the gloo backend; the product backend
is ``CudaCompute`` (libsagann kernels; NCCL for the collectives).
"""

import time

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from . import graph as G


def _ld(n, align=4):
    return (n + align - 1) // align * align


class ShardIndex:
    """Rank ``rank``'s share of the P = world chunk grid (device pass indices).

    ``balance``: re-encode the graph with reencode_balance(world) first; ``perm`` maps
    old -> new vertex ids and ``vertices`` lists the ORIGINAL ids of the local rows
    (select features / labels with it)."""

    def __init__(self, g, world, rank, split_edges="auto", device="cuda",
                 gcn_weights=True, balance=True, column=True):
        size = -(-g.V // world)
        if balance and world > 1:
            g, perm = G.reencode_balance(g, world)
        else:
            perm = np.arange(g.V, dtype=np.int64)
        inv = np.empty_like(perm)
        inv[perm] = np.arange(g.V, dtype=np.int64)
        part = G.partition_2d(g, size)
        if part.P != world:
            raise ValueError(f"V={g.V} too small to shard over {world} ranks")
        self.graph, self.perm = g, perm
        self.V, self.E, self.world, self.rank, self.size = g.V, g.E, world, rank, size
        self.sizes = [int(s) for s in part.sizes]
        self.begin = rank * size
        self.rows = self.sizes[rank]
        self.vertices = inv[self.begin: self.begin + self.rows]
        degs = g.degrees() if gcn_weights else None
        self.column = bool(column)
        self.csc, self.csr = {}, {}
        self.col_csc = self.col_csr = None
        if self.column:
            # the rank's whole column C_{*,r} (forward) and row C_{r,*} (backward) as ONE pass
            # index each over global (re-encoded) ids: per local row, the chunks' edges in
            # ascending block order -- for every row the in-edges sorted by global source, i.e.
            # the single-GPU P = 1 pass over the re-encoded graph, bit for bit.  One launch per
            # pass instead of world: at 8 ranks the per-chunk launches ran 2.5x below the
            # per-edge rate of one launch (tools/dist_proxy.py, profiles/r02_dist_proxy.jsonl)
            self.col_csc = self._column(part, g, degs, False, split_edges, device)
            self.col_csr = self._column(part, g, degs, True, split_edges, device)
            self.local_edges = self.col_csc.nnz if self.col_csc is not None else 0
            return
        for i in range(world):
            ch = part.chunk(i, rank)
            if ch["nnz"]:
                w = g.gcn_weights(ch["csc_eid"], degs) if degs is not None else None
                self.csc[i] = G.PassIndex(ch["csc_ptr"], ch["csc_idx"], w, self.rows, split_edges, device)
        for j in range(world):
            ch = part.chunk(rank, j)
            if ch["nnz"]:
                w = g.gcn_weights(ch["csr_eid"], degs) if degs is not None else None
                self.csr[j] = G.PassIndex(ch["csr_ptr"], ch["csr_idx"], w, self.rows, split_edges, device)
        self.local_edges = sum(pi.nnz for pi in self.csc.values())

    def _column(self, part, g, degs, csr, split_edges, device):
        keys, idx, w = [], [], []
        for k in range(self.world):
            ch = part.chunk(self.rank, k) if csr else part.chunk(k, self.rank)
            if not ch["nnz"]:
                continue
            ptr = ch["csr_ptr"] if csr else ch["csc_ptr"]
            rows = np.repeat(np.arange(self.rows, dtype=np.int64), np.diff(ptr))
            keys.append(rows * self.world + k)
            idx.append(ch["csr_idx" if csr else "csc_idx"].astype(np.int64) + k * self.size)
            if degs is not None:
                w.append(g.gcn_weights(ch["csr_eid" if csr else "csc_eid"], degs))
        if not keys:
            return None
        keys = np.concatenate(keys)
        o = np.argsort(keys, kind="stable")        # by row, then block; in-chunk order kept
        ptr = np.zeros(self.rows + 1, np.int64)
        ptr[1:] = np.cumsum(np.bincount(keys[o] // self.world, minlength=self.rows))
        idx = np.concatenate(idx)[o].astype(np.int32)
        w = np.concatenate(w)[o] if w else None
        return G.PassIndex(ptr, idx, w, self.rows, split_edges, device)


class CudaCompute:
    """Product backend: libsagann kernels on the current CUDA stream."""

    def __init__(self, device, gemm_prec=_lib.GEMM_TF32X3):
        from . import kernels as K

        self.K, self.device, self.prec = K, torch.device(device), gemm_prec
        self.ws = K.Workspace(self.device)

    def zeros(self, rows, cols):
        return torch.zeros((rows, _ld(cols)), dtype=torch.float32, device=self.device)[:, :cols]

    def propagate(self, pi, mode, Gm, out, F, *, g_off=0, R=None, r_off=0, out1=None, mask=None,
                  accumulate=False):
        self.K.propagate(pi, mode, Gm, out, F, g_off=g_off, R=R, r_off=r_off, out1=out1, mask=mask,
                         accumulate=accumulate, ws=self.ws)

    def gemm(self, A, B, C, trans_a=False, trans_b=False, relu_out=None):
        self.K.gemm(A, B, C, trans_a=trans_a, trans_b=trans_b, relu_out=relu_out, prec=self.prec,
                    ws=self.ws)

    def add(self, a, b, out):
        self.K.ewise(0, a, b, out)

    def mul(self, a, b, out):
        self.K.ewise(2, a, b, out)

    def relu_bwd(self, g, z, out):
        self.K.ewise(8, g, z, out)

    def xent(self, Z, labels, loss, dZ, err, n_total):
        self.K.softmax_xent(Z, labels, loss, dZ, err, relu_input=True, n_total=n_total, ws=self.ws)

    def sgd(self, W, dW, lr):
        self.K.sgd(W, dW, lr)

    def launches(self):
        return int(_lib.lib.sg_launch_count())


class DistSAGA:
    """L-layer GCN or G-GCN (dims = [F, H, ..., C]) sharded over the ranks of ``group``.

    Parameters per layer: GCN [W]; G-GCN [W_H, W_C, W] (the single-GPU executor's order).
    Parameter buffers are 16-B padded (the tensor-core GEMM's TMA path)."""

    def __init__(self, shard, dims, compute, model="gcn", weights=None, seed=2, group=None,
                 dtype=torch.float32):
        if model not in ("gcn", "ggcn"):
            raise ValueError(f"unknown model '{model}' (gcn | ggcn)")
        self.s, self.c, self.dims, self.group, self.model = shard, compute, list(dims), group, model
        self.dtype = dtype
        self.world = shard.world
        n, dev = shard.rows, compute.device
        L = len(dims) - 1
        shapes = []
        for fi, fo in zip(dims, dims[1:]):
            shapes += ([(fi, fi), (fi, fi)] if model == "ggcn" else []) + [(fi, fo)]
        if weights is None:
            rng = np.random.default_rng(seed)
            weights = []
            for fi, fo in shapes:
                lim = np.sqrt(6.0 / (fi + fo))
                weights.append(rng.uniform(-lim, lim, (fi, fo)).astype(np.float32))
        if len(weights) != len(shapes):
            raise ValueError("wrong number of weight matrices")
        self.params, self.grads_, self._bufs = [], [], []
        for (fi, fo), w in zip(shapes, weights):
            wb = torch.zeros((fi, _ld(fo)), dtype=dtype, device=dev)
            gb = torch.zeros_like(wb)
            wb[:, :fo].copy_(torch.as_tensor(np.asarray(w)).to(dtype))
            self._bufs.append((wb, gb))
            self.params.append(wb[:, :fo])
            self.grads_.append(gb[:, :fo])
        k = 3 if model == "ggcn" else 1
        self.W = [self.params[k * l + k - 1] for l in range(L)]
        self.dW = [self.grads_[k * l + k - 1] for l in range(L)]
        self.h = [compute.zeros(n, dims[0])] + [compute.zeros(n, dims[l + 1]) for l in range(L - 1)]
        self.a = [compute.zeros(n, dims[l]) for l in range(L)]
        self.z = [compute.zeros(n, dims[l + 1]) for l in range(L)]
        self.dz = [compute.zeros(n, dims[l + 1]) for l in range(L)]
        self.da = [compute.zeros(n, dims[l]) for l in range(L)]
        if model == "ggcn":
            self.WH = [self.params[3 * l] for l in range(L)]
            self.WC = [self.params[3 * l + 1] for l in range(L)]
            self.dWH = [self.grads_[3 * l] for l in range(L)]
            self.dWC = [self.grads_[3 * l + 1] for l in range(L)]
            self.goff = [_ld(dims[l]) for l in range(L)]
            # per-vertex [h | P] (forward gather operand) and [dA | Q] (backward pass B operand)
            self.HP = [compute.zeros(n, 2 * self.goff[l]) for l in range(L)]
            self.GQ = [compute.zeros(n, 2 * self.goff[l]) for l in range(L)]
            self.dQ = [compute.zeros(n, dims[l]) for l in range(L)]
            self.dP = [compute.zeros(n, dims[l]) for l in range(L)]
            self.dHt = [compute.zeros(n, dims[l]) for l in range(L)]
            self.S = [compute.zeros(n, dims[l]) for l in range(L)]  # GGCN_FWD_S second output
            F0 = max(dims[:-1])
            self.t1, self.t2 = compute.zeros(n, F0), compute.zeros(n, F0)
            self.h[0] = self.HP[0][:, : dims[0]]
            for l in range(1, L):
                self.h[l] = self.HP[l][:, : dims[l]]
        self._blocks = {}  # key -> per-source-interval landing buffers (views of _full[key])
        self._full = {}
        self.labels = torch.zeros(n, dtype=torch.int64, device=dev)
        self.loss = torch.zeros(1, dtype=dtype, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.prof = None

    # ---------------------------------------------------------------- data
    def load_features(self, X_local):
        self.h[0].copy_(torch.as_tensor(X_local)[:, : self.dims[0]], non_blocking=True)

    def load_labels(self, y_local):
        self.labels.copy_(torch.as_tensor(np.asarray(y_local, np.int64)), non_blocking=True)

    def prefetch_inputs(self, X_host, y_host):
        """Stage the next step's local feature / label shard (pinned host) on a copy stream,
        overlapping the running step; the next ``train_step`` waits for it and moves it into
        place (one D2D copy of the shard)."""
        h0 = self.h[0]
        base = h0._base if h0._base is not None else h0
        if getattr(self, "_cs", None) is None:
            self._cs = torch.cuda.Stream(device=self.c.device)
            self._sx = torch.empty_like(base)     # the padded device layout: contiguous copies
            self._sy = torch.empty_like(self.labels)
            self._used = None
        if self._used is not None:
            self._cs.wait_event(self._used)
        X_host = torch.as_tensor(X_host)
        with torch.cuda.stream(self._cs):
            if X_host.is_contiguous() and tuple(X_host.shape) == tuple(self._sx.shape):
                self._sx.copy_(X_host, non_blocking=True)
            else:
                self._sx[:, : self.dims[0]].copy_(X_host[:, : self.dims[0]], non_blocking=True)
            self._sy.copy_(torch.as_tensor(y_host), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self._cs)
        self._staged = ev

    def _take_staged(self):
        if getattr(self, "_staged", None) is None:
            return
        cur = torch.cuda.current_stream(self.c.device)
        cur.wait_event(self._staged)
        h0 = self.h[0]
        if h0._base is not None and h0._base.shape == self._sx.shape and h0.data_ptr() == h0._base.data_ptr():
            h0._base.copy_(self._sx)              # one contiguous device copy
        else:
            h0.copy_(self._sx[:, : self.dims[0]])
        self.labels.copy_(self._sy)
        self._used = torch.cuda.Event()
        self._used.record(cur)
        self._staged = None

    def weights(self):
        return [p.detach().cpu().numpy().copy() for p in self.params]

    def grads(self):
        return [g.detach().cpu().numpy().copy() for g in self.grads_]

    # ---------------------------------------------------------------- profiling
    def _mark(self, name):
        if self.prof is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.prof.append((name, e))

    def stage_times(self):
        out = {}
        for (_, a), (name, b) in zip(self.prof, self.prof[1:]):
            if name != "start":
                out[name] = out.get(name, 0.0) + a.elapsed_time(b)
        return out

    # ---------------------------------------------------------------- collectives
    def _stream_blocks(self, key, X, width):
        """Post one broadcast per source block (root = its owner), asynchronously and in
        ascending block order, and return [(block, work)].  The consumer waits for
        block i only right before the gather over chunk i, so the gather of block i
        overlaps the NVLink transfer of blocks i+1.. (the paper's ring streaming,
        PAPER.md:495-505, on NVSwitch).  Blocks are padded to 16-byte rows; the own
        block is copied in place (its broadcast is the send)."""
        ldw = _ld(width)
        if key not in self._blocks:
            # one [V, ldw] buffer, block i = rows of source interval i (a column pass reads it
            # whole with global ids)
            full = torch.zeros((self.s.V, ldw), dtype=X.dtype, device=X.device)
            self._full[key] = full
            self._blocks[key] = [full[i * self.s.size: i * self.s.size + n] for i, n in enumerate(self.s.sizes)]
        blocks = self._blocks[key]
        blocks[self.s.rank][:, :width].copy_(X[:, :width])
        works = [dist.broadcast(blocks[i], src=i, group=self.group, async_op=True)
                 for i in range(self.world)]
        return [(b[:, :width], w) for b, w in zip(blocks, works)]

    def _allreduce(self, t):
        """Sum a parameter gradient over ranks: the whole 16-B padded buffer behind the view
        (collectives need contiguous memory; the padding columns are zero on every rank)."""
        dist.all_reduce(t if t.is_contiguous() else t._base, group=self.group)

    @staticmethod
    def _drain(blocks):
        for _, w in blocks:
            w.wait()

    # ---------------------------------------------------------------- step
    def forward(self):
        s, c = self.s, self.c
        L = len(self.dims) - 1
        self._mark("start")
        for l in range(L):
            F = self.dims[l]
            chain = [i for i in range(self.world) if i in s.csc]
            if self.model == "ggcn":
                go = self.goff[l]
                HP = self.HP[l]
                c.gemm(self.h[l], self.WH[l], HP[:, go: go + F])          # P = h W_H (hoisted)
                c.gemm(self.h[l], self.WC[l], self.GQ[l][:, go: go + F])  # Q = h W_C
                self._mark(f"L{l}.fwd.hoist_gemm")
                blocks = self._stream_blocks(("HP", l), HP, go + F)
                if s.column:
                    self._drain(blocks)
                    if s.col_csc is not None:
                        c.propagate(s.col_csc, _lib.PROP_GGCN_FWD_S, self._full[("HP", l)][:, : go + F],
                                    self.a[l], F, g_off=go, R=self.GQ[l][:, go: go + F], out1=self.S[l])
                for k, i in enumerate(chain):
                    blocks[i][1].wait()
                    c.propagate(s.csc[i], _lib.PROP_GGCN_FWD_S, blocks[i][0], self.a[l], F, g_off=go,
                                R=self.GQ[l][:, go: go + F], out1=self.S[l], accumulate=k > 0)
            else:
                blocks = self._stream_blocks(("h", F), self.h[l], F)
                if s.column:
                    self._drain(blocks)
                    if s.col_csc is not None:
                        c.propagate(s.col_csc, _lib.PROP_GCN, self._full[("h", F)][:, :F], self.a[l], F)
                for k, i in enumerate(chain):   # source intervals ascending (Locality order)
                    blocks[i][1].wait()
                    c.propagate(s.csc[i], _lib.PROP_GCN, blocks[i][0], self.a[l], F,
                                accumulate=k > 0)
            if not chain and (not s.column or s.col_csc is None):
                self.a[l].zero_()
                if self.model == "ggcn":
                    self.S[l].zero_()
            self._drain(blocks)
            self._mark(f"L{l}.fwd.propagate")
            c.gemm(self.a[l], self.W[l], self.z[l], relu_out=self.h[l + 1] if l + 1 < L else None)
            self._mark(f"L{l}.fwd.apply_vertex")
        return self.z[-1]

    def backward(self):
        s, c = self.s, self.c
        L = len(self.dims) - 1
        c.xent(self.z[-1], self.labels, self.loss, self.dz[-1], self.err, n_total=s.V)
        dist.all_reduce(self.loss, group=self.group)
        self._mark("loss")
        for l in range(L - 1, -1, -1):
            F = self.dims[l]
            c.gemm(self.a[l], self.dz[l], self.dW[l], trans_a=True)
            self._allreduce(self.dW[l])
            if self.model == "ggcn":
                self._backward_ggcn(l)
                continue
            if l == 0:
                self._mark(f"L{l}.bwd.apply_vertex")
                continue
            c.gemm(self.dz[l], self.W[l], self.da[l], trans_b=True)
            self._mark(f"L{l}.bwd.apply_vertex")
            blocks = self._stream_blocks(("h", F), self.da[l], F)
            chain = [j for j in range(self.world) if j in s.csr]
            if s.column:
                self._drain(blocks)
                if s.col_csr is not None:
                    c.propagate(s.col_csr, _lib.PROP_GCN, self._full[("h", F)][:, :F], self.dz[l - 1], F,
                                mask=self.z[l - 1])
                else:
                    self.dz[l - 1].zero_()
            elif not chain:
                self.dz[l - 1].zero_()
            for k, j in enumerate(chain):  # destination intervals ascending
                blocks[j][1].wait()
                c.propagate(s.csr[j], _lib.PROP_GCN, blocks[j][0], self.dz[l - 1], F,
                            accumulate=k > 0, mask=self.z[l - 1] if k == len(chain) - 1 else None)
            self._drain(blocks)
            self._mark(f"L{l}.bwd.propagate")
        return self.loss

    def _backward_ggcn(self, l):
        s, c = self.s, self.c
        F, go = self.dims[l], self.goff[l]
        GQ = self.GQ[l]
        c.gemm(self.dz[l], self.W[l], GQ[:, :F], trans_b=True)          # dA = dz W^T
        self._mark(f"L{l}.bwd.apply_vertex")
        # dQ[u] = dA[u] (.) S[u], S summed by the forward (GGCN_FWD_S): no second CSC pass
        c.mul(GQ[:, :F], self.S[l], self.dQ[l])
        # pass B over the local CSR row: dP[v], dh_take[v], with streamed [dA | Q] blocks
        blocks = self._stream_blocks(("GQ", l), GQ, go + F)
        chain = [j for j in range(self.world) if j in s.csr]
        if s.column:
            self._drain(blocks)
            if s.col_csr is not None:
                c.propagate(s.col_csr, _lib.PROP_GGCN_BWD_SRC, self._full[("GQ", l)][:, : go + F], self.dP[l], F,
                            g_off=go, R=self.HP[l], r_off=go, out1=self.dHt[l])
            else:
                self.dP[l].zero_()
                self.dHt[l].zero_()
        elif not chain:
            self.dP[l].zero_()
            self.dHt[l].zero_()
        for k, j in enumerate(chain):
            blocks[j][1].wait()
            c.propagate(s.csr[j], _lib.PROP_GGCN_BWD_SRC, blocks[j][0], self.dP[l], F, g_off=go,
                        R=self.HP[l], r_off=go, out1=self.dHt[l], accumulate=k > 0)
        self._drain(blocks)
        self._mark(f"L{l}.bwd.propagate")
        c.gemm(self.h[l], self.dQ[l], self.dWC[l], trans_a=True)        # dW_C = h^T dQ
        c.gemm(self.h[l], self.dP[l], self.dWH[l], trans_a=True)        # dW_H = h^T dP
        self._allreduce(self.dWC[l])
        self._allreduce(self.dWH[l])
        if l > 0:
            t1, t2 = self.t1[:, :F], self.t2[:, :F]
            c.gemm(self.dQ[l], self.WC[l], t1, trans_b=True)
            c.add(self.dHt[l], t1, t1)                                  # take_rows part + Q part
            c.gemm(self.dP[l], self.WH[l], t2, trans_b=True)
            c.add(t1, t2, t1)                                           # + P part (tape order)
            c.relu_bwd(t1, self.z[l - 1], self.dz[l - 1])
        self._mark(f"L{l}.bwd.hoist_gemm")

    def sgd(self, lr):
        for wb, gb in self._bufs:
            self.c.sgd(wb, gb, lr)
        self._mark("sgd")

    def train_step(self, lr=0.01):
        self._take_staged()
        self.forward()
        self.backward()
        self.sgd(lr)
        return self.loss


DistGCN = DistSAGA  # the GCN engine of earlier revisions


def pass_bytes(model, nnz, rows, F, s=4):
    """SURVEY.md §8(d) algorithmic bytes of one forward gather pass over a chunk."""
    if model == "gcn":
        return nnz * (4 + 4 + F * s) + rows * (4 + F * s)
    return nnz * (4 + 2 * F * s) + rows * (4 + 3 * F * s)


def bench_main(a, cfg, metric, config, helpers):
    """bench.py --gpus N under torchrun: one process per GPU, NCCL over NVLink.

    Timing: W warm-up steps; K timed steps bracketed by barrier + synchronize, CUDA
    events per step with an L2 flush between steps, max over ranks; the per-stage
    times (and the roofline of the layer-1 gather) are max over ranks too."""
    import json
    import os

    rank, local = int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    # SG_DIST_BACKEND=gloo is a test hook: N ranks sharing the visible GPU(s) (NCCL refuses two
    # ranks on one device), so the multi-rank bench logic runs on a one-GPU box
    backend = os.environ.get("SG_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)
    V, E, F, H, C = cfg["V"], cfg["E"], cfg["F"], cfg["H"], cfg["C"]
    t0 = time.perf_counter()
    g = (G.rmat_graph if cfg["graph"] == "rmat" else G.uniform_graph)(V, E, seed=0)
    shard = ShardIndex(g, world, rank, split_edges=a.split_edges, device=dev,
                       gcn_weights=cfg["model"] == "gcn")
    del g
    t_setup = time.perf_counter() - t0
    comp = CudaCompute(dev)
    model = DistSAGA(shard, [F, H, C], comp, model=cfg["model"])
    X_all = G.synthetic_features(V, F, seed=1)
    y_all = np.random.default_rng(3).integers(0, C, V)
    Fp = (F + 3) // 4 * 4                   # host shard in the padded device row layout
    Xs = np.zeros((shard.rows, Fp), np.float32)
    Xs[:, :F] = X_all[shard.vertices]
    X_host = torch.from_numpy(Xs).pin_memory()
    y_host = torch.from_numpy(np.ascontiguousarray(y_all[shard.vertices])).pin_memory()
    del X_all, y_all
    model.load_features(X_host)
    model.load_labels(y_host)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(a.warmup):
        model.train_step(a.lr)
    torch.cuda.synchronize()

    clocks = helpers["Clocks"](local)
    clocks.start()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    marks = []
    n0 = comp.launches()
    dist.barrier()
    torch.cuda.synchronize()
    for k in range(a.steps):
        flush.zero_()
        model.prof = []
        starts[k].record()
        model.train_step(a.lr)
        ends[k].record()
        marks.append(model.prof)
    torch.cuda.synchronize()
    dist.barrier()
    launches = comp.launches() - n0
    clk = clocks.stop()
    step_ms = [s_.elapsed_time(e) for s_, e in zip(starts, ends)]
    stages = {}
    for mk in marks:
        model.prof = mk
        for kname, v in model.stage_times().items():
            stages[kname] = stages.get(kname, 0.0) + v / a.steps
    model.prof = None
    names = sorted(stages)
    vec = torch.tensor([float(np.mean(step_ms))] + [stages[k] for k in names], device=dev,
                       dtype=torch.float64)
    dist.all_reduce(vec, op=dist.ReduceOp.MAX)
    t_step = float(vec[0].item()) / 1e3
    stages_max = {k: float(v) for k, v in zip(names, vec[1:].tolist())}
    if int(model.err.item()):
        raise RuntimeError("label out of range")

    # roofline of the layer-1 forward gather: all ranks' algorithmic bytes over the
    # slowest rank's stage time (it includes waiting for streamed blocks)
    my_bytes = sum(pass_bytes(cfg["model"], pi.nnz, pi.n_rows, F) for pi in shard.csc.values())
    tb = torch.tensor([float(my_bytes)], device=dev, dtype=torch.float64)
    dist.all_reduce(tb)
    k_ms = stages_max.get("L0.fwd.propagate")
    peak, peak_src = helpers["measured_peaks"]()
    achieved = float(tb.item()) / (k_ms / 1e3) / 1e9 if k_ms else None

    # e2e: per step H2D of the local feature/label shard from pinned memory, the step,
    # and the loss read back; wall clock, max over ranks
    e2e = None
    if not a.no_e2e:
        n_e2e = max(5, a.steps)
        torch.cuda.synchronize()
        dist.barrier()
        t1 = time.perf_counter()
        model.prefetch_inputs(X_host, y_host)
        for k in range(n_e2e):
            model.train_step(a.lr)
            if k + 1 < n_e2e:
                model.prefetch_inputs(X_host, y_host)   # overlaps this step
            float(model.loss.item())
        te = torch.tensor([(time.perf_counter() - t1) / n_e2e], device=dev, dtype=torch.float64)
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
        bi = torch.tensor([float(X_host.numel() * 4 + y_host.numel() * 8)], device=dev,
                          dtype=torch.float64)
        dist.all_reduce(bi)
        t_e2e = float(te.item())
        e2e = {"value": E / t_e2e, "unit": "edges/s", "h2d_bytes_per_step": int(bi.item()),
               "d2h_bytes_per_step": 4 * world, "ms_per_step": t_e2e * 1e3,
               "note": "wall clock, max over ranks: per step, H2D of every rank's feature/label "
                       "shard (copy stream, overlapping the previous step), the step, loss D2H"}
    lt = torch.tensor([float(launches)], device=dev, dtype=torch.float64)
    dist.all_reduce(lt)
    shard_edges = _gather_ints(shard.local_edges, world, dev)
    if rank == 0:
        line = {"metric": metric, "value": E / t_step, "unit": "edges/s", "n_gpus": world,
                "steps": a.steps, "warmup": a.warmup, "ms_per_step": t_step * 1e3,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic", "config": config,
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak * world,
                             "unit": "GB/s", "frac": achieved / (peak * world) if achieved else None,
                             "traffic": None,
                             "kernel": f"L0.fwd.propagate ({cfg['model']} gather, F={F}), all ranks",
                             "algorithmic_bytes_per_launch": float(tb.item()), "launch_ms": k_ms,
                             "peak_source": peak_src + f" x {world} GPUs"},
                "e2e": e2e, "cpu_baseline": None, "gpu_launches": int(lt.item()),
                "backend": backend,
                "clocks": clk, "stages_ms": {k: round(v, 4) for k, v in stages_max.items()},
                "shard_edges": [int(x) for x in shard_edges],
                "setup_s": round(t_setup, 2),
                "step_ms_all": [round(x, 3) for x in step_ms]}
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def _gather_ints(x, world, dev):
    t = torch.zeros(world, dtype=torch.int64, device=dev)
    t[dist.get_rank()] = int(x)
    dist.all_reduce(t)
    return t.tolist()
