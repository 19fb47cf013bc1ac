"""Out-of-core GCN and G-GCN training: host-resident graph, streamed chunk dataflow
(SURVEY §8(f) rank 2).

The paper's original setting (PAPER.md:324-342; SPEC.md:306-315 insert_swaps, :351-359
Locality schedule, :376 prefetch depth 1): vertex features, activations and the 2D chunk
index live in pinned HOST memory; the device holds only a bounded working set --

* the accumulator A_j of the destination interval being gathered (resident through its
  whole chain and its ApplyVertex, the Locality schedule's reuse),
* two source-interval slots and two chunk-index slots: while chunk k runs, chunk k+1 and
  its source rows are copied host->device on a separate copy stream (prefetch depth 1),
* the layer weights and gradients.

Each chunk runs the same sm_100a kernels as the resident executor in the same order, so
GCN layer aggregates are bitwise identical to ``SAGAModel`` on the same grid; the loss and
weight gradients are summed per interval (fixed order) and agree to fp32 round-off.
Transfer volume is counted per epoch (``h2d_bytes`` / ``d2h_bytes``).

``StreamingGGCN`` does the same for G-GCN: per-interval hoist GEMMs write [h | P] rows back to
the host, the gather streams those blocks against the resident Q_j (GGCN_FWD_S, so the
backward's dQ = dA (.) S needs no CSC pass), and the backward streams [dA | Q] blocks through
the CSR dual against the resident [h | P]_i.
"""

import numpy as np
import torch

from . import _lib
from . import kernels as K
from ._lib import lib
from .errors import BudgetError, ConfigError, ShapeError
from .graph import DEFAULT_SPLIT_EDGES, partition_2d, plan


def _ld(n):
    return (n + 3) // 4 * 4


class HostPass:
    """One chunk pass index (CSC or CSR) in pinned host memory."""

    def __init__(self, ptr, idx, w, n_rows, split_edges):
        items, splits, n_slots = plan(ptr, split_edges)
        pin = torch.cuda.is_available()

        def t(a):
            x = torch.from_numpy(np.ascontiguousarray(a))
            return x.pin_memory() if pin else x

        self.n_rows, self.nnz = int(n_rows), int(ptr[-1])
        self.n_items, self.n_splits, self.n_slots = len(items), len(splits), n_slots
        self.ptr = t(np.asarray(ptr, np.int64))
        self.idx = t(np.asarray(idx, np.int32))
        self.w = None if w is None else t(np.asarray(w, np.float32))
        self.items = t(items.view(np.uint8))
        self.splits = t(splits.view(np.uint8)) if len(splits) else None

    def nbytes(self):
        return sum(x.numel() * x.element_size() for x in (self.ptr, self.idx, self.w, self.items,
                                                           self.splits) if x is not None)


class HostGrid:
    """The 2D chunk grid with every pass index kept on the host."""

    def __init__(self, g, interval_size, split_edges=DEFAULT_SPLIT_EDGES, gcn_weights=True,
                 partition=None):
        self.part = partition if partition is not None else partition_2d(g, interval_size)
        self.V, self.E, self.P = g.V, g.E, self.part.P
        degs = g.degrees() if gcn_weights else None
        self.csc, self.csr = {}, {}
        for i in range(self.P):
            for j in range(self.P):
                ch = self.part.chunk(i, j)
                if ch["nnz"] == 0:
                    continue
                wc = g.gcn_weights(ch["csc_eid"], degs) if gcn_weights else None
                wr = g.gcn_weights(ch["csr_eid"], degs) if gcn_weights else None
                self.csc[(i, j)] = HostPass(ch["csc_ptr"], ch["csc_idx"], wc, self.part.sizes[j], split_edges)
                self.csr[(i, j)] = HostPass(ch["csr_ptr"], ch["csr_idx"], wr, self.part.sizes[i], split_edges)

    def begin(self, k):
        return self.part.begin(k)

    def size(self, k):
        return int(self.part.sizes[k])


class _DevPass:
    """Device view of one streamed pass index (attributes as graph.PassIndex)."""

    def workspace_bytes(self, F, mode):
        return int(lib.sg_propagate_workspace_bytes(self.n_items, self.n_splits, self.n_slots, F, mode))


class _IndexSlot:
    """Device buffers able to hold any pass index of the grid."""

    def __init__(self, dev, grid):
        passes = list(grid.csc.values()) + list(grid.csr.values())
        mx = lambda f: max([f(p) for p in passes] + [1])  # noqa: E731
        self.ptr = torch.empty(mx(lambda p: p.ptr.numel()), dtype=torch.int64, device=dev)
        self.idx = torch.empty(mx(lambda p: p.nnz), dtype=torch.int32, device=dev)
        self.w = torch.empty(mx(lambda p: p.nnz), dtype=torch.float32, device=dev)
        self.items = torch.empty(mx(lambda p: p.items.numel()), dtype=torch.uint8, device=dev)
        self.splits = torch.empty(mx(lambda p: p.splits.numel() if p.splits is not None else 1),
                                  dtype=torch.uint8, device=dev)
        self.key = None

    def nbytes(self):
        return sum(x.numel() * x.element_size() for x in (self.ptr, self.idx, self.w, self.items, self.splits))

    def load(self, hp):
        """Async copies on the current stream; returns (device pass view, bytes copied)."""
        d = _DevPass()
        d.n_rows, d.nnz, d.n_items, d.n_splits, d.n_slots = hp.n_rows, hp.nnz, hp.n_items, hp.n_splits, hp.n_slots
        nb = 0
        d.ptr = self.ptr[: hp.ptr.numel()]
        d.ptr.copy_(hp.ptr, non_blocking=True)
        d.idx = self.idx[: hp.nnz]
        d.idx.copy_(hp.idx, non_blocking=True)
        nb += hp.ptr.numel() * 8 + hp.nnz * 4
        d.w = None
        if hp.w is not None:
            d.w = self.w[: hp.nnz]
            d.w.copy_(hp.w, non_blocking=True)
            nb += hp.nnz * 4
        d.items = self.items[: hp.items.numel()]
        d.items.copy_(hp.items, non_blocking=True)
        nb += hp.items.numel()
        d.splits = None
        if hp.splits is not None:
            d.splits = self.splits[: hp.splits.numel()]
            d.splits.copy_(hp.splits, non_blocking=True)
            nb += hp.splits.numel()
        return d, nb


def _pinned(r, c):
    """Pinned [r, ld(c)] host matrix (rows padded to 16 B, padding zero)."""
    t = torch.zeros((r, _ld(c)), dtype=torch.float32)
    return t.pin_memory() if torch.cuda.is_available() else t


def _block(buf, n, c):
    """Contiguous [n, ld(c)] view of a flat device scratch buffer (matches a host row block)."""
    return buf.view(-1)[: n * _ld(c)].view(n, _ld(c))


class _Streamer:
    """Shared host<->device plumbing: row blocks, counted copies, the prefetching chunk loop."""

    def _rows(self, t, k):
        b = self.grid.begin(k)
        return t[b: b + self.grid.size(k)]

    def _h2d(self, dst, src):
        dst.copy_(src, non_blocking=True)
        self.h2d_bytes += src.numel() * src.element_size()

    def _d2h(self, dst, src):
        dst.copy_(src, non_blocking=True)
        self.d2h_bytes += src.numel() * src.element_size()

    def _stream(self, tasks, index, source, F, body):
        """Run ``body(k, task, dev_pass, src_rows)`` over ``tasks`` = [(i, j, key)], each task
        reading pass ``index[key]`` and source rows ``source(task)`` (a host view), with the
        next task's index + source rows copied on the copy stream (prefetch depth 1)."""
        comp = torch.cuda.current_stream(self.dev)
        cs = self.copy_stream
        cs.wait_stream(comp)  # slots / scratch may still be read by earlier compute
        ready = [None, None]
        free = [None, None]
        loaded_src = [None, None]
        staged = [None, None]

        def prefetch(k):
            s = k % 2
            i, j, key, skey = tasks[k]
            with torch.cuda.stream(cs):
                if free[s] is not None:
                    cs.wait_event(free[s])
                dp, nb = self.slots[s].load(index[key])
                self.h2d_bytes += nb
                hs = source(tasks[k])                      # host row block [n, ld(F)]
                dst = _block(self.src[s], hs.shape[0], F)
                if loaded_src[s] != skey:
                    self._h2d(dst, hs)
                    loaded_src[s] = skey
                ev = torch.cuda.Event()
                ev.record(cs)
            ready[s] = ev
            staged[s] = (dp, dst[:, :F])

        if tasks:
            prefetch(0)
        for k in range(len(tasks)):
            s = k % 2
            if k + 1 < len(tasks):
                prefetch(k + 1)
            comp.wait_event(ready[s])
            dp, srows = staged[s]
            body(k, tasks[k], dp, srows)
            ev = torch.cuda.Event()
            ev.record(comp)
            free[s] = ev
        # the copy stream must not run ahead into buffers of the next pass
        comp.wait_stream(cs)


class StreamingGCN(_Streamer):
    """L-layer GCN trained out of core over a HostGrid.

    ``dims`` = [F, H, ..., C]; ``budget`` (bytes) bounds the device working set and raises
    BudgetError naming the widest interval/chunk when it cannot hold."""

    def __init__(self, grid, dims, weights=None, *, seed=2, budget=None, gemm_prec=_lib.GEMM_TF32X3,
                 device="cuda"):
        if not torch.cuda.is_available():
            raise RuntimeError("StreamingGCN needs a CUDA device (no CPU fallback)")
        if len(dims) < 2:
            raise ConfigError("dims must list at least [F, C]")
        self.grid, self.dims, self.dev = grid, list(dims), torch.device(device)
        self.prec = gemm_prec
        self.L = len(dims) - 1
        P, V = grid.P, grid.V
        nmax = max(grid.size(k) for k in range(P))
        Fmax = max(dims)
        dev = self.dev
        # ---------------- device working set
        self.W, self.dW, self._wbuf = [], [], []
        for a, b in zip(dims, dims[1:]):
            wb = torch.zeros((a, _ld(b)), dtype=torch.float32, device=dev)
            gb = torch.zeros_like(wb)
            self._wbuf.append((wb, gb))
            self.W.append(wb[:, :b])
            self.dW.append(gb[:, :b])
        self.src = [torch.zeros((nmax, _ld(Fmax)), dtype=torch.float32, device=dev) for _ in range(2)]
        self.slots = [_IndexSlot(dev, grid) for _ in range(2)]
        self.acc = torch.zeros((nmax, _ld(Fmax)), dtype=torch.float32, device=dev)
        self.zb = torch.zeros((nmax, _ld(Fmax)), dtype=torch.float32, device=dev)
        self.hb = torch.zeros((nmax, _ld(Fmax)), dtype=torch.float32, device=dev)
        self.tmpW = torch.zeros((Fmax, _ld(Fmax)), dtype=torch.float32, device=dev)
        self.lab = torch.zeros(nmax, dtype=torch.int64, device=dev)
        self.loss = torch.zeros(1, dtype=torch.float32, device=dev)
        self.lpart = torch.zeros(1, dtype=torch.float32, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.ws = K.Workspace(dev)
        self.working_set = (sum(x.numel() * 4 for x in self.src) + sum(s.nbytes() for s in self.slots) +
                            3 * self.acc.numel() * 4 + 2 * sum(w.numel() * 4 for w, _ in self._wbuf))
        if budget is not None and self.working_set > budget:
            big = max(list(grid.csc.items()) + list(grid.csr.items()), key=lambda kv: kv[1].nnz)
            raise BudgetError(f"device working set {self.working_set} B exceeds budget {budget} B "
                              f"(interval of {nmax} rows x {Fmax} features, largest chunk C{big[0]} "
                              f"with {big[1].nnz} edges); use a smaller interval_size")
        # ---------------- host-resident tensors (pinned)
        self.X = _pinned(V, dims[0])
        self.A = [_pinned(V, f) for f in dims[:-1]]      # aggregates (for dW)
        self.Z = [_pinned(V, f) for f in dims[1:]]       # pre-activations (ReLU masks)
        self.H = [_pinned(V, f) for f in dims[1:-1]]     # ReLU outputs = next layer inputs
        self.dZ = [_pinned(V, f) for f in dims[1:]]
        self.dA = [_pinned(V, f) for f in dims[:-1]]
        self.labels = torch.zeros(V, dtype=torch.int64).pin_memory()
        self.copy_stream = torch.cuda.Stream(device=dev)
        self.h2d_bytes = self.d2h_bytes = 0
        self.set_weights(weights if weights is not None else self.init_weights(seed))

    # ---------------------------------------------------------------- parameters
    def init_weights(self, seed=2):
        rng = np.random.default_rng(seed)
        out = []
        for a, b in zip(self.dims, self.dims[1:]):
            lim = np.sqrt(6.0 / (a + b))
            out.append(rng.uniform(-lim, lim, (a, b)).astype(np.float32))
        return out

    def set_weights(self, ws):
        if len(ws) != self.L:
            raise ShapeError("wrong number of weight matrices")
        for W, w in zip(self.W, ws):
            W.copy_(torch.as_tensor(np.asarray(w, np.float32)))

    def weights(self):
        return [W.cpu().numpy().copy() for W in self.W]

    def grads(self):
        return [g.cpu().numpy().copy() for g in self.dW]

    def load_features(self, X):
        X = torch.as_tensor(X)
        self.X[:, : self.dims[0]].copy_(X[:, : self.dims[0]])

    def load_labels(self, y):
        self.labels.copy_(torch.as_tensor(np.asarray(y, np.int64)))

    # ---------------------------------------------------------------- streaming
    def forward(self):
        """All layers: per destination interval j, gather over C_0j..C_{P-1,j} into the
        resident A_j, then ApplyVertex (and the loss on the last layer) before moving on."""
        g, P = self.grid, self.grid.P
        self.loss.zero_()
        for l in range(self.L):
            F, O = self.dims[l], self.dims[l + 1]
            hin = self.X if l == 0 else self.H[l - 1]
            chains = {j: [i for i in range(P) if (i, j) in g.csc] for j in range(P)}
            tasks = [(i, j, (i, j), (l, i)) for j in range(P) for i in chains[j]]
            A = self.acc

            def finish_column(j, l=l, F=F, O=O):
                n = g.size(j)
                a, z, h = _block(A, n, F), _block(self.zb, n, O), _block(self.hb, n, O)
                last = l == self.L - 1
                K.gemm(a[:, :F], self.W[l], z[:, :O], relu_out=None if last else h[:, :O], prec=self.prec,
                       ws=self.ws)
                self._d2h(self._rows(self.A[l], j), a)
                self._d2h(self._rows(self.Z[l], j), z)
                if not last:
                    self._d2h(self._rows(self.H[l], j), h)
                else:  # softmax-CE on ReLU(z_j) over the global row count (tensor.py:487-506)
                    lab = self.lab[:n]
                    self._h2d(lab, self._rows(self.labels, j))
                    K.softmax_xent(z[:, :O], lab, self.lpart, h[:, :O], self.err, relu_input=True,
                                   n_total=g.V, ws=self.ws)
                    K.ewise(0, self.loss.view(1, 1), self.lpart.view(1, 1), self.loss.view(1, 1))
                    self._d2h(self._rows(self.dZ[l], j), h)

            def body(k, task, dp, srows, F=F, chains=chains, finish_column=finish_column):
                i, j, _, _ = task
                n = g.size(j)
                K.propagate(dp, _lib.PROP_GCN, srows, _block(A, n, F)[:, :F], F,
                            accumulate=i != chains[j][0], ws=self.ws, hub=False)
                if i == chains[j][-1]:
                    finish_column(j)

            # empty destination columns: A_j = 0
            for j in range(P):
                if not chains[j]:
                    _block(A, g.size(j), F).zero_()
                    finish_column(j)
            self._stream(tasks, g.csc, lambda t, hin=hin: self._rows(hin, t[0]), F, body)
        return self.loss

    def backward(self):
        """Reverse stages: dW_l = sum_j A_j^T dz_j (fixed j order), dA = dz W^T per interval,
        then the CSR dual per source interval i over C_i0..C_i,P-1 with the ReLU mask."""
        g, P = self.grid, self.grid.P
        for l in range(self.L - 1, -1, -1):
            F, O = self.dims[l], self.dims[l + 1]
            self.dW[l].zero_()
            for j in range(P):
                n = g.size(j)
                a, dz = _block(self.src[0], n, F), _block(self.zb, n, O)
                self._h2d(a, self._rows(self.A[l], j))
                self._h2d(dz, self._rows(self.dZ[l], j))
                t = self.tmpW[:F, :O]
                K.gemm(a[:, :F], dz[:, :O], t, trans_a=True, prec=self.prec, ws=self.ws)
                K.ewise(0, self.dW[l], t, self.dW[l])
                if l > 0:
                    da = _block(self.hb, n, F)
                    K.gemm(dz[:, :O], self.W[l], da[:, :F], trans_b=True, prec=self.prec, ws=self.ws)
                    self._d2h(self._rows(self.dA[l], j), da)
            if l == 0:
                break
            chains = {i: [j for j in range(P) if (i, j) in g.csr] for i in range(P)}
            tasks = [(i, j, (i, j), (l, j)) for i in range(P) for j in chains[i]]
            out, mask = self.acc, self.zb

            def body(k, task, dp, srows, F=F, chains=chains, l=l):
                i, j, _, _ = task
                n = g.size(i)
                first, last = j == chains[i][0], j == chains[i][-1]
                o = _block(out, n, F)
                m = None
                if last:
                    mb = _block(mask, n, F)
                    self._h2d(mb, self._rows(self.Z[l - 1], i))
                    m = mb[:, :F]
                K.propagate(dp, _lib.PROP_GCN, srows, o[:, :F], F, accumulate=not first, mask=m,
                            ws=self.ws, hub=False)
                if last:
                    self._d2h(self._rows(self.dZ[l - 1], i), o)

            for i in range(P):
                if not chains[i]:
                    self._rows(self.dZ[l - 1], i).zero_()
            self._stream(tasks, g.csr, lambda t, l=l: self._rows(self.dA[l], t[1]), F, body)
        return self.loss

    def sgd(self, lr):
        for wb, gb in self._wbuf:
            K.sgd(wb, gb, lr)

    def train_step(self, lr=0.01):
        self.h2d_bytes = self.d2h_bytes = 0
        self.forward()
        self.backward()
        self.sgd(lr)
        return self.loss

    def check_status(self):
        torch.cuda.synchronize(self.dev)
        if int(self.err.item()):
            raise ShapeError("label out of range [0, classes)")


class StreamingGGCN(_Streamer):
    """L-layer G-GCN (listing :172-173) trained out of core over a HostGrid
    built without GCN weights.  Parameters per layer: W_H [F, F], W_C [F, F], W [F, O] (the
    resident executor's order).  Host-resident per layer: [h | P] and [dA | Q] rows
    (interleaved, so each streamed source block is one contiguous row range), the aggregate A,
    S, z, dz and dQ.  Device: the accumulators of one interval, one resident row block, two
    streamed source blocks and two chunk-index slots."""

    def __init__(self, grid, dims, weights=None, *, seed=2, budget=None, gemm_prec=_lib.GEMM_TF32X3,
                 device="cuda"):
        if not torch.cuda.is_available():
            raise RuntimeError("StreamingGGCN needs a CUDA device (no CPU fallback)")
        if len(dims) < 2:
            raise ConfigError("dims must list at least [F, C]")
        self.grid, self.dims, self.dev = grid, list(dims), torch.device(device)
        self.prec = gemm_prec
        self.L = len(dims) - 1
        P, V = grid.P, grid.V
        nmax = max(grid.size(k) for k in range(P))
        dev = self.dev
        self.go = [_ld(f) for f in dims[:-1]]
        G2 = 2 * max(self.go)
        Fmax = max(dims)
        # ---------------- parameters (16-B padded buffers)
        self._wbuf, self.params, self.dparams = [], [], []
        for a, b in zip(dims, dims[1:]):
            for (r, c) in ((a, a), (a, a), (a, b)):
                wb = torch.zeros((r, _ld(c)), dtype=torch.float32, device=dev)
                gb = torch.zeros_like(wb)
                self._wbuf.append((wb, gb))
                self.params.append(wb[:, :c])
                self.dparams.append(gb[:, :c])
        # ---------------- device working set
        self.src = [torch.zeros((nmax, G2), dtype=torch.float32, device=dev) for _ in range(2)]
        self.slots = [_IndexSlot(dev, grid) for _ in range(2)]
        self.rowb = torch.zeros((nmax, G2), dtype=torch.float32, device=dev)   # resident block
        self.acc = torch.zeros((nmax, _ld(Fmax)), dtype=torch.float32, device=dev)
        self.acc2 = torch.zeros((nmax, _ld(Fmax)), dtype=torch.float32, device=dev)
        self.zb = torch.zeros((nmax, _ld(Fmax)), dtype=torch.float32, device=dev)
        self.hb = torch.zeros((nmax, G2), dtype=torch.float32, device=dev)
        self.t1 = torch.zeros((nmax, _ld(Fmax)), dtype=torch.float32, device=dev)
        self.t2 = torch.zeros((nmax, _ld(Fmax)), dtype=torch.float32, device=dev)
        self.tmpW = torch.zeros((Fmax, _ld(Fmax)), dtype=torch.float32, device=dev)
        self.lab = torch.zeros(nmax, dtype=torch.int64, device=dev)
        self.loss = torch.zeros(1, dtype=torch.float32, device=dev)
        self.lpart = torch.zeros(1, dtype=torch.float32, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.ws = K.Workspace(dev)
        bufs = self.src + [self.rowb, self.acc, self.acc2, self.zb, self.hb, self.t1, self.t2, self.tmpW]
        self.working_set = (sum(x.numel() * 4 for x in bufs) + sum(s.nbytes() for s in self.slots) +
                            2 * sum(w.numel() * 4 for w, _ in self._wbuf))
        if budget is not None and self.working_set > budget:
            raise BudgetError(f"device working set {self.working_set} B exceeds budget {budget} B "
                              f"(interval of {nmax} rows x {Fmax} features); use a smaller interval_size")
        # ---------------- host-resident tensors (pinned)
        self.HP = [_pinned(V, 2 * go) for go in self.go]        # [h | P] per layer
        self.GQ = [_pinned(V, 2 * go) for go in self.go]        # [dA | Q] per layer
        self.A = [_pinned(V, f) for f in dims[:-1]]
        self.S = [_pinned(V, f) for f in dims[:-1]]
        self.dQ = [_pinned(V, f) for f in dims[:-1]]
        self.Z = [_pinned(V, f) for f in dims[1:]]
        self.dZ = [_pinned(V, f) for f in dims[1:]]
        self.labels = torch.zeros(V, dtype=torch.int64).pin_memory()
        self.copy_stream = torch.cuda.Stream(device=dev)
        self.h2d_bytes = self.d2h_bytes = 0
        self.set_weights(weights if weights is not None else self.init_weights(seed))

    # ---------------------------------------------------------------- parameters
    def _layer(self, l, grads=False):
        ps = self.dparams if grads else self.params
        return ps[3 * l], ps[3 * l + 1], ps[3 * l + 2]          # W_H, W_C, W

    def init_weights(self, seed=2):
        rng = np.random.default_rng(seed)
        out = []
        for a, b in zip(self.dims, self.dims[1:]):
            for (r, c) in ((a, a), (a, a), (a, b)):
                lim = np.sqrt(6.0 / (r + c))
                out.append(rng.uniform(-lim, lim, (r, c)).astype(np.float32))
        return out

    def set_weights(self, ws):
        if len(ws) != 3 * self.L:
            raise ShapeError("wrong number of weight matrices")
        for W, w in zip(self.params, ws):
            W.copy_(torch.as_tensor(np.asarray(w, np.float32)))

    def weights(self):
        return [W.cpu().numpy().copy() for W in self.params]

    def grads(self):
        return [g.cpu().numpy().copy() for g in self.dparams]

    def load_features(self, X):
        X = torch.as_tensor(X)
        self.HP[0][:, : self.dims[0]].copy_(X[:, : self.dims[0]])

    def load_labels(self, y):
        self.labels.copy_(torch.as_tensor(np.asarray(y, np.int64)))

    def _gemm(self, A, B, C, **kw):
        K.gemm(A, B, C, prec=self.prec, ws=self.ws, **kw)

    def _acc_grad(self, dW, A, B):
        """dW += A^T B (per-interval partial through tmpW, fixed interval order)."""
        t = self.tmpW[: dW.shape[0], : dW.shape[1]]
        self._gemm(A, B, t, trans_a=True)
        K.ewise(0, dW, t, dW)

    # ---------------------------------------------------------------- step
    def forward(self):
        """Per layer: hoist P = h W_H and Q = h W_C per interval (back to the host), then per
        destination interval j the gated gather over C_0j..C_{P-1,j} (streamed [h | P] blocks,
        resident Q_j) into A_j and S_j, then ApplyVertex."""
        g, P = self.grid, self.grid.P
        self.loss.zero_()
        for l in range(self.L):
            F, O, go = self.dims[l], self.dims[l + 1], self.go[l]
            WH, WC, W = self._layer(l)
            for k in range(P):                          # hoist, per interval
                n = g.size(k)
                hp, gq = _block(self.rowb, n, 2 * go), _block(self.hb, n, 2 * go)
                self._h2d(hp, self._rows(self.HP[l], k))
                self._gemm(hp[:, :F], WH, hp[:, go:go + F])
                gq.zero_()
                self._gemm(hp[:, :F], WC, gq[:, go:go + F])
                self._d2h(self._rows(self.HP[l], k), hp)
                self._d2h(self._rows(self.GQ[l], k), gq)
            chains = {j: [i for i in range(P) if (i, j) in g.csc] for j in range(P)}
            tasks = [(i, j, (i, j), (l, i)) for j in range(P) for i in chains[j]]

            def finish_column(j, l=l, F=F, O=O, go=go, W=W):
                n = g.size(j)
                a, sS = _block(self.acc, n, F), _block(self.acc2, n, F)
                z = _block(self.zb, n, O)
                last = l == self.L - 1
                self._d2h(self._rows(self.A[l], j), a)
                self._d2h(self._rows(self.S[l], j), sS)
                if not last:
                    go2 = self.go[l + 1]
                    hn = _block(self.hb, n, 2 * go2)
                    hn.zero_()
                    self._gemm(a[:, :F], W, z[:, :O], relu_out=hn[:, :O])
                    self._d2h(self._rows(self.Z[l], j), z)
                    self._d2h(self._rows(self.HP[l + 1], j), hn)   # P half filled by the next hoist
                else:
                    self._gemm(a[:, :F], W, z[:, :O])
                    self._d2h(self._rows(self.Z[l], j), z)
                    lab = self.lab[:n]
                    dz = _block(self.t1, n, O)
                    self._h2d(lab, self._rows(self.labels, j))
                    K.softmax_xent(z[:, :O], lab, self.lpart, dz[:, :O], self.err, relu_input=True,
                                   n_total=g.V, ws=self.ws)
                    K.ewise(0, self.loss.view(1, 1), self.lpart.view(1, 1), self.loss.view(1, 1))
                    self._d2h(self._rows(self.dZ[l], j), dz)

            def body(k, task, dp, srows, F=F, go=go, chains=chains, finish_column=finish_column, l=l):
                i, j, _, _ = task
                n = g.size(j)
                if i == chains[j][0]:                   # resident Q_j for the whole chain
                    self.rowb_j = _block(self.rowb, n, 2 * go)
                    self.rowb_j.copy_(self._rows(self.GQ[l], j), non_blocking=True)
                    self.h2d_bytes += n * 2 * go * 4
                K.propagate(dp, _lib.PROP_GGCN_FWD_S, srows, _block(self.acc, n, F)[:, :F], F, g_off=go,
                            R=self.rowb_j[:, go:go + F], out1=_block(self.acc2, n, F)[:, :F],
                            accumulate=i != chains[j][0], ws=self.ws, hub=False)
                if i == chains[j][-1]:
                    finish_column(j)

            for j in range(P):
                if not chains[j]:
                    _block(self.acc, g.size(j), F).zero_()
                    _block(self.acc2, g.size(j), F).zero_()
                    finish_column(j)
            self._stream(tasks, g.csc, lambda t, l=l: self._rows(self.HP[l], t[0]), 2 * go, body)
        return self.loss

    def backward(self):
        """Reverse stages per layer: per interval dW += a^T dz, dA = dz W^T (into the host
        [dA | Q] rows), dQ = dA (.) S, dW_C += h^T dQ; then per source interval i the CSR dual
        over streamed [dA | Q] blocks against the resident [h | P]_i (dP, the take_rows part of
        dh), dW_H += h^T dP and dz of the layer below (ReLU mask)."""
        g, P = self.grid, self.grid.P
        for p in self.dparams:
            p.zero_()
        for l in range(self.L - 1, -1, -1):
            F, O, go = self.dims[l], self.dims[l + 1], self.go[l]
            WH, WC, W = self._layer(l)
            dWH, dWC, dW = self._layer(l, grads=True)
            for j in range(P):
                n = g.size(j)
                a, dz = _block(self.acc, n, F), _block(self.zb, n, O)
                gq, hp = _block(self.hb, n, 2 * go), _block(self.rowb, n, 2 * go)
                sS = _block(self.acc2, n, F)
                self._h2d(a, self._rows(self.A[l], j))
                self._h2d(dz, self._rows(self.dZ[l], j))
                self._acc_grad(dW, a[:, :F], dz[:, :O])
                self._h2d(gq, self._rows(self.GQ[l], j))
                self._gemm(dz[:, :O], W, gq[:, :F], trans_b=True)   # dA = dz W^T
                self._d2h(self._rows(self.GQ[l], j), gq)
                self._h2d(sS, self._rows(self.S[l], j))
                dq = _block(self.t1, n, F)
                K.ewise(2, gq[:, :F], sS[:, :F], dq[:, :F])           # dQ = dA (.) S
                self._d2h(self._rows(self.dQ[l], j), dq)
                self._h2d(hp, self._rows(self.HP[l], j))
                self._acc_grad(dWC, hp[:, :F], dq[:, :F])             # dW_C += h^T dQ
            chains = {i: [j for j in range(P) if (i, j) in g.csr] for i in range(P)}
            tasks = [(i, j, (i, j), (l, j)) for i in range(P) for j in chains[i]]

            def finish_row(i, l=l, F=F, go=go, WH=WH, WC=WC, dWH=dWH):
                n = g.size(i)
                hp = self.rowb_i
                dP, dHt = _block(self.acc, n, F), _block(self.acc2, n, F)
                self._acc_grad(dWH, hp[:, :F], dP[:, :F])             # dW_H += h^T dP
                if l == 0:
                    return
                t1, t2 = _block(self.t1, n, F), _block(self.t2, n, F)
                dq = _block(self.zb, n, F)
                self._h2d(dq, self._rows(self.dQ[l], i))
                self._gemm(dq[:, :F], WC, t1[:, :F], trans_b=True)
                K.ewise(0, dHt[:, :F], t1[:, :F], t1[:, :F])         # take_rows part + Q part
                self._gemm(dP[:, :F], WH, t2[:, :F], trans_b=True)
                K.ewise(0, t1[:, :F], t2[:, :F], t1[:, :F])          # + P part (tape order)
                zb = _block(self.hb, n, F)
                self._h2d(zb, self._rows(self.Z[l - 1], i))
                K.ewise(8, t1[:, :F], zb[:, :F], t1[:, :F])          # relu bwd of the layer below
                self._d2h(self._rows(self.dZ[l - 1], i), t1)

            def body(k, task, dp, srows, F=F, go=go, chains=chains, finish_row=finish_row, l=l):
                i, j, _, _ = task
                n = g.size(i)
                if j == chains[i][0]:                   # resident [h | P]_i for the whole chain
                    self.rowb_i = _block(self.rowb, n, 2 * go)
                    self.rowb_i.copy_(self._rows(self.HP[l], i), non_blocking=True)
                    self.h2d_bytes += n * 2 * go * 4
                K.propagate(dp, _lib.PROP_GGCN_BWD_SRC, srows, _block(self.acc, n, F)[:, :F], F, g_off=go,
                            R=self.rowb_i, r_off=go, out1=_block(self.acc2, n, F)[:, :F],
                            accumulate=j != chains[i][0], ws=self.ws, hub=False)
                if j == chains[i][-1]:
                    finish_row(i)

            for i in range(P):
                if not chains[i]:
                    n = g.size(i)
                    _block(self.acc, n, F).zero_()
                    _block(self.acc2, n, F).zero_()
                    self.rowb_i = _block(self.rowb, n, 2 * go)
                    self.rowb_i.copy_(self._rows(self.HP[l], i), non_blocking=True)
                    finish_row(i)
            self._stream(tasks, g.csr, lambda t, l=l: self._rows(self.GQ[l], t[1]), 2 * go, body)
        return self.loss

    def sgd(self, lr):
        for wb, gb in self._wbuf:
            K.sgd(wb, gb, lr)

    def train_step(self, lr=0.01):
        self.h2d_bytes = self.d2h_bytes = 0
        self.forward()
        self.backward()
        self.sgd(lr)
        return self.loss

    def check_status(self):
        torch.cuda.synchronize(self.dev)
        if int(self.err.item()):
            raise ShapeError("label out of range [0, classes)")
