"""Multi-GPU engine: destination-interval sharding with streamed source blocks.

SURVEY.md §8(e), replacing the reference's ring-streaming simulator
 with real collectives over NVLink/NVSwitch:

* the 2D grid uses P = world intervals; rank r owns destination interval D_r (and,
  since layer outputs are indexed like inputs, source interval S_r = D_r of the next
  layer), the CSC chunks C_{i,r} of its column and the CSR chunks C_{r,j} of its row;
* forward, per layer: every source-feature block h_i is broadcast by its owner (NCCL,
  posted asynchronously in ascending i); the fused gather over C_{i,r} waits only for
  block i, so it overlaps the transfer of the later blocks, and accumulates into the
  resident A_r in ascending i -- the chunked engine's Locality order, so the result
  equals the 1-GPU chunked run with P = world bit for bit -- then ApplyVertex on the
  local rows;
* loss: softmax-CE over local rows normalised by the global |V|, loss all-reduced;
* backward: dW_r = a_r^T dz_r all-reduced; dA blocks streamed the same way; the CSR
  duals over C_{r,j} (ascending j) produce dz for the local sources with the ReLU mask
  of the layer below fused.
NVSwitch gives every GPU full bandwidth to every peer, so the reference's fat-tree /
ring ordering (built to avoid shared PCIe links) reduces to per-block broadcasts.

Compute is behind a small backend interface so the host-side logic (sharding,
ordering, collectives) runs in CPU tests with the gloo backend; the product backend
is ``CudaCompute`` (libsagann kernels + NCCL).
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
    """Rank ``rank``'s share of the P = world chunk grid (device pass indices)."""

    def __init__(self, g, world, rank, split_edges=G.DEFAULT_SPLIT_EDGES, device="cuda",
                 gcn_weights=True):
        size = -(-g.V // world)
        part = G.partition_2d(g, size)
        if part.P != world:
            raise ValueError(f"V={g.V} too small to shard over {world} ranks")
        self.V, self.E, self.world, self.rank, self.size = g.V, g.E, world, rank, size
        self.sizes = [int(s) for s in part.sizes]
        self.begin = rank * size
        self.rows = self.sizes[rank]
        degs = g.degrees() if gcn_weights else None
        self.csc, self.csr = {}, {}
        for i in range(world):
            ch = part.chunk(i, rank)
            if ch["nnz"]:
                w = g.gcn_weights(ch["csc_eid"], degs) if gcn_weights else None
                self.csc[i] = G.PassIndex(ch["csc_ptr"], ch["csc_idx"], w, self.rows, split_edges, device)
        for j in range(world):
            ch = part.chunk(rank, j)
            if ch["nnz"]:
                w = g.gcn_weights(ch["csr_eid"], degs) if gcn_weights else None
                self.csr[j] = G.PassIndex(ch["csr_ptr"], ch["csr_idx"], w, self.rows, split_edges, device)
        self.local_edges = sum(pi.nnz for pi in self.csc.values())


class CudaCompute:
    """Product backend: libsagann kernels on the current CUDA stream."""

    def __init__(self, device, gemm_prec=_lib.GEMM_TF32X3):
        from . import kernels as K

        self.K, self.device, self.prec = K, torch.device(device), gemm_prec
        self.ws = K.Workspace(self.device)

    def zeros(self, rows, cols):
        return torch.zeros((rows, _ld(cols)), dtype=torch.float32, device=self.device)[:, :cols]

    def gather(self, pi, H, out, F, accumulate, mask=None):
        self.K.propagate(pi, _lib.PROP_GCN, H, out, F, accumulate=accumulate, mask=mask, ws=self.ws)

    def gemm(self, A, B, C, trans_a=False, trans_b=False, relu_out=None):
        self.K.gemm(A, B, C, trans_a=trans_a, trans_b=trans_b, relu_out=relu_out, prec=self.prec,
                    ws=self.ws)

    def xent(self, Z, labels, loss, dZ, err, n_total):
        self.K.softmax_xent(Z, labels, loss, dZ, err, relu_input=True, n_total=n_total, ws=self.ws)

    def sgd(self, W, dW, lr):
        self.K.sgd(W, dW, lr)


class DistGCN:
    """L-layer GCN (dims = [F, H, ..., C]) sharded over the ranks of ``group``."""

    def __init__(self, shard, dims, compute, weights=None, seed=2, group=None, dtype=torch.float32):
        self.s, self.c, self.dims, self.group = shard, compute, list(dims), group
        self.dtype = dtype
        self.world = shard.world
        n, dev = shard.rows, compute.device
        self.W, self.dW = [], []
        rng = np.random.default_rng(seed)
        for k, (fi, fo) in enumerate(zip(dims, dims[1:])):
            if weights is None:
                lim = np.sqrt(6.0 / (fi + fo))
                w = rng.uniform(-lim, lim, (fi, fo)).astype(np.float32)
            else:
                w = np.asarray(weights[k])
            self.W.append(torch.from_numpy(w.copy()).to(dev, dtype))
            self.dW.append(torch.zeros((fi, fo), dtype=dtype, device=dev))
        L = len(dims) - 1
        self.h = [compute.zeros(n, dims[0])] + [compute.zeros(n, dims[k + 1]) for k in range(L - 1)]
        self.a = [compute.zeros(n, dims[k]) for k in range(L)]
        self.z = [compute.zeros(n, dims[k + 1]) for k in range(L)]
        self.dz = [compute.zeros(n, dims[k + 1]) for k in range(L)]
        self.da = [compute.zeros(n, dims[k]) for k in range(L)]
        self._blocks = {}  # (F, dtype) -> per-source-interval landing buffers
        self.labels = torch.zeros(n, dtype=torch.int64, device=dev)
        self.loss = torch.zeros(1, dtype=dtype, device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        self.comm_s = 0.0

    # ---------------------------------------------------------------- data
    def load_features(self, X_local):
        self.h[0].copy_(torch.as_tensor(X_local)[:, : self.dims[0]])

    def load_labels(self, y_local):
        self.labels.copy_(torch.as_tensor(np.asarray(y_local, np.int64)))

    # ---------------------------------------------------------------- collectives
    def _stream_blocks(self, X, F):
        """Post one broadcast per source block (root = its owner), asynchronously and in
        ascending block order, and return [(block view, work)].  The consumer waits for
        block i only right before the gather over C_{i,r}, so the gather of block i
        overlaps the NVLink transfer of blocks i+1.. (the paper's ring streaming,
        PAPER.md:495-505, on NVSwitch).  Blocks are padded to 16-byte rows."""
        ldF = _ld(F)
        key = (F, X.dtype)
        if key not in self._blocks:
            self._blocks[key] = [torch.zeros((n, ldF), dtype=X.dtype, device=X.device)
                                 for n in self.s.sizes]
        blocks = self._blocks[key]
        blocks[self.s.rank][:, :F].copy_(X)
        works = [dist.broadcast(blocks[i], src=i, group=self.group, async_op=True)
                 for i in range(self.world)]
        return [(b[:, :F], w) for b, w in zip(blocks, works)]

    # ---------------------------------------------------------------- step
    def forward(self):
        s, c = self.s, self.c
        L = len(self.dims) - 1
        for l in range(L):
            F = self.dims[l]
            blocks = self._stream_blocks(self.h[l], F)
            chain = [i for i in range(self.world) if i in s.csc]
            if not chain:
                self.a[l].zero_()
            for k, i in enumerate(chain):   # source intervals ascending (Locality order)
                blocks[i][1].wait()
                c.gather(s.csc[i], blocks[i][0], self.a[l], F, accumulate=k > 0)
            for _, w in blocks:
                w.wait()
            c.gemm(self.a[l], self.W[l], self.z[l], relu_out=self.h[l + 1] if l + 1 < L else None)
        return self.z[-1]

    def backward(self):
        s, c = self.s, self.c
        L = len(self.dims) - 1
        c.xent(self.z[-1], self.labels, self.loss, self.dz[-1], self.err, n_total=s.V)
        dist.all_reduce(self.loss, group=self.group)
        for l in range(L - 1, -1, -1):
            c.gemm(self.a[l], self.dz[l], self.dW[l], trans_a=True)
            dist.all_reduce(self.dW[l], group=self.group)
            if l > 0:
                F = self.dims[l]
                c.gemm(self.dz[l], self.W[l], self.da[l], trans_b=True)
                blocks = self._stream_blocks(self.da[l], F)
                chain = [j for j in range(self.world) if j in s.csr]
                if not chain:
                    self.dz[l - 1].zero_()
                for k, j in enumerate(chain):  # destination intervals ascending
                    blocks[j][1].wait()
                    c.gather(s.csr[j], blocks[j][0], self.dz[l - 1], F, accumulate=k > 0,
                             mask=self.z[l - 1] if k == len(chain) - 1 else None)
                for _, w in blocks:
                    w.wait()
        return self.loss

    def train_step(self, lr=0.01):
        self.forward()
        self.backward()
        for W, dW in zip(self.W, self.dW):
            self.c.sgd(W, dW, lr)
        return self.loss


def bench_main(a, cfg, metric, config):
    """bench.py --gpus N under torchrun: one process per GPU, NCCL over NVLink."""
    import json
    import os

    rank, local = int(os.environ["RANK"]), int(os.environ.get("LOCAL_RANK", 0))
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    V, E, F, H, C = cfg["V"], cfg["E"], cfg["F"], cfg["H"], cfg["C"]
    if cfg["model"] != "gcn":
        raise SystemExit("multi-GPU bench implements the GCN workload")
    g = (G.rmat_graph if cfg["graph"] == "rmat" else G.uniform_graph)(V, E, seed=0)
    shard = ShardIndex(g, world, rank, split_edges=a.split_edges, device=f"cuda:{local}")
    model = DistGCN(shard, [F, H, C], CudaCompute(f"cuda:{local}"))
    X = G.synthetic_features(V, F, seed=1)[shard.begin: shard.begin + shard.rows]
    y = np.random.default_rng(3).integers(0, C, V)[shard.begin: shard.begin + shard.rows]
    model.load_features(torch.from_numpy(X))
    model.load_labels(y)
    for _ in range(a.warmup):
        model.train_step(a.lr)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(a.steps):
        model.train_step(a.lr)
    ev1.record()
    torch.cuda.synchronize()
    dist.barrier()
    ms = torch.tensor([ev0.elapsed_time(ev1) / a.steps], device=f"cuda:{local}")
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    t = float(ms.item()) / 1e3
    if rank == 0:
        line = {"metric": metric, "value": E / t, "unit": "edges/s", "n_gpus": world,
                "steps": a.steps, "warmup": a.warmup, "ms_per_step": t * 1e3,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic", "config": config,
                "wall_s": time.perf_counter() - t0,
                "gpu_launches": None, "e2e": None, "roofline": None, "cpu_baseline": None}
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()
