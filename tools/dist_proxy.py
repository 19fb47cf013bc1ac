"""Single-GPU proxy of the N-GPU sharded epoch (DistSAGA, dist.py) on the bench workload.

For N = 1, 2, 4, 8: build every rank's shard (reencode_balance + P = N grid, ShardIndex), then
run rank r's whole step on this one GPU -- its CSC column C_{*,r} (forward, both layers), its
ApplyVertex GEMMs on |D_r| rows, softmax-CE, its CSR row C_{r,*} (backward dual, ReLU mask) and
the weight-gradient GEMMs -- with every source block already resident (what the streamed NCCL
broadcasts deliver), captured in a CUDA graph and CUDA-event timed, 3 warm-up + 10 timed steps
each; one more eager step with events between stages gives the slowest rank's breakdown
(host-enqueue gaps included there).  The N-GPU epoch is
bounded below by max_r T_r (compute) and by the per-rank broadcast volume over NVLink; the
predicted speedup is T_1 / max(max_r T_r, comm) with comm at NVLINK_GBS (0 if fully overlapped).

    python tools/dist_proxy.py [config] [Ns...]     -> one JSON line per N
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1810_08403_b200 as sg  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_1810_08403_b200 import _lib  # noqa: E402
from paper_1810_08403_b200 import dist as D  # noqa: E402
from paper_1810_08403_b200 import kernels as K  # noqa: E402

NVLINK_GBS = 900.0   # per direction, NVLink 5 through NVSwitch
name = sys.argv[1] if len(sys.argv) > 1 else "reddit"
Ns = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
cfg = CONFIGS[name]
V, E, F, H, C = cfg["V"], cfg["E"], cfg["F"], cfg["H"], cfg["C"]
g = sg.rmat_graph(V, E, seed=0) if cfg["graph"] == "rmat" else sg.uniform_graph(V, E, seed=0)
dev = torch.device("cuda")
ws = K.Workspace(dev)
P3 = _lib.GEMM_TF32X3


def mat(n, f):
    return torch.zeros((n, (f + 3) // 4 * 4), device=dev)[:, :f]


X = mat(V, F)
X.copy_(torch.from_numpy(sg.synthetic_features(V, F, seed=1)))
W0 = mat(F, H).uniform_(-0.1, 0.1)
W1 = mat(H, C).uniform_(-0.1, 0.1)
h1 = mat(V, H).uniform_(-1, 1)      # layer-1 input of every rank (all blocks resident)
da1 = mat(V, H).uniform_(-1, 1)     # layer-1 dA of every rank (backward blocks resident)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
t1 = None
COLUMN = os.environ.get("SG_PROXY_COLUMN", "1") == "1"   # dist.ShardIndex's default
SPLIT = os.environ.get("SG_PROXY_SPLIT", "auto")          # subgroup size T of the rank passes
# SG_PROXY_RECV=1: before each pass, rewrite the blocks it reads (X, h1, dA) from a second copy --
# what the NCCL broadcasts (and, for the rank's own block, its GEMM / H2D) write into the landing
# buffer each step, so the pass sees the L2 state a received block leaves; the copies are timed as
# their own "recv.*" stages and left out of the rank's compute time
RECV = os.environ.get("SG_PROXY_RECV", "0") == "1"
if RECV:
    Xs, h1s, da1s = X.clone(), h1.clone(), da1.clone()


for N in Ns:
    shards = [D.ShardIndex(g, N, r, device=dev, column=COLUMN,
                           split_edges=SPLIT if SPLIT == "auto" else int(SPLIT)) for r in range(N)]
    size = shards[0].size
    blk = lambda t, i: t[i * size: i * size + shards[0].sizes[i]]  # noqa: E731
    per_rank, stages = [], []
    for r, s in enumerate(shards):
        n = s.rows
        a0, a1, z0, hz, z1, dz1, dz0 = mat(n, F), mat(n, H), mat(n, H), mat(n, H), mat(n, C), mat(n, C), mat(n, H)
        dW0, dW1 = mat(F, H), mat(H, C)
        lab = torch.zeros(n, dtype=torch.int64, device=dev)
        loss, err = torch.zeros(1, device=dev), torch.zeros(1, dtype=torch.int32, device=dev)

        marks = []

        def mark(name):
            if timing:
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                marks.append((name, e))

        colc, colr = s.col_csc, s.col_csr

        def step():
            mark("start")
            if COLUMN:
                if RECV:
                    X.copy_(Xs)
                    mark("recv.X")
                K.propagate(colc, _lib.PROP_GCN, X, a0, F, ws=ws)
                mark("L0.fwd.propagate")
                K.gemm(a0, W0, z0, relu_out=hz, prec=P3, ws=ws)
                mark("L0.fwd.gemm")
                if RECV:
                    h1.copy_(h1s)
                    mark("recv.h1")
                K.propagate(colc, _lib.PROP_GCN, h1, a1, H, ws=ws)
                mark("L1.fwd.propagate")
                K.gemm(a1, W1, z1, prec=P3, ws=ws)
                K.softmax_xent(z1, lab, loss, dz1, err, ws=ws)
                K.gemm(a1, dz1, dW1, trans_a=True, prec=P3, ws=ws)
                mark("L1.gemms+loss")
                if RECV:
                    da1.copy_(da1s)
                    mark("recv.dA")
                K.propagate(colr, _lib.PROP_GCN, da1, dz0, H, mask=z0, ws=ws)
                mark("L1.bwd.propagate")
                K.gemm(a0, dz0, dW0, trans_a=True, prec=P3, ws=ws)
                mark("L0.dW.gemm")
                return
            mark("start")
            for k, i in enumerate(sorted(s.csc)):
                K.propagate(s.csc[i], _lib.PROP_GCN, blk(X, i), a0, F, accumulate=k > 0, ws=ws)
            mark("L0.fwd.propagate")
            K.gemm(a0, W0, z0, relu_out=hz, prec=P3, ws=ws)
            mark("L0.fwd.gemm")
            for k, i in enumerate(sorted(s.csc)):
                K.propagate(s.csc[i], _lib.PROP_GCN, blk(h1, i), a1, H, accumulate=k > 0, ws=ws)
            mark("L1.fwd.propagate")
            K.gemm(a1, W1, z1, prec=P3, ws=ws)
            K.softmax_xent(z1, lab, loss, dz1, err, ws=ws)
            K.gemm(a1, dz1, dW1, trans_a=True, prec=P3, ws=ws)
            mark("L1.gemms+loss")
            chain = sorted(s.csr)
            for k, j in enumerate(chain):
                K.propagate(s.csr[j], _lib.PROP_GCN, blk(da1, j), dz0, H, accumulate=k > 0,
                            mask=z0 if k == len(chain) - 1 else None, ws=ws)
            mark("L1.bwd.propagate")
            K.gemm(a0, dz0, dW0, trans_a=True, prec=P3, ws=ws)
            mark("L0.dW.gemm")

        timing = False

        for _ in range(3):
            step()
        # the rank's step captured in a CUDA graph (as the engine's graph mode runs it): at N = 8
        # a chunk pass is ~0.05-0.5 ms of GPU work, less than its Python enqueue
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        graph.replay()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(10)]
        for e0, e1 in ev:
            flush.zero_()
            e0.record()
            graph.replay()
            e1.record()
        torch.cuda.synchronize()
        per_rank.append(float(np.mean([e0.elapsed_time(e1) for e0, e1 in ev])))
        # one more step with a CUDA event between stages (the stage breakdown of this rank)
        flush.zero_()
        timing = True
        step()
        torch.cuda.synchronize()
        timing = False
        stages.append({n: round(marks[k - 1][1].elapsed_time(e), 3) for k, (n, e) in enumerate(marks) if k})
        if RECV:
            # compute-only step: the graph-timed step minus the (eager-timed) simulated receives
            recv = sum(v for k, v in stages[-1].items() if k.startswith("recv."))
            per_rank[-1] = per_rank[-1] - recv
            stages[-1]["recv_ms_total"] = round(recv, 3)
        stages[-1]["edges"] = int(s.local_edges)
        stages[-1]["launches_per_pass"] = 1 if COLUMN else len(s.csc)
    del shards
    torch.cuda.empty_cache()
    tmax = max(per_rank)
    t1 = tmax if N == 1 else t1
    # per rank and epoch: (N-1)/N of the layer-1 (F) and layer-2 (H) inputs and the layer-2 dA (H)
    comm_bytes = (N - 1) / N * V * 4 * ((F + 3) // 4 * 4 + 2 * ((H + 3) // 4 * 4))
    comm_ms = comm_bytes / (NVLINK_GBS * 1e9) * 1e3
    out = {"config": name, "N": N, "column_pass": COLUMN, "split_edges": SPLIT, "rank_step_ms": [round(x, 3) for x in per_rank],
           "max_ms": round(tmax, 3), "mean_ms": round(float(np.mean(per_rank)), 3),
           "imbalance": round(tmax / float(np.mean(per_rank)), 3),
           "comm_mb_per_rank": round(comm_bytes / 1e6, 1), "comm_ms_at_nvlink": round(comm_ms, 3),
           "recv_simulated": RECV,
           "stages_slowest_rank": stages[int(np.argmax(per_rank))],
           "stages_all_ranks": stages}
    if t1:
        out["speedup_overlapped"] = round(t1 / tmax, 2)
        out["speedup_serial_comm"] = round(t1 / (tmax + comm_ms), 2)
    print(json.dumps(out), flush=True)
