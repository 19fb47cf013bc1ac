"""Multi-GPU engine host logic on CPU: world_size 2 over gloo, oracle as the compute backend.

The sharding / all-gather / ordering / all-reduce logic of paper_1810_08403_b200.dist is
exactly what runs on GPUs (NCCL + libsagann kernels); here the per-chunk compute is the
numpy oracle, so the test checks that the distributed dataflow reproduces the chunked
oracle with P = world.
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import graph as og
from oracle import primitives as prim
from oracle import rng
from oracle import saga


class NumpyCompute:
    """Test backend: the oracle's ordered gathers (seq_sum_rows) on CPU tensors, fp64."""

    def __init__(self, T):
        self.device, self.T = torch.device("cpu"), T

    def zeros(self, rows, cols):
        return torch.zeros((rows, cols), dtype=torch.float64)

    def propagate(self, pi, mode, Gm, out, F, *, g_off=0, R=None, r_off=0, out1=None, mask=None,
                  accumulate=False):
        from paper_1810_08403_b200 import _lib

        ptr, idx = pi.ptr.numpy(), pi.idx.numpy().astype(np.int64)
        rows = saga.local_rows(ptr)
        Gn = Gm.numpy()
        if mode == _lib.PROP_GCN:
            t = Gn[idx][:, :F]
            if pi.w is not None:
                t = t * pi.w.numpy().astype(np.float64)[:, None]
        elif mode in (_lib.PROP_GGCN_FWD, _lib.PROP_GGCN_FWD_S):  # G = [h | P], R = Q of the rows
            eta = prim.sigmoid(Gn[idx, g_off:g_off + F] + R.numpy()[rows, :F])
            t = eta * Gn[idx, :F]
            if mode == _lib.PROP_GGCN_FWD_S:   # S = sum (h eta)(1 - eta)
                base1 = out1.numpy().copy() if accumulate else None
                out1.copy_(torch.from_numpy(saga.seq_sum_rows(ptr, (Gn[idx, :F] * eta) * (1.0 - eta), base1,
                                                              self.T, F=F, dtype=np.float64)))
        elif mode == _lib.PROP_GGCN_BWD_DST:  # G = [h | P] sources, R = [dA | Q] rows
            Rn = R.numpy()
            eta = prim.sigmoid(Gn[idx, g_off:g_off + F] + Rn[rows, r_off:r_off + F])
            t = prim.sigmoid_bwd(Rn[rows, :F] * Gn[idx, :F], eta)
        elif mode == _lib.PROP_GGCN_BWD_SRC:  # G = [dA | Q] destinations, R = [h | P] rows
            Rn = R.numpy()
            Gu = Gn[idx, :F]
            eta = prim.sigmoid(Rn[rows, r_off:r_off + F] + Gn[idx, g_off:g_off + F])
            t = prim.sigmoid_bwd(Gu * Rn[rows, :F], eta)
            base1 = out1.numpy().copy() if accumulate else None
            out1.copy_(torch.from_numpy(saga.seq_sum_rows(ptr, Gu * eta, base1, self.T, F=F,
                                                          dtype=np.float64)))
        else:
            raise AssertionError(mode)
        base = out.numpy().copy() if accumulate else None
        res = saga.seq_sum_rows(ptr, t, base, self.T, F=F, dtype=np.float64)
        if mask is not None:
            res = prim.relu_bwd(res, mask.numpy())
        out.copy_(torch.from_numpy(res))

    def gemm(self, A, B, C, trans_a=False, trans_b=False, relu_out=None):
        a = A.numpy().T if trans_a else A.numpy()
        b = B.numpy().T if trans_b else B.numpy()
        C.copy_(torch.from_numpy(a @ b))
        if relu_out is not None:
            relu_out.copy_(torch.from_numpy(np.maximum(a @ b, 0.0)))

    def add(self, a, b, out):
        out.copy_(a + b)

    def mul(self, a, b, out):
        out.copy_(a * b)

    def relu_bwd(self, g, z, out):
        out.copy_(torch.from_numpy(prim.relu_bwd(g.numpy(), z.numpy())))

    def xent(self, Z, labels, loss, dZ, err, n_total):
        z = Z.numpy()
        lg = np.maximum(z, 0.0)
        lab = labels.numpy()
        m = lg.max(axis=1, keepdims=True)
        ez = np.exp(lg - m)
        d = ez.sum(axis=1, keepdims=True)
        p = ez / d
        logp = (lg - m) - np.log(d)
        loss.fill_(-logp[np.arange(len(lab)), lab].sum() / n_total)
        g = p.copy()
        g[np.arange(len(lab)), lab] -= 1.0
        dZ.copy_(torch.from_numpy(prim.relu_bwd(g / n_total, z)))

    def sgd(self, W, dW, lr):
        W.sub_(lr * dW)


def _case_params(model, F, H, C):
    if model == "gcn":
        return rng.glorot([(F, H), (H, C)], seed=2, dtype=np.float64)
    return rng.glorot([(F, F), (F, F), (F, H), (H, H), (H, H), (H, C)], seed=2, dtype=np.float64)


def _worker(rank, world, port, case, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1810_08403_b200 as sg
    from paper_1810_08403_b200 import dist as D

    model, V, E, F, H, C, gen, T, column = case
    s, d = (rng.rmat_edges if gen == "rmat" else rng.uniform_edges)(V, E, seed=4)
    g = sg.Graph(V, s, d)
    shard = D.ShardIndex(g, world, rank, split_edges=T, device="cpu", gcn_weights=model == "gcn",
                         column=column)
    m = D.DistSAGA(shard, [F, H, C], NumpyCompute(T), model=model,
                   weights=_case_params(model, F, H, C), dtype=torch.float64)
    X = rng.features(V, F, seed=1, dtype=np.float64)
    y = rng.labels(V, C)
    m.load_features(torch.from_numpy(X[shard.vertices]))
    m.load_labels(y[shard.vertices])
    m.forward()
    m.backward()
    out = dict(loss=m.loss.numpy(), a0=m.a[0].numpy(), z1=m.z[1].numpy(), begin=shard.begin,
               perm=shard.perm)
    for k, gr in enumerate(m.grads()):
        out[f"g{k}"] = gr
    np.savez(os.path.join(outdir, f"r{rank}.npz"), **out)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        return sck.getsockname()[1]


CASES = [("gcn", 40, 300, 6, 5, 3, "uniform", 4096), ("gcn", 64, 900, 7, 4, 3, "rmat", 5),
         ("ggcn", 48, 500, 6, 5, 3, "rmat", 7), ("ggcn", 30, 200, 5, 4, 3, "uniform", 4096)]


@pytest.mark.parametrize("column", [True, False])
@pytest.mark.parametrize("case", CASES)
def test_dist_world2_matches_chunked_oracle(case, column):
    """Sharded epoch (re-encoded by reencode_balance) == the chunked oracle on the re-encoded
    graph: with column passes (the default) the P = 1 oracle (each row's in-edges in ascending
    global source), with per-chunk passes the P = world oracle (chained in ascending block);
    aggregates bitwise, loss and gradients to fp64 rounding."""
    world = 2
    with tempfile.TemporaryDirectory() as outdir:
        mp.start_processes(_worker, args=(world, _free_port(), case + (column,), outdir), nprocs=world,
                           join=True, start_method="spawn")
        res = [dict(np.load(os.path.join(outdir, f"r{r}.npz"))) for r in range(world)]
    model, V, E, F, H, C, gen, T = case
    s, d = (rng.rmat_edges if gen == "rmat" else rng.uniform_edges)(V, E, seed=4)
    perm = og.reencode_balance(s, d, V, world)
    assert np.array_equal(res[0]["perm"], perm)  # native re-encode == oracle restatement
    s, d = perm[s], perm[d]
    inv = np.argsort(perm)
    X = rng.features(V, F, seed=1, dtype=np.float64)[inv]
    y = rng.labels(V, C)[inv]
    part = og.partition_2d(s, d, V, V if column else -(-V // world))
    P = _case_params(model, F, H, C)
    if model == "gcn":
        w = og.gcn_edge_weights(s, d, V, np.float32).astype(np.float64)  # the index stores fp32 w_e
        ref = saga.gcn_epoch(part, X, P, y, w, T=T)
        a0, z1, grads = ref["a"][0], ref["z"][1], ref["grads"]
    else:
        ref = saga.ggcn_epoch(part, X, [tuple(P[0:3]), tuple(P[3:6])], y, T=T)
        a0, z1 = None, ref["cache"][1][4]
        grads = [g for lay in ref["grads"] for g in lay]
    for r in range(world):
        b = int(res[r]["begin"])
        n = res[r]["z1"].shape[0]
        if a0 is not None:
            # the sharded aggregate is the chunked oracle's, bit for bit (same order)
            assert np.array_equal(res[r]["a0"], a0[b: b + n])
        assert np.allclose(res[r]["z1"], z1[b: b + n], rtol=0, atol=1e-12)
        assert abs(float(res[r]["loss"][0]) - float(np.ravel(ref["loss"])[0])) <= 1e-12
        errs = [float(np.abs(res[r][f"g{k}"] - g).max()) for k, g in enumerate(grads)]
        assert max(errs) <= 1e-12, (r, errs)
