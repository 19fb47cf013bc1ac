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
    """Test backend: the oracle's ordered gather (seq_sum_rows) on CPU tensors, fp64."""

    def __init__(self, T):
        self.device, self.T = torch.device("cpu"), T

    def zeros(self, rows, cols):
        return torch.zeros((rows, cols), dtype=torch.float64)

    def gather(self, pi, H, out, F, accumulate, mask=None):
        ptr, idx = pi.ptr.numpy(), pi.idx.numpy().astype(np.int64)
        t = H.numpy()[idx]
        if pi.w is not None:
            t = t * pi.w.numpy().astype(np.float64)[:, None]
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


def _worker(rank, world, port, case, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1810_08403_b200 as sg
    from paper_1810_08403_b200 import dist as D

    V, E, F, H, C, gen, T = case
    s, d = (rng.rmat_edges if gen == "rmat" else rng.uniform_edges)(V, E, seed=4)
    g = sg.Graph(V, s, d)
    shard = D.ShardIndex(g, world, rank, split_edges=T, device="cpu")
    W = rng.glorot([(F, H), (H, C)], seed=2, dtype=np.float64)
    m = D.DistGCN(shard, [F, H, C], NumpyCompute(T), weights=W, dtype=torch.float64)
    X = rng.features(V, F, seed=1, dtype=np.float64)
    y = rng.labels(V, C)
    m.load_features(torch.from_numpy(X[shard.begin: shard.begin + shard.rows]))
    m.load_labels(y[shard.begin: shard.begin + shard.rows])
    m.forward()
    m.backward()
    np.savez(os.path.join(outdir, f"r{rank}.npz"), loss=m.loss.numpy(), dW0=m.dW[0].numpy(),
             dW1=m.dW[1].numpy(), a0=m.a[0].numpy(), z1=m.z[1].numpy(), begin=shard.begin)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        return sck.getsockname()[1]


@pytest.mark.parametrize("case", [(40, 300, 6, 5, 3, "uniform", 4096), (64, 900, 7, 4, 3, "rmat", 5)])
def test_dist_gcn_world2_matches_chunked_oracle(case):
    world = 2
    with tempfile.TemporaryDirectory() as outdir:
        mp.start_processes(_worker, args=(world, _free_port(), case, outdir), nprocs=world,
                           join=True, start_method="spawn")
        res = [dict(np.load(os.path.join(outdir, f"r{r}.npz"))) for r in range(world)]
    V, E, F, H, C, gen, T = case
    s, d = (rng.rmat_edges if gen == "rmat" else rng.uniform_edges)(V, E, seed=4)
    part = og.partition_2d(s, d, V, -(-V // world))
    w = og.gcn_edge_weights(s, d, V, np.float32).astype(np.float64)  # the index stores fp32 w_e
    W = rng.glorot([(F, H), (H, C)], seed=2, dtype=np.float64)
    ref = saga.gcn_epoch(part, rng.features(V, F, seed=1, dtype=np.float64), W, rng.labels(V, C), w, T=T)
    for r in range(world):
        b = int(res[r]["begin"])
        n = res[r]["a0"].shape[0]
        # the sharded aggregate is the chunked oracle's, bit for bit (same order)
        assert np.array_equal(res[r]["a0"], ref["a"][0][b: b + n])
        assert np.allclose(res[r]["z1"], ref["z"][1][b: b + n], rtol=0, atol=1e-12)
        assert abs(float(res[r]["loss"][0]) - float(np.ravel(ref["loss"])[0])) <= 1e-12
        assert np.abs(res[r]["dW0"] - ref["grads"][0]).max() <= 1e-12
        assert np.abs(res[r]["dW1"] - ref["grads"][1]).max() <= 1e-12
