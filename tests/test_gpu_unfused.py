"""The unfused chunk-level stage ops and executor (stages.py) on the GPU.

Checks, in order: the SPEC's stage-op known-answer examples; fused == unfused (GCN aggregates
bitwise; G-GCN within tolerance, :426); programs fuse_sag cannot fuse, against a
dense fp64 evaluation of the same traced program (torch autograd on the CPU -- the checker,
SPEC.md:439 "scatter/gather composition equals dense adjacency-matrix formulation"); and the
executor against the fp64 oracle's model epochs."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import assert_close  # noqa: E402
from oracle import graph as og  # noqa: E402
from oracle import rng  # noqa: E402
from oracle import saga  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sg():
    import paper_1810_08403_b200 as m

    return m


def _graph(kind, V, E, seed):
    return (rng.rmat_edges if kind == "rmat" else rng.uniform_edges)(V, E, seed=seed)


# ------------------------------------------------------------------ dense fp64 checker
def _dense(e, b):
    """Evaluate a traced Expr on fp64 CPU torch tensors (autograd on)."""
    op = e.op
    if op in ("input", "param", "pre"):
        return b[e.name]
    a = [_dense(x, b) for x in e.args]
    if op == "matmul":
        return a[0] @ a[1]
    if op == "sigmoid":
        return 1.0 / (1.0 + torch.exp(-a[0]))
    if op == "tanh":
        return torch.tanh(a[0])
    if op == "relu":
        return torch.relu(a[0])
    if op == "add":
        return a[0] + a[1]
    if op == "sub":
        return a[0] - a[1]
    if op == "mul":
        return a[0] * a[1]
    if op == "div":
        return a[0] / a[1]
    if op == "max":
        return torch.maximum(a[0], a[1])
    if op == "gru":
        h, acc, Wz, Uz, Wr, Ur, Wh, Uh = a
        z = torch.sigmoid(acc @ Wz + h @ Uz)
        r = torch.sigmoid(acc @ Wr + h @ Ur)
        c = torch.tanh(acc @ Wh + (r * h) @ Uh)
        return (1 - z) * h + z * c
    raise AssertionError(op)


def _dense_epoch(programs, X, weights, src, dst, w, labels, V):
    """Loss and parameter gradients of the programs as written (no hoist, no chunking)."""
    ps, k = [], 0
    for p in programs:
        d = {}
        for n in p.params:
            d[n] = torch.tensor(np.asarray(weights[k], np.float64), requires_grad=True)
            k += 1
        ps.append(d)
    h = torch.tensor(X, dtype=torch.float64)
    s_t, d_t = torch.from_numpy(src.astype(np.int64)), torch.from_numpy(dst.astype(np.int64))
    wt = torch.tensor(w, dtype=torch.float64).reshape(-1, 1)
    As = []
    for p, P in zip(programs, ps):
        b = dict(P)
        b.update({"edge.src": h[s_t], "edge.dest": h[d_t], "edge.data": wt})
        acc = _dense(p.apply_edge, b)
        A0 = torch.zeros((V, acc.shape[1]), dtype=torch.float64)
        if p.accumulator == "sum":
            A = A0.index_add(0, d_t, acc)
        else:
            A = A0.scatter_reduce(0, d_t[:, None].expand_as(acc), acc, "amax", include_self=False)
        As.append(A.detach().numpy())
        b = dict(P)
        b.update({"vertex": h, "accum": A})
        h = _dense(p.apply_vertex, b)
    loss = torch.nn.functional.cross_entropy(h, torch.from_numpy(np.asarray(labels, np.int64)))
    loss.backward()
    return float(loss), [P[n].grad.numpy() for P in ps for n in P], As


def _run(sg, programs, g, size, T, X, lab, **kw):
    grid = sg.ChunkGrid(g, size, split_edges=T)
    m = sg.UnfusedSAGAModel(programs, grid, **kw)
    m.load_features(X)
    m.load_labels(lab)
    m.forward()
    m.backward()
    torch.cuda.synchronize()
    m.check_status()
    return m


# ------------------------------------------------------------------ SPEC stage-op KATs
def _tiny(sg, V, src, dst, size=None):
    g = sg.Graph(V, np.asarray(src, np.int64), np.asarray(dst, np.int64))
    return sg.ChunkGrid(g, size or V, split_edges=4096)


def test_scatter_chunk_kats(sg):
    from paper_1810_08403_b200 import stages as S

    # single edge 0 -> 1, src features [1, 2] -> edge.src row [1, 2]
    grid = _tiny(sg, 2, [0], [1])
    ec = S.EdgeChunkDev(grid, 0, 0)
    h = torch.tensor([[1.0, 2.0], [5.0, 6.0]], device="cuda")
    et = S.scatter_chunk(h, h, ec)
    assert et["edge.src"].cpu().tolist() == [[1.0, 2.0]]
    assert et["edge.dest"].cpu().tolist() == [[5.0, 6.0]]
    # in-degree 3: the destination's features replicated on 3 rows
    grid = _tiny(sg, 4, [1, 2, 3], [0, 0, 0])
    ec = S.EdgeChunkDev(grid, 0, 0)
    h = torch.arange(8, dtype=torch.float32, device="cuda").reshape(4, 2)
    et = S.scatter_chunk(h, h, ec)
    assert et["edge.dest"].cpu().tolist() == [[0.0, 1.0]] * 3
    assert et["edge.src"].cpu().tolist() == [[2.0, 3.0], [4.0, 5.0], [6.0, 7.0]]


def test_apply_edge_chunk_kats(sg):
    from paper_1810_08403_b200 import program as prog
    from paper_1810_08403_b200 import stages as S

    grid = _tiny(sg, 3, [0, 1], [2, 2])
    ec = S.EdgeChunkDev(grid, 0, 0)
    h = torch.tensor([[1.0, 2.0], [3.0, 4.0], [0.0, 0.0]], device="cuda")
    et = S.scatter_chunk(h, h, ec)
    # passthrough -> acc == edge.src; GCN with edge.data = 1 -> acc == edge.src
    p = prog.make_program(lambda e, q: e.src, lambda v, a, q: a, "sum", {}, 2, 2)
    assert torch.equal(S.apply_edge_chunk(p.apply_edge, et, {}), et["edge.src"])
    ones = dict(et, **{"edge.data": torch.ones((2, 1), device="cuda")})
    p = prog.build_gcn(2, 2)
    assert torch.equal(S.apply_edge_chunk(p.apply_edge, ones, {}), et["edge.src"])
    # GCN ApplyEdge src = [1, 2], data = 0.5 -> [0.5, 1.0]
    half = dict(et, **{"edge.data": torch.full((2, 1), 0.5, device="cuda")})
    assert S.apply_edge_chunk(p.apply_edge, half, {})[0].cpu().tolist() == [0.5, 1.0]


def test_gather_chunk_kats(sg):
    from paper_1810_08403_b200 import stages as S

    # two in-edges of vertex 0 with acc rows [1,2], [3,4]: sum [4,6]; max [3,4] + argmax;
    # vertex 1 has in-degree 0 -> identity, post-filled 0
    grid = _tiny(sg, 3, [1, 2], [0, 0])
    ec = S.EdgeChunkDev(grid, 0, 0)
    acc = torch.tensor([[1.0, 2.0], [3.0, 4.0]], device="cuda")
    A = torch.empty((3, 2), device="cuda")
    S.gather_chunk(acc, ec, "sum", A, first=True)
    assert A.cpu().tolist() == [[4.0, 6.0], [0.0, 0.0], [0.0, 0.0]]
    arg = torch.empty((3, 2), dtype=torch.int32, device="cuda")
    S.gather_chunk(acc, ec, "max", A, first=True, argmax=arg)
    assert A.cpu().tolist() == [[3.0, 4.0], [0.0, 0.0], [0.0, 0.0]]
    assert arg[0].cpu().tolist() == [1, 1]
    # sum backward: dA = [1, 1] -> every d acc row [1, 1]
    dA = torch.tensor([[1.0, 1.0], [0.0, 0.0], [0.0, 0.0]], device="cuda")
    assert S.backward_gather(dA, ec, "sum").cpu().tolist() == [[1.0, 1.0], [1.0, 1.0]]
    # max backward: the non-argmax edge gets 0
    assert S.backward_gather(dA, ec, "max", arg).cpu().tolist() == [[0.0, 0.0], [1.0, 1.0]]
    # ties: the lowest position wins (tensor.py:467-469)
    tie = torch.tensor([[3.0, 4.0], [3.0, 4.0]], device="cuda")
    S.gather_chunk(tie, ec, "max", A, first=True, argmax=arg)
    assert arg[0].cpu().tolist() == [0, 0]


def test_gather_chunk_accumulates_across_chunks(sg):
    """A_j is an in/out accumulator: chunk after chunk continues the same
    per-destination sum order as one pass over the concatenated in-edges."""
    from paper_1810_08403_b200 import stages as S

    V, E = 600, 9000
    s, d = _graph("rmat", V, E, 4)
    g = sg.Graph(V, s, d)
    grid = sg.ChunkGrid(g, 200, split_edges=64)
    h = torch.from_numpy(rng.features(V, 24, seed=2)).cuda()
    for j in range(grid.P):
        j0, nj = grid.begin(j), grid.size(j)
        A = torch.empty((nj, 24), device="cuda")
        ecs = [S.EdgeChunkDev(grid, i, j) for i in range(grid.P) if (i, j) in grid.csc]
        for k, ec in enumerate(ecs):
            i0, ni = grid.begin(ec.i), grid.size(ec.i)
            et = S.scatter_chunk(h[i0:i0 + ni], h[j0:j0 + nj], ec, ("src",))
            S.gather_chunk(et["edge.src"], ec, "sum", A, first=k == 0)
        ref = og.partition_2d(s, d, V, 200)
        want = saga.gcn_propagate_fwd(ref, h.cpu().numpy(), np.ones(E, np.float32), T=64)
        assert np.array_equal(A.cpu().numpy(), want[j0:j0 + nj]), j


# ------------------------------------------------------------------ fused == unfused
@pytest.mark.parametrize("P,T", [(1, 4096), (3, 64)])
def test_unfused_gcn_equals_fused(sg, P, T):
    """fused GCN == unfused GCN bitwise (same accumulation order) -- both layers'
    aggregates; loss and gradients to fp32 round-off of the different GEMM groupings."""
    V, E, dims = 3000, 60000, [40, 16, 5]
    s, d = _graph("rmat", V, E, 2)
    g = sg.Graph(V, s, d)
    size = -(-V // P)
    X = rng.features(V, dims[0], seed=1)
    lab = rng.labels(V, dims[-1])
    fused = sg.gcn_model(sg.ChunkGrid(g, size, split_edges=T), dims)
    W = fused.weights()
    fused.load_features(torch.from_numpy(X))
    fused.load_labels(lab)
    fused.forward()
    fused.backward()
    un = _run(sg, [sg.build_gcn(a, b) for a, b in zip(dims, dims[1:])], g, size, T, X, lab, weights=W)
    for l in range(2):
        assert np.array_equal(un.A[l].detach().cpu().numpy(), fused.layers[l].a.cpu().numpy()), l
    assert abs(un.loss.item() - fused.loss.item()) <= 1e-6 * abs(fused.loss.item())
    for k, (a, b) in enumerate(zip(un.grads(), fused.grads())):
        assert_close(a, b, 1e-5, f"dW{k} unfused vs fused")
    # and both against the fp64 oracle
    part = og.partition_2d(s, d, V, size)
    ref = saga.gcn_epoch(part, X.astype(np.float64), [w.astype(np.float64) for w in W], lab,
                         og.gcn_edge_weights(s, d, V, np.float64), T=T)
    assert abs(un.loss.item() - float(np.ravel(ref["loss"])[0])) <= 1e-4 * float(np.ravel(ref["loss"])[0])
    for k, (a, b) in enumerate(zip(un.grads(), ref["grads"])):
        assert_close(a, b, 1e-4, f"dW{k} unfused vs oracle")


@pytest.mark.parametrize("hoist", [True, False])
def test_unfused_ggcn_vs_fused_and_oracle(sg, hoist):
    """fused G-GCN == unfused within tolerance; unhoisted (edge-rows matmuls, the
    program exactly as written) == hoisted.  Against the fp64 oracle epoch."""
    V, E, dims = 1500, 20000, [24, 12, 4]
    s, d = _graph("uniform", V, E, 5)
    g = sg.Graph(V, s, d)
    X = rng.features(V, dims[0], seed=1)
    lab = rng.labels(V, dims[-1])
    grid = sg.ChunkGrid(g, 500, split_edges=4096, gcn_weights=False)
    fused = sg.ggcn_model(grid, dims)
    W = fused.weights()
    fused.load_features(torch.from_numpy(X))
    fused.load_labels(lab)
    fused.forward()
    fused.backward()
    un = sg.UnfusedSAGAModel([sg.build_ggcn(a, b) for a, b in zip(dims, dims[1:])],
                             sg.ChunkGrid(g, 500, gcn_weights=False), weights=W, hoist=hoist)
    un.load_features(X)
    un.load_labels(lab)
    un.forward()
    un.backward()
    part = og.partition_2d(s, d, V, 500)
    ref, r32 = (saga.ggcn_epoch(part, X.astype(dt), [tuple(x.astype(dt) for x in W[3 * l: 3 * l + 3])
                                                      for l in range(2)], lab) for dt in (np.float64, np.float32))
    for l in range(2):
        assert_close(un.A[l].detach().cpu().numpy(), fused.layers[l].a.cpu().numpy(), 1e-5, f"A{l} vs fused")
        assert_close(un.A[l].detach().cpu().numpy(), ref["cache"][l][3], 1e-5, f"A{l} vs oracle",
                     ref32=r32["cache"][l][3])
    rl = float(np.ravel(ref["loss"])[0])
    assert abs(un.loss.item() - rl) <= 1e-4 * rl
    for k, (a, b, b32) in enumerate(zip(un.grads(), [x for L in ref["grads"] for x in L],
                                        [x for L in r32["grads"] for x in L])):
        assert_close(a, b, 1e-4, f"grad {k}", ref32=b32)


def test_unfused_mpgcn_vs_fused(sg):
    """MP-GCN (max accumulator, hoisted edge network): the chained max gather of the unfused
    executor against the fused executor (aggregates, loss, gradients)."""
    V, E, dims, pool = 2000, 30000, [20, 12, 5], [16, 8]
    s, d = _graph("uniform", V, E, 6)
    g = sg.Graph(V, s, d)
    X = rng.features(V, dims[0], seed=1)
    lab = rng.labels(V, dims[-1])
    fused = sg.mpgcn_model(sg.ChunkGrid(g, 700, gcn_weights=False), dims, pool=pool)
    W = fused.weights()
    fused.load_features(torch.from_numpy(X))
    fused.load_labels(lab)
    fused.forward()
    fused.backward()
    un = _run(sg, [sg.build_mpgcn(a, p, b) for a, p, b in zip(dims, pool, dims[1:])], g, 700, 4096,
              X, lab, weights=W)
    for l in range(2):
        assert_close(un.A[l].detach().cpu().numpy(), fused.layers[l].a.cpu().numpy()[:, :pool[l]],
                     1e-5, f"A{l}")
    assert abs(un.loss.item() - fused.loss.item()) <= 1e-5 * abs(fused.loss.item())
    for k, (a, b) in enumerate(zip(un.grads(), fused.grads())):
        assert_close(a, np.reshape(b, np.shape(a)), 1e-4, f"grad {k}")


# ------------------------------------------------------------------ programs fuse_sag cannot fuse
def _progs(sg, name, dims):
    from paper_1810_08403_b200 import program as prog

    out = []
    for a, b in zip(dims, dims[1:]):
        if name == "tanh_diff":     # tanh(src - dest) * data, sum
            out.append(prog.make_program(lambda e, p: prog.tanh(e.src - e.dest) * e.data,
                                         lambda v, acc, p: prog.relu(prog.matmul(acc, p.W)),
                                         "sum", {"W": (a, b)}, a, b))
        elif name == "max_pair":    # max(src * data, dest), max accumulator
            out.append(prog.make_program(lambda e, p: prog.maximum(e.src * e.data, e.dest),
                                         lambda v, acc, p: prog.relu(prog.matmul(acc, p.W)),
                                         "max", {"W": (a, b)}, a, b))
        elif name == "edge_mlp":    # relu(src @ W_e + dest @ W_d) / (1 + data): matmuls on edge rows
            out.append(prog.make_program(
                lambda e, p: prog.relu(prog.matmul(e.src, p.W_e) + prog.matmul(e.dest, p.W_d)) * e.data,
                lambda v, acc, p: prog.relu(prog.matmul(acc, p.W) + prog.matmul(v, p.W_v)),
                "sum", {"W_e": (a, a), "W_d": (a, a), "W": (a, b), "W_v": (a, b)}, a, b))
        elif name == "gru":         # passthrough sum + GRU ApplyVertex (untyped GG-NN)
            assert a == b
            out.append(prog.make_program(
                lambda e, p: e.src * e.data,
                lambda v, acc, p: prog.gru(v, acc, p.W_z, p.U_z, p.W_r, p.U_r, p.W_h, p.U_h),
                "sum", {k: (a, a) for k in ("W_z", "U_z", "W_r", "U_r", "W_h", "U_h")}, a, b))
    return out


@pytest.mark.parametrize("name,dims,hoist", [("tanh_diff", [20, 12, 5], True),
                                             ("max_pair", [16, 10, 4], True),
                                             ("edge_mlp", [12, 10, 4], True),
                                             ("edge_mlp", [12, 10, 4], False),
                                             ("gru", [8, 8, 8], True)])
def test_unfused_generic_programs_vs_dense(sg, name, dims, hoist):
    """Programs the fused executor rejects run stage by stage and equal the dense fp64
    evaluation of the same traced program, loss and every gradient."""
    from paper_1810_08403_b200 import engine

    progs = _progs(sg, name, dims)
    if name != "edge_mlp" or hoist:
        with pytest.raises(sg.ProgramError):
            engine.lower_programs(progs)          # not fusable: the fused executor refuses it
    V, E = 900, 7000
    s, d = _graph("rmat", V, E, 8)
    g = sg.Graph(V, s, d)
    X = rng.features(V, dims[0], seed=1)
    lab = rng.labels(V, dims[-1])
    m = _run(sg, progs, g, 300, 64, X, lab, hoist=hoist)
    w = og.gcn_edge_weights(s, d, V, np.float64)
    loss, grads, As = _dense_epoch(progs, X.astype(np.float64), m.weights(), s, d, w, lab, V)
    assert abs(m.loss.item() - loss) <= 1e-4 * abs(loss), (m.loss.item(), loss)
    for l in range(2):
        assert_close(m.A[l].detach().cpu().numpy(), As[l], 1e-4, f"A{l}", floor=0.05)
    for k, (a, b) in enumerate(zip(m.grads(), grads)):
        assert_close(a, b, 1e-4, f"{name} grad {k}", floor=0.05)


def test_unfused_train_step_decreases_loss(sg):
    progs = _progs(sg, "tanh_diff", [16, 8, 4])
    V, E = 400, 4000
    s, d = _graph("uniform", V, E, 9)
    m = sg.UnfusedSAGAModel(progs, sg.ChunkGrid(sg.Graph(V, s, d), 200))
    m.load_features(rng.features(V, 16, seed=1))
    m.load_labels(rng.labels(V, 4))
    losses = [float(m.train_step(0.5).item()) for _ in range(5)]
    assert all(b < a for a, b in zip(losses, losses[1:])), losses
