"""bf16 storage mode of the propagation kernels (fp32 accumulation), GPU vs oracle.

bf16 rows are widened to fp32 exactly, every edge term and every add is the fp32 path's, and
the output row is rounded to bf16 once per pass (round-to-nearest-even).  So for PASS / GCN the
bf16 result is a deterministic function the oracle can emulate exactly: run the bit-exact fp32
oracle (oracle/saga.py) on the widened inputs, continuing each chunk chain from the widened bf16
accumulator, and round -- the kernels must match it **bit for bit**.  Max / take_rows move values
without arithmetic and are bitwise too.  The gated G-GCN modes (device SFU gate) are checked
against the fp64 oracle on the widened inputs at the stated bf16 tolerance (SURVEY.md §8(c):
normwise 1e-2, elementwise 2e-2 |ref| + 1e-2 max|ref|).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import assert_close, route_relu_masks  # noqa: E402
from oracle import graph as og  # noqa: E402
from oracle import primitives as prim  # noqa: E402
from oracle import rng  # noqa: E402
from oracle import saga  # noqa: E402

pytestmark = pytest.mark.gpu

# elementwise 2e-2 |ref| + 0.5 * 2e-2 * max|ref|: bf16 rounds every stored input, aggregate
# and activation to 8 significant bits (2^-9 = 2e-3 relative), and an output element that is a
# cancelling sum of K such terms keeps an absolute error of ~2^-9 sqrt(K) max|term|, i.e. up to
# a few 1e-3 of max|ref| (measured: Pubmed-shaped h1 8.4e-3 abs at max 2.3); the normwise bar
# (1e-2) bounds the aggregate error
BF16_REL, BF16_FLOOR = 2e-2, 0.5
BF16_NORM = 1e-2


def assert_close_bf16(got, ref, what=""):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    nrm = np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300)
    assert nrm <= BF16_NORM, f"{what}: normwise {nrm:.3e} > {BF16_NORM}"
    assert_close(got, ref, BF16_REL, what, floor=BF16_FLOOR)


@pytest.fixture(scope="module")
def sg():
    import paper_1810_08403_b200 as m

    return m


def to_bf16(x):
    """Round fp32 -> bf16 (RN-even) and return (device bf16 tensor [V, ld8] view, widened fp32)."""
    t = torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.bfloat16)
    V, F = t.shape
    ld = (F + 7) // 8 * 8
    d = torch.zeros((V, ld), dtype=torch.bfloat16, device="cuda")
    d[:, :F] = t.cuda()
    return d[:, :F], t.float().numpy()


def round_bf16(x):
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).to(torch.bfloat16).float().numpy()


def zeros_bf16(V, F):
    ld = (F + 7) // 8 * 8
    return torch.zeros((V, ld), dtype=torch.bfloat16, device="cuda")[:, :F]


def emulate_chain(part, H, w, T, csr=False):
    """The bf16 pass as the kernels define it: per destination interval, each chunk continues
    the chain from the widened bf16 accumulator in fp32 (oracle seq_sum_rows, split rule T)
    and the result is rounded to bf16 when the chunk's pass stores it."""
    F = H.shape[1]
    out = np.zeros((part.V, F), np.float32)
    for a in range(part.P):
        acc = np.zeros((int(part.sizes[a]), F), np.float32)
        for b in range(part.P):
            ch = part.chunk(b, a) if not csr else part.chunk(a, b)
            if ch["nnz"] == 0:
                continue
            key = "csr" if csr else "csc"
            t = H[part.begin(b): part.begin(b) + int(part.sizes[b])][ch[f"{key}_idx"]]
            if w is not None:
                t = t * w[ch[f"{key}_eid"]][:, None]
            acc = round_bf16(saga.seq_sum_rows(ch[f"{key}_ptr"], t, acc, T))
        out[part.begin(a): part.begin(a) + int(part.sizes[a])] = acc
    return out


CASES = [  # kind, V, E, F, P, T
    ("rmat", 4000, 120000, 602, 1, 4096),
    ("uniform", 2500, 11000, 500, 1, 4096),
    ("rmat", 3000, 60000, 128, 3, 256),
    ("uniform", 500, 4000, 16, 1, 4096),
    ("rmat", 800, 20000, 7, 2, 64),
]


@pytest.mark.parametrize("kind,V,E,F,P,T", CASES)
@pytest.mark.parametrize("mode", ["gcn", "pass"])
def test_bf16_propagate_fwd_bitwise(sg, kind, V, E, F, P, T, mode):
    from paper_1810_08403_b200 import _lib
    from paper_1810_08403_b200 import kernels as K

    s, d = (rng.rmat_edges if kind == "rmat" else rng.uniform_edges)(V, E, seed=5)
    size = -(-V // P)
    grid = sg.ChunkGrid(sg.Graph(V, s, d), size, split_edges=T, gcn_weights=(mode == "gcn"))
    Xd, Xw = to_bf16(rng.features(V, F, seed=1))
    out = zeros_bf16(V, F)
    pm = _lib.PROP_GCN if mode == "gcn" else _lib.PROP_PASS
    for j in range(grid.P):
        chain = [i for i in range(grid.P) if (i, j) in grid.csc]
        for k, i in enumerate(chain):
            K.propagate(grid.csc[(i, j)], pm, Xd[grid.begin(i): grid.begin(i) + grid.size(i)],
                        out[grid.begin(j): grid.begin(j) + grid.size(j)], F, accumulate=k > 0)
    part = og.partition_2d(s, d, V, size)
    w = og.gcn_edge_weights(s, d, V, np.float32) if mode == "gcn" else None
    ref = emulate_chain(part, Xw, w, T)
    assert np.array_equal(out.float().cpu().numpy(), ref)


@pytest.mark.parametrize("kind,V,E,F,P,T", CASES)
def test_bf16_gcn_backward_masked_bitwise(sg, kind, V, E, F, P, T):
    from paper_1810_08403_b200 import _lib
    from paper_1810_08403_b200 import kernels as K

    s, d = (rng.rmat_edges if kind == "rmat" else rng.uniform_edges)(V, E, seed=6)
    size = -(-V // P)
    grid = sg.ChunkGrid(sg.Graph(V, s, d), size, split_edges=T)
    Gd, Gw = to_bf16(rng.features(V, F, seed=4))
    Zd, Zw = to_bf16(rng.features(V, F, seed=8))
    out = zeros_bf16(V, F)
    for i in range(grid.P):
        chain = [j for j in range(grid.P) if (i, j) in grid.csr]
        rows = slice(grid.begin(i), grid.begin(i) + grid.size(i))
        for k, j in enumerate(chain):
            K.propagate(grid.csr[(i, j)], _lib.PROP_GCN, Gd[grid.begin(j): grid.begin(j) + grid.size(j)],
                        out[rows], F, accumulate=k > 0,
                        mask=Zd[rows] if k == len(chain) - 1 else None)
    part = og.partition_2d(s, d, V, size)
    w = og.gcn_edge_weights(s, d, V, np.float32)
    ref = prim.relu_bwd(emulate_chain(part, Gw, w, T, csr=True), Zw)
    assert np.array_equal(out.float().cpu().numpy(), ref)


def test_bf16_ggcn_modes_within_bf16_tolerance(sg):
    """GGCN_FWD, GGCN_FWD_S, GGCN_BWD_DST, GGCN_BWD_SRC on bf16 rows vs the fp64 oracle."""
    from paper_1810_08403_b200 import _lib
    from paper_1810_08403_b200 import kernels as K

    V, E, F, T = 1500, 40000, 128, 4096
    s, d = rng.rmat_edges(V, E, seed=3)
    grid = sg.ChunkGrid(sg.Graph(V, s, d), V, split_edges=T, gcn_weights=False)
    part = og.partition_2d(s, d, V, V)
    h = rng.features(V, F, seed=1)
    Pm = rng.features(V, F, seed=2)
    Qm = rng.features(V, F, seed=3)
    Ga = rng.features(V, F, seed=4) * np.float32(0.1)
    HPd, HPw = to_bf16(np.concatenate([h, Pm], 1))
    GQd, GQw = to_bf16(np.concatenate([Ga, Qm], 1))
    hw, Pw, Gw, Qw = HPw[:, :F], HPw[:, F:], GQw[:, :F], GQw[:, F:]
    A, A2, S, dQ, dP, dH = (zeros_bf16(V, F) for _ in range(6))
    ci, ri = grid.csc[(0, 0)], grid.csr[(0, 0)]
    K.propagate(ci, _lib.PROP_GGCN_FWD, HPd, A, F, g_off=F, R=GQd[:, F:])
    K.propagate(ci, _lib.PROP_GGCN_FWD_S, HPd, A2, F, g_off=F, R=GQd[:, F:], out1=S)
    K.propagate(ci, _lib.PROP_GGCN_BWD_DST, HPd, dQ, F, g_off=F, R=GQd, r_off=F)
    K.propagate(ri, _lib.PROP_GGCN_BWD_SRC, GQd, dP, F, g_off=F, R=HPd, r_off=F, out1=dH)
    f64 = lambda x: x.astype(np.float64)  # noqa: E731
    refA = saga.ggcn_propagate_fwd(part, f64(hw), f64(Pw), f64(Qw))
    rQ, rP, rH = saga.ggcn_propagate_bwd(part, f64(hw), f64(Pw), f64(Qw), f64(Gw))
    host = lambda t: t.float().cpu().numpy()  # noqa: E731
    assert torch.equal(A, A2)
    assert_close_bf16(host(A), refA, "A")
    assert_close_bf16(f64(Gw) * host(S), rQ, "dA*S")
    assert_close_bf16(host(dQ), rQ, "dQ")
    assert_close_bf16(host(dP), rP, "dP")
    assert_close_bf16(host(dH), rH, "dH")


def test_bf16_segment_max_and_take_rows_bitwise(sg):
    """Max and row moves are exact in any storage type (tensor.py:424-436, :453-484)."""
    from paper_1810_08403_b200 import ops

    V, E, F = 700, 9000, 24
    s, d = rng.rmat_edges(V, E, seed=9)
    Xd, Xw = to_bf16(rng.features(V, F, seed=1))
    order = np.argsort(d, kind="stable")
    seg = d[order].astype(np.int64)
    rows = torch.from_numpy(s[order].astype(np.int64)).cuda()
    taken = ops.take_rows(Xd, rows)
    assert taken.dtype == torch.bfloat16
    assert np.array_equal(taken.float().cpu().numpy(), Xw[s[order]])
    mx = ops.segment_max(taken, torch.from_numpy(seg).cuda(), V)
    ref, _ = prim.segment_max(Xw[s[order]], seg, V)
    assert np.array_equal(mx.float().cpu().numpy(), ref)


@pytest.mark.parametrize("M,N,K,ta,tb", [(1000, 128, 608, 0, 0), (608, 128, 20000, 1, 1),
                                         (608, 128, 20000, 1, 0), (3000, 48, 128, 0, 1),
                                         (8, 8, 8, 0, 0), (136, 8, 64, 1, 1), (300, 200, 72, 1, 1),
                                         (4096, 64, 608, 0, 0), (128, 48, 40000, 1, 0), (50, 72, 0, 0, 0)])
@pytest.mark.parametrize("out", ["f32", "bf16"])
def test_gemm_tcgen05_bf16(sg, M, N, K, ta, tb, out):
    """tcgen05 kind::f16 GEMM on bf16 operands (all four operand majors, split-K) vs the fp64
    product of the same (widened) bf16 values: the products are exact in fp32, so the only
    error is fp32 accumulation (+ one bf16 rounding of a bf16 output)."""
    from paper_1810_08403_b200 import _lib
    from paper_1810_08403_b200 import kernels as Kn

    r = np.random.default_rng(M * 5 + N + K)
    A = r.uniform(-1, 1, (K, M) if ta else (M, K)).astype(np.float32)
    B = r.uniform(-1, 1, (N, K) if tb else (K, N)).astype(np.float32)
    Ad, Aw = to_bf16(A)
    Bd, Bw = to_bf16(B)
    if out == "bf16" and K >= 8000:
        pytest.skip("split-K GEMMs write fp32 outputs")
    C = zeros_bf16(M, N) if out == "bf16" else torch.zeros((M, (N + 3) // 4 * 4), device="cuda")[:, :N]
    D = zeros_bf16(M, N)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    Kn.gemm(Ad, Bd, C, trans_a=bool(ta), trans_b=bool(tb), relu_out=D, prec=_lib.GEMM_BF16,
            nonfinite=flag)
    A64 = (Aw.T if ta else Aw).astype(np.float64)
    B64 = (Bw.T if tb else Bw).astype(np.float64)
    ref = A64 @ B64
    got = C.float().cpu().numpy()
    absprod = np.abs(A64) @ np.abs(B64)
    bound = (K + 2) * 2.0 ** -24 * absprod + 1e-30
    if out == "bf16":
        bound = bound * (1 + 2.0 ** -8) + 2.0 ** -8 * np.abs(ref)
    assert np.all(np.abs(got - ref) <= bound), float(np.max(np.abs(got - ref) / bound))
    assert np.array_equal(D.float().cpu().numpy(), round_bf16(np.maximum(got, 0)))
    assert int(flag.item()) == 0


def test_gemm_nonfinite_flag_and_nan_relu(sg):
    """Strict mode fused into the GEMM epilogue: a NaN / Inf input row raises the flag, and the
    ReLU dual propagates NaN like np.maximum (tensor.py:207) for every precision."""
    from paper_1810_08403_b200 import _lib
    from paper_1810_08403_b200 import kernels as Kn

    M, N, K = 300, 64, 128
    r = np.random.default_rng(0)
    A = r.uniform(-1, 1, (M, K)).astype(np.float32)
    A[7, 3] = np.nan
    A[11, 5] = np.inf
    B = r.uniform(-1, 1, (K, N)).astype(np.float32)
    for prec in (_lib.GEMM_F32, _lib.GEMM_TF32X3, _lib.GEMM_BF16):
        if prec == _lib.GEMM_BF16:
            Ad, _ = to_bf16(A)
            Bd, _ = to_bf16(B)
        else:
            Ad = torch.from_numpy(A).cuda()
            Bd = torch.from_numpy(B).cuda()
        C = torch.zeros((M, N), device="cuda")
        D = torch.zeros((M, N), device="cuda")
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        Kn.gemm(Ad, Bd, C, relu_out=D, prec=prec, nonfinite=flag)
        assert int(flag.item()) == 1, prec
        d = D.cpu().numpy()
        assert np.isnan(d[7]).all() and not np.isfinite(d[11]).all()
        assert np.isfinite(np.delete(d, [7, 11], 0)).all()
        flag.zero_()
        Kn.gemm(Ad[20:], Bd, C[20:], relu_out=D[20:], prec=prec, nonfinite=flag)
        assert int(flag.item()) == 0, prec


def _bf16_epoch(sg, g, V, F, H, C, dtype):
    from oracle import rng as orng

    grid = sg.ChunkGrid(g, V)
    m = sg.gcn_model(grid, [F, H, C], dtype=dtype)
    X = sg.synthetic_features(V, F, seed=1)
    m.load_features(torch.from_numpy(X))
    m.load_labels(orng.labels(V, C, seed=3))
    m.forward()
    m.backward()
    torch.cuda.synchronize()
    m.check_status()
    return m, X


def _bf16_outs(m):
    hs = [L.hout for L in m.layers[:-1]] + [torch.relu(m.layers[-1].z)]
    return [h.float().cpu().numpy() for h in hs]


def test_bf16_gcn_epoch_pubmed_config_vs_fp64_oracle(sg):
    """bf16 storage mode (SAGAModel(dtype='bf16')) on BASELINE config 1's exact shape vs the
    fp64 oracle at the stated bf16 tolerance: loss, activations, dW0, dW1."""
    V, E, F, H, C = 19717, 88648, 500, 16, 3
    g = sg.uniform_graph(V, E, seed=0)
    m, X = _bf16_epoch(sg, g, V, F, H, C, "bf16")
    part = og.partition_2d(g.src, g.dst, V, V)
    args = (part, X.astype(np.float64), [w.astype(np.float64) for w in m.weights()],
            rng.labels(V, C, seed=3), og.gcn_edge_weights(g.src, g.dst, V, np.float64))
    free = saga.gcn_epoch(*args)
    ref = saga.gcn_epoch(*args, masks=_bf16_masks(m, free["z"], "pubmed bf16"))
    rl = float(np.ravel(ref["loss"])[0])
    assert abs(m.loss.item() - rl) <= BF16_NORM * abs(rl), (m.loss.item(), rl)
    for k, (got, want) in enumerate(zip(_bf16_outs(m), ref["out"])):
        assert_close_bf16(got, want, f"h{k + 1}")
    for k, (got, want) in enumerate(zip(m.grads(), ref["grads"])):
        assert_close_bf16(got, want, f"dW{k}")


def _bf16_masks(m, z_ref, what):
    """The bf16 run's ReLU masks (h_out > 0 of the hidden layers, z > 0 of the top) routed into
    the oracle's backward; flips allowed only at bf16-level kinks (|z| <= 5e-3 max|z|)."""
    zg = [L.hout.float().cpu().numpy() for L in m.layers[:-1]] + [m.layers[-1].z.cpu().numpy()]
    return route_relu_masks(zg, z_ref, tie=5e-3, max_frac=5e-3, what=what)


def test_bf16_gcn_epoch_reddit_config_vs_fp64_oracle(sg, reddit_oracle):
    """The bf16 Reddit epoch the bench reports (BASELINE config 2, full size) vs the fp64
    full-size oracle (live, routed through the bf16 run's ReLU masks) at the bf16 tolerance."""
    from oracle import fullsize as fs

    R = reddit_oracle
    m, _ = _bf16_epoch(sg, R["g"], R["V"], R["F"], R["H"], R["C"], "bf16")
    f = R["fwd"]
    grads = fs.gcn_backward(f, _bf16_masks(m, f["z"], "reddit bf16"))
    rl = float(np.ravel(f["loss"])[0])
    assert abs(m.loss.item() - rl) <= BF16_NORM * abs(rl), (m.loss.item(), rl)
    rows = np.random.default_rng(11).choice(R["V"], 256, replace=False)
    for k, h in enumerate(_bf16_outs(m)):
        assert_close_bf16(h[rows], f["out"][k][rows], f"h{k + 1} rows")
    for k, (got, want) in enumerate(zip(m.grads(), grads)):
        assert_close_bf16(got, want, f"dW{k}")


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("bad", [np.nan, -np.inf])
def test_strict_mode_raises_on_nonfinite_preactivation(sg, dtype, bad):
    """tensor.py:161-163: a non-finite op output raises NumericError.  A NaN / -Inf feature
    reaches the aggregate and the pre-activation z = a W; the GEMM epilogue's flag makes
    check_status() raise (the ReLU propagates NaN like np.maximum, so it cannot hide it)."""
    from paper_1810_08403_b200.errors import NumericError

    V, E, F, H, C = 500, 6000, 64, 16, 4
    s, d = rng.rmat_edges(V, E, seed=2)
    g = sg.Graph(V, s, d)
    grid = sg.ChunkGrid(g, V)
    m = sg.gcn_model(grid, [F, H, C], dtype=dtype)
    X = rng.features(V, F, seed=1)
    m.load_features(torch.from_numpy(X))
    m.load_labels(rng.labels(V, C))
    m.forward()
    m.backward()
    m.check_status()                       # clean inputs: no flag
    X[int(s[0])] = bad                     # a source row with at least one out-edge
    m.load_features(torch.from_numpy(X))
    m.forward()
    m.backward()
    with pytest.raises(NumericError):
        m.check_status()
    m_off = sg.gcn_model(grid, [F, H, C], dtype=dtype, strict=False)
    m_off.load_features(torch.from_numpy(X))
    m_off.load_labels(rng.labels(V, C))
    m_off.forward()
    m_off.backward()
    m_off.check_status()                   # strict=False: no check (reference STRICT = False)
