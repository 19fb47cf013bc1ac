"""Oracle vs the reference's own unit tests and the SPEC known-answer examples (CPU only).

Restates the hot-path cases of /root/reference/pkg/tests/test_tensor.py and the
SPEC KATs listed in SURVEY.md §8(c) against the numpy oracle.
"""

import numpy as np
import pytest

from oracle import graph as og
from oracle import primitives as prim
from oracle import rng
from oracle import saga


# ---------------------------------------------------------- test_tensor.py restated
def test_sigmoid_zero():  # test_tensor.py:13-14
    assert prim.sigmoid(np.array([0.0])) == pytest.approx([0.5])


def test_relu():  # test_tensor.py:19-20
    assert np.array_equal(prim.relu(np.array([-1.0, 2.0])), [0, 2])


def test_row_scalar_broadcast():  # test_tensor.py:42-45
    out = prim.mul(np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([[2.0], [10.0]]))
    assert np.array_equal(out, [[2, 4], [30, 40]])


def test_middle_axis_broadcast_rejected():  # test_tensor.py:35-37
    with pytest.raises(prim.ShapeError):
        prim.add(np.zeros((2, 3)), np.zeros((2,)))


def test_nan_surfaces():  # test_tensor.py:51-54
    with pytest.raises(prim.NumericError):
        prim.mul(np.array([1e308]), np.array([1e308]))


def test_matmul_identity_and_selector():  # test_tensor.py:58-65
    m = np.array([[1.0, 2.0], [3.0, 4.0]])
    assert np.array_equal(prim.matmul(np.eye(2), m), m)
    assert np.array_equal(prim.matmul(np.array([[1.0, 0.0]]), np.array([[7.0], [9.0]])), [[7.0]])


def test_matmul_inner_mismatch():  # test_tensor.py:79-81
    with pytest.raises(prim.ShapeError):
        prim.matmul(np.zeros((2, 3)), np.zeros((2, 3)))


def test_relu_gradient_zero_at_zero():  # test_tensor.py:149-155
    x = np.array([0.0, -1.0, 2.0])
    assert np.array_equal(prim.relu_bwd(np.ones(3), x), [0.0, 0.0, 1.0])


def test_take_rows_roundtrip():  # test_tensor.py:198-205
    x = np.array([[1.0, 2.0], [3.0, 4.0], [5.0, 6.0]])
    y = prim.take_rows(x, [2, 0, 2])
    assert np.array_equal(y, [[5, 6], [1, 2], [5, 6]])
    assert np.array_equal(prim.take_rows_bwd(np.ones((3, 2)), [2, 0, 2], 3), [[1, 1], [0, 0], [2, 2]])


def test_take_rows_out_of_range():  # tensor.py:427-428
    with pytest.raises(prim.ShapeError):
        prim.take_rows(np.zeros((2, 2)), [2])


def test_segment_sum():  # test_tensor.py:207-209
    y = prim.segment_sum(np.array([[1.0, 2.0], [3.0, 4.0], [5.0, 6.0]]), [0, 0, 2], 3)
    assert np.array_equal(y, [[4, 6], [0, 0], [5, 6]])


def test_segment_max_with_argmax_grad():  # test_tensor.py:211-218
    x = np.array([[1.0, 5.0], [3.0, 4.0]])
    y, arg = prim.segment_max(x, [0, 0], 2)
    assert np.array_equal(y, [[3, 5], [0, 0]])
    assert np.array_equal(prim.segment_max_bwd(np.ones((2, 2)), arg, 2), [[0, 1], [1, 0]])


def test_segment_max_ties_lowest_row():  # tensor.py:467-469 strict '>'
    x = np.array([[2.0, 1.0], [2.0, 3.0], [0.0, 3.0]])
    _, arg = prim.segment_max(x, [0, 0, 0], 1)
    assert np.array_equal(arg, [[0, 1]])


def test_softmax_cross_entropy_grad_fd():  # test_tensor.py:263-282
    r = np.random.default_rng(5)
    z0 = r.uniform(-1, 1, (4, 3))
    labels = [0, 2, 1, 2]
    loss, p = prim.softmax_cross_entropy(z0, labels)
    g = prim.softmax_cross_entropy_bwd(np.asarray(1.0), p, labels)
    eps = 1e-6
    fd = np.zeros_like(z0)
    for idx in np.ndindex(z0.shape):
        up, dn = z0.copy(), z0.copy()
        up[idx] += eps
        dn[idx] -= eps
        fd[idx] = (prim.softmax_cross_entropy(up, labels)[0] - prim.softmax_cross_entropy(dn, labels)[0]) / (2 * eps)
    assert g == pytest.approx(fd, rel=1e-5, abs=1e-8)
    assert float(loss) > 0


# ---------------------------------------------------------- SPEC KATs
def _part(src, dst, V, size=None):
    return og.partition_2d(np.asarray(src), np.asarray(dst), V, size or V)


def test_scatter_single_edge():
    h = np.array([[1.0, 2.0], [0.0, 0.0]])
    assert np.array_equal(prim.take_rows(h, [0]), [[1.0, 2.0]])


def test_scatter_dest_replicated_by_in_degree():
    h = np.arange(8.0).reshape(4, 2)
    dst = np.array([3, 3, 3])
    assert np.array_equal(prim.take_rows(h, dst), np.repeat(h[3:4], 3, axis=0))


def test_gather_sum_and_max_kat():
    acc = np.array([[1.0, 2.0], [3.0, 4.0]])
    ptr = np.array([0, 2, 2])  # vertex 0 has both edges, vertex 1 none
    assert np.array_equal(saga.seq_sum_rows(ptr, acc), [[4, 6], [0, 0]])
    m, arg = prim.segment_max(acc, [0, 0], 2)
    assert np.array_equal(m, [[3, 4], [0, 0]]) and np.array_equal(arg[0], [1, 1])


def test_gcn_apply_edge_kat():
    assert np.array_equal(prim.mul(np.array([[1.0, 2.0]]), np.array([[0.5]])), [[0.5, 1.0]])


def test_sum_backward_kat():
    assert np.array_equal(prim.segment_sum_bwd(np.array([[1.0, 1.0]]), [0, 0]), [[1, 1], [1, 1]])


def test_ggcn_zero_gates_closed_form():
    V, F = 5, 3
    src = np.array([0, 1, 2, 3, 0])
    dst = np.array([1, 1, 4, 4, 4])
    part = _part(src, dst, V)
    h = rng.features(V, F, dtype=np.float64)
    Z = np.zeros((F, F))
    P_ = h @ Z
    a = saga.ggcn_propagate_fwd(part, h, P_, P_)
    want = np.zeros((V, F))
    np.add.at(want, dst, 0.5 * h[src])
    assert np.allclose(prim.relu(a @ np.eye(F)), np.maximum(want, 0))


def test_gcn_unit_weights_identity_closed_form():
    V, F = 6, 4
    src, dst = rng.uniform_edges(V, 20, seed=4)
    part = _part(src, dst, V, 2)
    h = rng.features(V, F, dtype=np.float64)
    a = saga.gcn_propagate_fwd(part, h, np.ones(len(src)))
    want = np.zeros((V, F))
    np.add.at(want, dst, h[src])
    assert np.allclose(a, want, atol=1e-12)


def test_partition_index_arithmetic():
    part = _part([4], [1], 6, 2)
    assert part.P == 3
    ch = part.chunk(2, 0)
    assert ch["nnz"] == 1 and ch["csc_idx"][0] == 0 and list(ch["csc_ptr"]) == [0, 0, 1]
    assert sum(part.chunk(i, j)["nnz"] for i in range(3) for j in range(3)) == 1


def test_partition_empty_graph():
    part = _part(np.zeros(0, np.int64), np.zeros(0, np.int64), 7, 3)
    assert part.P == 3 and all(part.chunk(i, j)["nnz"] == 0 for i in range(3) for j in range(3))


@pytest.mark.parametrize("seed", range(5))
def test_partition_flatten_is_identity_and_csc_eq_csr(seed):
    V, E = 50, 400
    src, dst = rng.uniform_edges(V, E, seed=seed)
    part = _part(src, dst, V, 13)
    fs, fd = og.flatten_edges(part)
    a = sorted(zip(src.tolist(), dst.tolist()))
    assert sorted(zip(fs.tolist(), fd.tolist())) == a
    for i in range(part.P):
        for j in range(part.P):
            ch = part.chunk(i, j)
            assert sorted(ch["csc_eid"].tolist()) == sorted(ch["csr_eid"].tolist())
            # every edge's endpoints fall in intervals i and j
            assert np.all(src[ch["csc_eid"]] // 13 == i) and np.all(dst[ch["csc_eid"]] // 13 == j)


def test_reencode_star_graph_not_worse():
    V = 8
    src = np.zeros(7, np.int64)
    dst = np.arange(1, 8)
    perm = og.reencode_balance(src, dst, V, 2)
    assert sorted(perm.tolist()) == list(range(V))
    assert og.max_chunk_edges(perm[src], perm[dst], V, 4) <= og.max_chunk_edges(src, dst, V, 4)


@pytest.mark.parametrize("seed", range(4))
def test_reencode_bijection_roundtrip_never_worse(seed):
    V, E = 97, 900
    src, dst = rng.rmat_edges(V, E, seed=seed)
    for P in (1, 2, 3, 5):
        perm = og.reencode_balance(src, dst, V, P)
        assert np.array_equal(np.sort(perm), np.arange(V))
        inv = np.empty_like(perm)
        inv[perm] = np.arange(V)
        assert np.array_equal(inv[perm[src]], src)
        size = -(-V // P)
        assert og.max_chunk_edges(perm[src], perm[dst], V, size) <= og.max_chunk_edges(src, dst, V, size)


def test_scatter_gather_equals_dense_adjacency():  # SPEC.md:439, acceptance 7
    V, F = 40, 5
    src, dst = rng.uniform_edges(V, 300, seed=9)
    part = _part(src, dst, V, 9)
    h = rng.features(V, F, dtype=np.float64)
    A = np.zeros((V, V))
    np.add.at(A, (src, dst), 1.0)
    a = saga.gcn_propagate_fwd(part, h, None, T=4)
    assert np.abs(a - A.T @ h).max() <= 1e-10


def test_split_subgroup_semantics():  # SPEC.md:443 subgroups combined in fixed order
    t = np.arange(10, dtype=np.float64).reshape(5, 2) + 0.25
    ptr = np.array([0, 5])
    out = saga.seq_sum_rows(ptr, t, T=2)
    p0, p1, p2 = t[0] + t[1], t[2] + t[3], t[4] + 0.0
    assert np.array_equal(out[0], ((0.0 + p0) + p1) + p2)


def _ggcn_loss(X, layers, labels, part):
    return float(np.ravel(saga.ggcn_epoch(part, X, layers, labels)["loss"])[0])


def test_ggcn_finite_differences():  # SPEC.md:75, :436, acceptance 2
    V, F, C = 6, 3, 2
    src, dst = rng.uniform_edges(V, 14, seed=21)
    part = _part(src, dst, V, 4)
    X = rng.features(V, F, dtype=np.float64)
    Ls = rng.glorot([(F, F), (F, F), (F, C)], seed=2, dtype=np.float64)
    layers = [tuple(Ls)]
    lab = rng.labels(V, C)
    r = saga.ggcn_epoch(part, X, layers, lab)
    eps = 1e-6
    for k in range(3):
        fd = np.zeros_like(Ls[k])
        for idx in np.ndindex(fd.shape):
            up = [m.copy() for m in Ls]
            dn = [m.copy() for m in Ls]
            up[k][idx] += eps
            dn[k][idx] -= eps
            fd[idx] = (_ggcn_loss(X, [tuple(up)], lab, part) - _ggcn_loss(X, [tuple(dn)], lab, part)) / (2 * eps)
        assert r["grads"][0][k] == pytest.approx(fd, rel=1e-5, abs=1e-8), k


def test_gcn_training_loss_decreases():  # SPEC.md:601, acceptance 8
    V, F, H, C = 20, 6, 8, 3
    src, dst = rng.uniform_edges(V, 80, seed=5)
    part = _part(src, dst, V, 7)
    w = og.gcn_edge_weights(src, dst, V, dtype=np.float64)
    X = rng.features(V, F, dtype=np.float64)
    Ws = rng.glorot([(F, H), (H, C)], dtype=np.float64)
    lab = rng.labels(V, C)
    losses = []
    for _ in range(10):
        r = saga.gcn_epoch(part, X, Ws, lab, w)
        losses.append(float(np.ravel(r["loss"])[0]))
        Ws = saga.sgd(Ws, r["grads"], 0.01)
    assert all(b < a for a, b in zip(losses, losses[1:]))
