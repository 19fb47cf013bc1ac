"""Pin the oracle to the real reference: bitwise vs golden fixtures (CPU only)."""

import numpy as np
import pytest

from conftest import GOLDEN_CASES, load_golden
from oracle import graph as og
from oracle import saga

DT = {"f64": np.float64, "f32": np.float32}


def sc(x):
    return float(np.ravel(x)[0])


def _grid(g, interval_size=None):
    V = int(g["V"])
    return og.partition_2d(g["src_in"], g["dst_in"], V, interval_size or V)


@pytest.mark.parametrize("case", GOLDEN_CASES)
@pytest.mark.parametrize("tag", ["f64", "f32"])
def test_gcn_reference_composition_bitwise(case, tag):
    g = load_golden(case)
    V = int(g["V"])
    X = g[f"gcn_{tag}_X"]
    Ws = [g[f"gcn_{tag}_W0"], g[f"gcn_{tag}_W1"]]
    r = saga.ref_gcn_epoch(X, Ws, g["labels"], g["src"], g["dst"], g[f"gcn_{tag}_w"], V)
    assert r["loss"].dtype == DT[tag]
    assert np.array_equal(np.ravel(r["loss"]), np.ravel(g[f"gcn_{tag}_loss"]))
    for l in range(2):
        assert np.array_equal(r["a"][l], g[f"gcn_{tag}_a{l}"])
        assert np.array_equal(r["z"][l], g[f"gcn_{tag}_z{l}"])
        assert np.array_equal(r["grads"][l], g[f"gcn_{tag}_dW{l}"])


@pytest.mark.parametrize("case", GOLDEN_CASES)
@pytest.mark.parametrize("tag", ["f64", "f32"])
def test_gcn_chunked_p1_bitwise(case, tag):
    """Chunked engine semantics at P=1, no split == the reference tape, bit for bit."""
    g = load_golden(case)
    V = int(g["V"])
    part = _grid(g)
    w = og.gcn_edge_weights(g["src_in"], g["dst_in"], V, dtype=DT[tag])
    X = g[f"gcn_{tag}_X"]
    Ws = [g[f"gcn_{tag}_W0"], g[f"gcn_{tag}_W1"]]
    r = saga.gcn_epoch(part, X, Ws, g["labels"], w)
    assert np.array_equal(np.ravel(r["loss"]), np.ravel(g[f"gcn_{tag}_loss"]))
    for l in range(2):
        assert np.array_equal(r["a"][l], g[f"gcn_{tag}_a{l}"])
        assert np.array_equal(r["grads"][l], g[f"gcn_{tag}_dW{l}"])


@pytest.mark.parametrize("case", GOLDEN_CASES)
@pytest.mark.parametrize("P", [2, 4])
def test_gcn_chunked_grid_matches_reference(case, P):
    """SPEC acceptance 1: chunked engine (P>1, split subgroups) vs dense <= 1e-10 at fp64."""
    g = load_golden(case)
    V = int(g["V"])
    part = _grid(g, -(-V // P))
    w = og.gcn_edge_weights(g["src_in"], g["dst_in"], V, dtype=np.float64)
    Ws = [g["gcn_f64_W0"], g["gcn_f64_W1"]]
    r = saga.gcn_epoch(part, g["gcn_f64_X"], Ws, g["labels"], w, T=3)
    assert abs(sc(r["loss"]) - sc(g["gcn_f64_loss"])) <= 1e-10
    for l in range(2):
        assert np.abs(r["grads"][l] - g[f"gcn_f64_dW{l}"]).max() <= 1e-10
        assert np.abs(r["a"][l] - g[f"gcn_f64_a{l}"]).max() <= 1e-10


@pytest.mark.parametrize("case", GOLDEN_CASES)
@pytest.mark.parametrize("tag", ["f64", "f32"])
def test_ggcn_hoisted_chunked_bitwise(case, tag):
    g = load_golden(case)
    V = int(g["V"])
    part = _grid(g)
    layers = [tuple(g[f"ggcn_{tag}_L{l}_{k}"] for k in range(3)) for l in range(2)]
    r = saga.ggcn_epoch(part, g[f"gcn_{tag}_X"], layers, g["labels"])
    assert np.array_equal(np.ravel(r["loss"]), np.ravel(g[f"ggcnh_{tag}_loss"]))
    for l in range(2):
        for k in range(3):
            assert np.array_equal(r["grads"][l][k], g[f"ggcnh_{tag}_dL{l}_{k}"]), (l, k)


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_ggcn_hoist_semantics_preserving(case):
    """hoisted vs unhoisted G-GCN within 1e-12 at fp64; matmul rows 2|E| -> 2|V| (:249)."""
    g = load_golden(case)
    V, E = int(g["V"]), int(g["E"])
    assert abs(sc(g["ggcnh_f64_loss"]) - sc(g["ggcnu_f64_loss"])) <= 1e-12
    for l in range(2):
        for k in range(3):
            assert np.abs(g[f"ggcnh_f64_dL{l}_{k}"] - g[f"ggcnu_f64_dL{l}_{k}"]).max() <= 1e-12
    # two layers, two gate matmuls each: hoisted counts V rows, unhoisted E rows
    assert int(g["ggcnh_f64_mm_edge"]) == 2 * 2 * V
    assert int(g["ggcnu_f64_mm_edge"]) == 2 * 2 * E


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_ggcn_chunked_grid_matches_reference(case):
    g = load_golden(case)
    V = int(g["V"])
    part = _grid(g, -(-V // 3))
    layers = [tuple(g[f"ggcn_f64_L{l}_{k}"] for k in range(3)) for l in range(2)]
    r = saga.ggcn_epoch(part, g["gcn_f64_X"], layers, g["labels"], T=4)
    assert abs(sc(r["loss"]) - sc(g["ggcnh_f64_loss"])) <= 1e-10
    for l in range(2):
        for k in range(3):
            assert np.abs(r["grads"][l][k] - g[f"ggcnh_f64_dL{l}_{k}"]).max() <= 1e-10


@pytest.mark.parametrize("case", GOLDEN_CASES)
@pytest.mark.parametrize("tag", ["f64", "f32"])
def test_mpgcn_oracle_bitwise(case, tag):
    """MP-GCN (max accumulator) oracle == the real reference, bit for bit."""
    g = load_golden(case)
    V = int(g["V"])
    part = _grid(g)
    layers = [tuple(g[f"mpgcn_{tag}_L{l}_{k}"] for k in range(3)) for l in range(2)]
    r = saga.mpgcn_epoch(part, g[f"gcn_{tag}_X"], layers, g["labels"])
    assert np.array_equal(np.ravel(r["loss"]), np.ravel(g[f"mpgcnh_{tag}_loss"]))
    for l in range(2):
        for k in range(3):
            assert np.array_equal(r["grads"][l][k], g[f"mpgcnh_{tag}_dL{l}_{k}"]), (l, k)


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_mpgcn_hoist_semantics_preserving(case):
    g = load_golden(case)
    assert abs(sc(g["mpgcnh_f64_loss"]) - sc(g["mpgcnu_f64_loss"])) <= 1e-12
    for l in range(2):
        for k in range(3):
            assert np.abs(g[f"mpgcnh_f64_dL{l}_{k}"] - g[f"mpgcnu_f64_dL{l}_{k}"]).max() <= 1e-12


@pytest.mark.parametrize("case", GOLDEN_CASES)
def test_mpgcn_oracle_2d_grid_matches_one_chunk(case):
    """The 2D-grid edge order (source-interval-major flattening) changes only summation
    order and tie positions: loss and gradients agree with P = 1 to fp64 round-off."""
    g = load_golden(case)
    V = int(g["V"])
    layers = [tuple(g[f"mpgcn_f64_L{l}_{k}"] for k in range(3)) for l in range(2)]
    r1 = saga.mpgcn_epoch(og.partition_2d(g["src_in"], g["dst_in"], V, V), g["gcn_f64_X"], layers,
                          g["labels"])
    r3 = saga.mpgcn_epoch(og.partition_2d(g["src_in"], g["dst_in"], V, -(-V // 3)), g["gcn_f64_X"],
                          layers, g["labels"])
    assert abs(sc(r1["loss"]) - sc(r3["loss"])) <= 1e-12
    for l in range(2):
        assert np.array_equal(r1["cache"][l][2], r3["cache"][l][2])  # max values are order-free
        for k in range(3):
            assert np.abs(r1["grads"][l][k] - r3["grads"][l][k]).max() <= 1e-12


@pytest.mark.parametrize("case", GOLDEN_CASES)
@pytest.mark.parametrize("tag", ["f64", "f32"])
def test_commnet_oracle_bitwise(case, tag):
    """CommNet (passthrough edge, ReLU(W_H h + W_C accum)) oracle ==
    the real reference, bit for bit."""
    g = load_golden(case)
    part = _grid(g)
    layers = [tuple(g[f"commnet_{tag}_L{l}_{k}"] for k in range(2)) for l in range(2)]
    r = saga.commnet_epoch(part, g[f"gcn_{tag}_X"], layers, g["labels"])
    assert np.array_equal(np.ravel(r["loss"]), np.ravel(g[f"commnet_{tag}_loss"]))
    for l in range(2):
        assert np.array_equal(r["a"][l], g[f"commnet_{tag}_a{l}"])
        assert np.array_equal(r["z"][l], g[f"commnet_{tag}_z{l}"])
        for k in range(2):
            assert np.array_equal(r["grads"][l][k], g[f"commnet_{tag}_dL{l}_{k}"]), (l, k)


def _ggnn_layers(g, tag):
    layers = []
    for l in range(2):
        As = [g[f"ggnn_{tag}_L{l}_A{t}"] for t in range(3)]
        layers.append((As,) + tuple(g[f"ggnn_{tag}_L{l}_{k}"] for k in range(6)))
    return layers


@pytest.mark.parametrize("name", GOLDEN_CASES)
@pytest.mark.parametrize("tag", ["f64", "f32"])
def test_ggnn_oracle_bitwise(name, tag):
    """GG-NN oracle (P = 1, no split) == the real reference's tape (typed per-vertex hoist +
    select_rows_by_label + GRU) bit for bit: loss, logits, aggregates, every gradient."""
    g = load_golden(name)
    V = int(g["V"])
    types_in = np.empty_like(g["ggnn_types"])
    part = og.partition_2d(g["src_in"], g["dst_in"], V, V)
    types_in[part.csc_eid] = g["ggnn_types"]
    layers = _ggnn_layers(g, tag)
    res = saga.ggnn_epoch(part, g[f"gcn_{tag}_X"], layers, g[f"ggnn_{tag}_Wo"], types_in, g["labels"])
    assert np.array_equal(np.ravel(res["loss"]), np.ravel(g[f"ggnn_{tag}_loss"]))
    assert np.array_equal(res["logits"], g[f"ggnn_{tag}_logits"])
    for l in range(2):
        assert np.array_equal(res["a"][l], g[f"ggnn_{tag}_a{l}"])
        assert np.array_equal(res["out"][l], g[f"ggnn_{tag}_h{l}"])
        for t in range(3):
            assert np.array_equal(res["grads"][l][0][t], g[f"ggnn_{tag}_dL{l}_A{t}"]), (l, t)
        for k in range(6):
            assert np.array_equal(res["grads"][l][1 + k], g[f"ggnn_{tag}_dL{l}_{k}"]), (l, k)
    assert np.array_equal(res["grads_Wo"], g[f"ggnn_{tag}_dWo"])


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_ggnn_oracle_2d_grid_matches_reference(name):
    """P = 3 grid with split subgroups: same function, fp64 rounding only."""
    g = load_golden(name)
    V = int(g["V"])
    part1 = og.partition_2d(g["src_in"], g["dst_in"], V, V)
    types_in = np.empty_like(g["ggnn_types"])
    types_in[part1.csc_eid] = g["ggnn_types"]
    part = og.partition_2d(g["src_in"], g["dst_in"], V, -(-V // 3))
    res = saga.ggnn_epoch(part, g["gcn_f64_X"], _ggnn_layers(g, "f64"), g["ggnn_f64_Wo"], types_in,
                          g["labels"], T=3)
    assert abs(float(np.ravel(res["loss"])[0]) - float(np.ravel(g["ggnn_f64_loss"])[0])) < 1e-12
    for l in range(2):
        for k in range(6):
            assert np.allclose(res["grads"][l][1 + k], g[f"ggnn_f64_dL{l}_{k}"], rtol=1e-9, atol=1e-12)
        for t in range(3):
            assert np.allclose(res["grads"][l][0][t], g[f"ggnn_f64_dL{l}_A{t}"], rtol=1e-9, atol=1e-12)
