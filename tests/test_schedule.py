"""Chunk scheduler cost model (paper_1810_08403_b200/schedule.py), CPU only."""

import numpy as np
import pytest

from paper_1810_08403_b200 import schedule as S
from paper_1810_08403_b200.errors import BudgetError, ConfigError
from oracle import rng


class _G:
    def __init__(self, V, E, seed=0, kind="rmat"):
        self.V = V
        self.src, self.dst = (rng.rmat_edges if kind == "rmat" else rng.uniform_edges)(V, E, seed=seed)


@pytest.fixture(scope="module")
def reddit_like():
    # the Reddit-shaped vertex count and degree mix at 1/40 of the edges (CPU-test sized)
    return _G(232965, 114615892 // 40)


def test_resident_single_gpu_picks_p1(reddit_like):
    s = S.build_schedule(reddit_like, [602, 128, 41])
    assert s.mode == "resident" and s.P == 1 and s.interval_size == reddit_like.V
    # every extra interval adds launches and an accumulator read-modify-write
    t = [sum(S.pass_compute_ms(reddit_like.V, len(reddit_like.src), f, P, S.chunk_stats(
        reddit_like.src, reddit_like.dst, reddit_like.V, P)[1]) for f in (602, 128)) for P in (1, 2, 8)]
    assert t[0] < t[1] < t[2]


def test_sharded_picks_world(reddit_like):
    for w in (2, 4, 8):
        s = S.build_schedule(reddit_like, [602, 128, 41], world=w)
        assert s.mode == "sharded" and s.P == w and s.interval_size == -(-reddit_like.V // w)


def test_streaming_smallest_feasible_p(reddit_like):
    dims = [602, 128, 41]
    V = reddit_like.V
    budget = 400 << 20
    s = S.build_schedule(reddit_like, dims, budget=budget)
    assert s.mode == "streaming" and s.strategy == "locality"
    assert s.resident_bytes <= budget
    # the next smaller candidate does not fit
    smaller = [p for p in (1, 2, 4, 8, 16, 32, 64, 128) if p < s.P]
    for p in smaller:
        mx, _ = S.chunk_stats(reddit_like.src, reddit_like.dst, V, p)
        assert S.streaming_working_set(V, dims, p, mx) > budget
    assert s.swap_h2d_bytes > 0 and s.makespan_ms > 0
    for L in s.layers:   # two resources: makespan >= max(compute, transfer)
        assert L.makespan_ms >= max(L.compute_ms, L.transfer_ms)


def test_locality_moves_fewest_bytes(reddit_like):
    """in the streaming regime swap_bytes(Locality) <= the other strategies."""
    V, E = reddit_like.V, len(reddit_like.src)
    for P in (2, 4, 16):
        loc = sum(S.swap_bytes(V, E, 602, P, "locality"))
        assert loc <= sum(S.swap_bytes(V, E, 602, P, "dest_order"))
        assert loc < sum(S.swap_bytes(V, E, 602, P, "stage_based"))
    assert S.swap_bytes(V, E, 602, 1, "locality") == S.swap_bytes(V, E, 602, 1, "dest_order")


def test_infeasible_budget_and_bad_strategy(reddit_like):
    with pytest.raises(BudgetError):
        S.build_schedule(reddit_like, [602, 128, 41], budget=1 << 20)
    with pytest.raises(ConfigError):
        S.build_schedule(reddit_like, [602, 128, 41], strategy="fastest")


def test_ggcn_resident_bytes_exceed_gcn():
    assert S.resident_bytes(1000, 5000, [64, 32, 4], "ggcn") > S.resident_bytes(1000, 5000, [64, 32, 4])
    assert np.all(np.array(S.chunk_stats(np.array([0, 5]), np.array([9, 1]), 10, 2)) == [1, 2])


def test_run_bench_unbounded_rows_equal_swaps():
    """SPEC.md:610 (P = 1 -> identical rows): with no budget every strategy is resident with
    the same swap bytes; the config is validated like run_train's."""
    import paper_1810_08403_b200 as sg
    import paper_1810_08403_b200.engine as E

    g = sg.uniform_graph(500, 4000, seed=0)
    rows = [S.build_schedule(g, [16, 8, 4], strategy=s) for s in S.STRATEGIES]
    assert {(r.mode, r.swap_h2d_bytes, r.swap_d2h_bytes) for r in rows} == {("resident", 0, 0)}
    with pytest.raises(sg.ConfigError):
        E.run_bench({"model": "gcn", "V": 10, "E": 10, "features": 4, "classes": 2, "bogus": 1})
    with pytest.raises(sg.ConfigError):
        E.run_bench({"model": "mpgcn", "V": 10, "E": 10, "features": 4, "classes": 2})
