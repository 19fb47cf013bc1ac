"""Chunk scheduler: interval size (P) and visit order per layer from a cost model and a budget.

The reference's scheduler (``build_schedule(df, strategy, budget)`` and
``simulate_timeline``) orders chunk operators under a device-memory budget and models a
compute + transfer overlap; PAPER.md:324-342 motivates it with PCIe-era GPUs that could not hold
the graph.  On a 180-GB B200 the same decision has three outcomes, which this module makes from
measured rates (the constants below cite the measurement):

* **resident** (the whole layer fits): P = 1.  Every extra source interval costs one more launch
  and tail per destination column plus a read-modify-write of the accumulator A_j, and the pass
  is bound by L2 -> SM gather bandwidth, not DRAM, so tiling sources to L2-sized intervals does
  not pay (profiles/r01_tile_ab.txt: Reddit F = 602 P = 1/2/4/8 -> 16.0/16.3/22.6/51.8 ms);
* **sharded** over ``world`` GPUs: P = world (dest-interval sharding, dist.py);
* **streaming** (out of core, stream.py): the smallest P whose device working set fits the
  budget, in Locality order (A_j pinned while its column streams: SPEC.md:354), with the
  transfer/compute overlap of ``simulate_timeline`` (prefetch depth 1).

``build_schedule`` returns a ``Schedule`` whose fields mirror the reference's Schedule type
(strategy, per-layer estimated times, swap byte counters, resident bytes).
"""

from dataclasses import dataclass, field

import numpy as np

from .errors import BudgetError, ConfigError

# measured rates (B200, fp32) -- see DESIGN.md §4
L2_GATHER_GBS = 16400.0     # random 2.4-KB row gathers, L2 -> SM (profiles/r01_l2_probe.txt)
HBM_GBS = 6550.0            # MEASURED_PEAKS.json copy bandwidth
PCIE_H2D_GBS = 50.0         # pinned H2D, measured 35-55 GB/s (profiles/r01_stream_reddit.jsonl)
CHUNK_LAUNCH_US = 15.0      # launch + tail per chunk pass (small-chunk passes, profiles/r01_tile_ab.txt)
STRATEGIES = ("locality", "dest_order", "stage_based")


def _ld(n, align=4):
    return (n + align - 1) // align * align


def chunk_stats(src, dst, V, P):
    """(max chunk edge count, number of non-empty chunks) of the P x P grid."""
    size = -(-V // P)
    if len(src) == 0:
        return 0, 0
    key = (np.asarray(src, np.int64) // size) * P + np.asarray(dst, np.int64) // size
    cnt = np.bincount(key, minlength=P * P)
    return int(cnt.max()), int((cnt > 0).sum())


def resident_bytes(V, E, dims, model="gcn"):
    """Device bytes of the resident executor (engine.SAGAModel) for an L-layer model: features,
    per-layer aggregate / pre-activation / gradients, the CSC + CSR index (idx + weight + ptr,
    both directions) and the G-GCN [h | P] / [dA | Q] rows."""
    b = V * _ld(dims[0]) * 4
    for f_in, f_out in zip(dims, dims[1:]):
        rows = 3 * _ld(f_in) + 3 * _ld(f_out)          # a, da, tmp / z, dz, h_out
        if model == "ggcn":
            rows += 8 * _ld(f_in)                       # HP, GQ (2x), dQ, dP, dHt, S
        b += V * rows * 4
    b += 2 * (E * 8 + (V + 1) * 8)                      # CSC + CSR: int32 idx, fp32 w, int64 ptr
    return b


def streaming_working_set(V, dims, P, max_chunk_nnz, model="gcn"):
    """Device working set of the out-of-core executors (stream.py) for interval count P: two
    source-row buffers (current + prefetched), two index slots sized for the largest chunk, the
    interval accumulators and the parameters (StreamingGCN / StreamingGGCN.working_set)."""
    nmax = -(-V // P)
    Fmax = max(dims)
    # one index slot (stream._IndexSlot): ptr, idx + weight, the plan's items (at most one per
    # 32 edges or 256 rows, 32 B each) and split records (16 B per 4096 edges)
    nz = max_chunk_nnz
    slot = (nmax + 1) * 8 + nz * 8 + (nz // 32 + nmax // 256 + 2) * 32 + (nz // 4096 + 1) * 16
    wbytes = 2 * sum(a * _ld(b) * 4 for a, b in zip(dims, dims[1:]))
    if model == "ggcn":
        g2 = 2 * _ld(Fmax)
        return 2 * nmax * g2 * 4 + 2 * slot + nmax * (g2 + 5 * _ld(Fmax)) * 4 + \
            Fmax * _ld(Fmax) * 4 + wbytes
    return 2 * nmax * _ld(Fmax) * 4 + 2 * slot + 3 * nmax * _ld(Fmax) * 4 + \
        Fmax * _ld(Fmax) * 4 + wbytes


@dataclass
class LayerPlan:
    width: int
    compute_ms: float
    transfer_ms: float
    makespan_ms: float


@dataclass
class Schedule:
    """SPEC.md:343-348 Schedule: the strategy, the interval count, per-layer estimates
    (simulate_timeline's compute / transfer / makespan) and the swap byte counters."""
    mode: str                 # resident | sharded | streaming
    strategy: str
    P: int
    interval_size: int
    resident_bytes: int
    swap_h2d_bytes: int = 0
    swap_d2h_bytes: int = 0
    layers: list = field(default_factory=list)
    reason: str = ""

    @property
    def makespan_ms(self):
        return sum(L.makespan_ms for L in self.layers)


def pass_compute_ms(V, E, F, P, nonempty_chunks):
    """Fused gather pass: every edge streams one F-wide fp32 row through L2 -> SM, plus one
    launch per chunk and an accumulator read-modify-write per extra source interval."""
    gather = E * F * 4 / (L2_GATHER_GBS * 1e9)
    rmw = (P - 1) * V * _ld(F) * 8 / (HBM_GBS * 1e9)
    return (gather + rmw) * 1e3 + nonempty_chunks * CHUNK_LAUNCH_US * 1e-3


def swap_bytes(V, E, F, P, strategy):
    """H2D / D2H bytes of one streamed layer pass.  Locality: every source
    interval is loaded once per destination column (P^2 chunks of V/P rows), A_j stays resident
    and is written back once; DestOrder: sources loaded once, but A_j is swapped in and out on
    every visit; StageBased: each stage materialises its whole output (edge tensors E x F) and
    reads it back."""
    rows = V * _ld(F) * 4
    index = E * 8 + (V + P) * 8
    if P == 1:
        return rows + index, rows
    if strategy == "locality":
        return P * rows + index, rows
    if strategy == "dest_order":
        return rows + index + P * rows, P * rows
    edge = E * _ld(F) * 4
    return rows + index + edge, rows + edge


def build_schedule(g, dims, *, budget=None, world=1, model="gcn", strategy="locality",
                   candidates=(1, 2, 4, 8, 16, 32, 64, 128, 256, 512)):
    """Choose the interval count and order for ``dims`` = [F, H, ..., C] on graph ``g``
    (anything with V, src, dst).  ``budget`` = device bytes available (None: unbounded);
    ``world`` > 1 shards destination intervals over that many GPUs.  Raises BudgetError when
    no candidate P fits."""
    if strategy not in STRATEGIES:
        raise ConfigError(f"unknown strategy '{strategy}'; valid: {', '.join(STRATEGIES)}")
    V, E = int(g.V), int(len(g.src))
    res = resident_bytes(V, E, dims, model)
    if world > 1:
        P = int(world)
        mx, ne = chunk_stats(g.src, g.dst, V, P)
        layers = [LayerPlan(f, pass_compute_ms(V, E, f, P, ne) / P, 0.0,
                            pass_compute_ms(V, E, f, P, ne) / P) for f in dims[:-1]]
        return Schedule("sharded", "locality", P, -(-V // P), res // P, layers=layers,
                        reason=f"dest-interval sharding over {P} GPUs (P = world)")
    if budget is None or res <= budget:
        best = None
        for P in candidates:
            if P > V:
                break
            _, ne = chunk_stats(g.src, g.dst, V, P)
            t = sum(pass_compute_ms(V, E, f, P, ne) for f in dims[:-1])
            if best is None or t < best[0]:
                best = (t, P, ne)
        _, P, ne = best
        layers = [LayerPlan(f, pass_compute_ms(V, E, f, P, ne), 0.0, pass_compute_ms(V, E, f, P, ne))
                  for f in dims[:-1]]
        return Schedule("resident", strategy, P, -(-V // P), res, layers=layers,
                        reason="the resident set fits: P minimising the modelled pass time")
    for P in candidates:
        if P > V:
            break
        mx, ne = chunk_stats(g.src, g.dst, V, P)
        ws = streaming_working_set(V, dims, P, mx, model)
        if ws > budget:
            continue
        layers, h2d, d2h = [], 0, 0
        for f in dims[:-1]:
            hb, db = swap_bytes(V, E, f, P, strategy)
            h2d, d2h = h2d + hb, d2h + db
            c = pass_compute_ms(V, E, f, P, ne)
            t = (hb + db) / (PCIE_H2D_GBS * 1e9) * 1e3
            # two resources, prefetch depth 1: makespan >= max(compute, transfer)
            layers.append(LayerPlan(f, c, t, max(c, t) + min(c, t) / max(P * P, 1)))
        return Schedule("streaming", strategy, P, -(-V // P), ws, h2d, d2h, layers,
                        reason=f"resident set {res} B exceeds the budget {budget} B: smallest P "
                               f"whose streamed working set ({ws} B) fits")
    raise BudgetError(f"no interval count in {list(candidates)} fits a {budget}-byte device "
                      f"budget (resident set {res} B)")
