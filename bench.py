#!/usr/bin/env python
"""Benchmark: 2-layer GCN training epoch on a synthetic Reddit-shaped graph (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config reddit]

One "step" = one full training epoch (forward both layers, softmax-CE, backward,
SGD) over the whole graph: the SAGA-NN hot path of the north star.  Prints ONE
JSON line (rank 0).  ``value`` is whole-graph edges per second of epoch time
(E / epoch seconds); ``ms_per_step`` is the epoch time.  The roofline object is
for the dominant kernel, the layer-1 fused Scatter-ApplyEdge-Gather pass
(SURVEY.md §8(d)): algorithmic bytes E*(4+4+F*4) + V*(4+F*4) per launch over its
CUDA-event duration, against MEASURED_PEAKS.json's HBM copy bandwidth.

``--impl reference`` times the reference algorithm's CPU implementation (the
numpy oracle port of tensor.py's composition, oracle/) on this host's cores on
a bounded sample of the same workload, and prints the same metric.
"""

import argparse
import json
import os
import subprocess
import sys
import time

# torchrun sets OMP_NUM_THREADS=1 in every rank; the reference arm runs on rank 0 alone with every
# host thread, so undo that before numpy loads OpenBLAS
_argv = " ".join(sys.argv[1:]).replace("=", " ")
if "--impl reference" in _argv and "LOCAL_RANK" in os.environ:
    for _k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
        os.environ[_k] = str(len(os.sched_getaffinity(0)))

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[1]; hidden/classes pinned in SURVEY.md §8(d)
    "reddit": dict(workload="2-layer GCN epoch (fwd+bwd+SGD), synthetic Reddit-shaped graph",
                   model="gcn", graph="rmat", V=232965, E=114615892, F=602, H=128, C=41),
    # BASELINE.json configs[0] / configs[2]
    "pubmed": dict(workload="2-layer GCN epoch, synthetic Pubmed-shaped graph", model="gcn",
                   graph="uniform", V=19717, E=88648, F=500, H=16, C=3),
    "blogcatalog10": dict(workload="2-layer G-GCN epoch, BlogCatalog-shaped graph x10 edges",
                          model="ggcn", graph="uniform", V=10312, E=6680000, F=128, H=128, C=39),
    # BASELINE.json configs[3]: the multi-GPU power-law graph (runs on 1 GPU too)
    "powerlaw_gcn": dict(workload="2-layer GCN epoch, synthetic power-law graph 4M V / 1B E",
                         model="gcn", graph="rmat", V=4000000, E=1000000000, F=128, H=128, C=16),
    "powerlaw_ggcn": dict(workload="2-layer G-GCN epoch, synthetic power-law graph 4M V / 1B E",
                          model="ggcn", graph="rmat", V=4000000, E=1000000000, F=128, H=128, C=16),
}
# bounded CPU samples: ~3-6 s per oracle epoch on one host core (propagation is
# single-threaded numpy), so --impl reference with the default K/W ends in ~1-2 minutes
CPU_SAMPLE_EDGES = {"reddit": 150_000, "pubmed": 88_648, "blogcatalog10": 50_000,
                    "powerlaw_gcn": 300_000, "powerlaw_ggcn": 60_000}
METRIC = "GCN epoch throughput (whole-graph edges per second of 2-layer fwd+bwd epoch)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="reddit")
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--cpu-sample-edges", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--split-edges", type=int, default=4096)
    ap.add_argument("--no-reorder", action="store_true",
                    help="skip the secondary reorder_linear_gather measurement")
    ap.add_argument("--engine", choices=["auto", "dist"], default="auto",
                    help="dist: run the sharded multi-GPU engine (NCCL) even at N=1")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("hbm_gbs", 6650.0), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def gcn_pass_bytes(V, E, F, s=4):
    """GCN fused pass moves E*(4 + 4 + F*s) + V*(4 + F*s) bytes."""
    return E * (4 + 4 + F * s) + V * (4 + F * s)


# ---------------------------------------------------------------- CPU reference arm
def cpu_sample(cfg, n_edges, use_native_inputs):
    """Bounded sample: the first n_edges edges of the same R-MAT/uniform stream over all V
    vertices, full F/H/C widths; per-epoch cost scales with edges."""
    from oracle import graph as og
    from oracle import rng

    V = cfg["V"]
    gen = rng.rmat_edges if cfg["graph"] == "rmat" else rng.uniform_edges
    s, d = gen(V, n_edges, seed=0)
    if use_native_inputs:
        import paper_1810_08403_b200 as sg

        X = sg.synthetic_features(V, cfg["F"], seed=1)
    else:
        X = rng.features(V, cfg["F"], seed=1)
    part = og.partition_2d(s, d, V, V)
    dims = [cfg["F"], cfg["H"], cfg["C"]]
    if cfg["model"] == "gcn":
        Ws = rng.glorot(list(zip(dims, dims[1:])), seed=2)
        w = og.gcn_edge_weights(s, d, V, np.float32)
        args = (part, X, Ws, rng.labels(V, cfg["C"]), w)
    else:
        shapes = []
        for a, b in zip(dims, dims[1:]):
            shapes += [(a, a), (a, a), (a, b)]
        Ls = rng.glorot(shapes, seed=2)
        args = (part, X, [tuple(Ls[3 * k: 3 * k + 3]) for k in range(2)], rng.labels(V, cfg["C"]))
    return args


def cpu_epoch(cfg, args):
    from oracle import saga

    t0 = time.perf_counter()
    if cfg["model"] == "gcn":
        saga.gcn_epoch(*args)
    else:
        saga.ggcn_epoch(*args)
    return time.perf_counter() - t0


def cpu_threads():
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS"):
        if os.environ.get(k):
            return int(os.environ[k])
    return os.cpu_count() or 1


def run_reference(a, cfg):
    rank, _, world = dist_env()
    if rank != 0:
        return  # under torchrun only rank 0 runs and prints
    n = a.cpu_sample_edges or CPU_SAMPLE_EDGES[a.config]
    args = cpu_sample(cfg, n, use_native_inputs=False)
    for _ in range(a.warmup):
        cpu_epoch(cfg, args)
    times = [cpu_epoch(cfg, args) for _ in range(a.steps)]
    t = float(np.mean(times))
    v = n / t
    cores = cpu_threads()
    sample = (f"first {n} edges of the {cfg['graph']} edge stream over all {cfg['V']} vertices "
              f"(F={cfg['F']}, H={cfg['H']}, C={cfg['C']}); numpy oracle port of tensor.py "
              f"(propagation single-threaded numpy, matmul on {cores} OpenBLAS threads)")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "edges/s", "n_gpus": world,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": cfg["E"] / v * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": config_of(cfg, a, world),
        "cpu_baseline": {"value": v, "unit": "edges/s", "cores": cores, "kind": "port",
                         "sample": sample, "sample_epoch_s": t},
        "e2e": {"value": v, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_of(cfg, a, world):
    return {"workload": cfg["workload"], "graph": cfg["graph"] + (" (0.57,0.19,0.19,0.05)" if cfg["graph"] == "rmat" else ""),
            "V": cfg["V"], "E": cfg["E"], "F": cfg["F"], "H": cfg["H"], "C": cfg["C"],
            "layers": 2, "split_edges": a.split_edges,
            "interval_size": cfg["V"] if (world == 1 and a.engine != "dist") else -(-cfg["V"] // world),
            "parallelism": ("single GPU" if world == 1 and a.engine != "dist" else
                            f"dest-interval sharding x{world} (reencode_balance, "
                            f"{os.environ.get('SG_DIST_BACKEND', 'nccl').upper()} block broadcasts)"),
            "l2": "256 MiB L2 flush between timed steps; inputs (X, edge index) > L2"}


# ---------------------------------------------------------------- clocks
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.p, self.path = index, None, None

    def start(self):
        try:
            import tempfile

            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        rows = []
        for ln in open(self.path).read().strip().splitlines():
            f = [x.strip() for x in ln.split(",")]
            if len(f) >= 9:
                rows.append(f)
        os.unlink(self.path)
        if not rows:
            return None
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------- GPU arm
def run_ours(a, cfg):
    import torch

    import paper_1810_08403_b200 as sg
    from paper_1810_08403_b200 import _lib

    rank, local, world = dist_env()
    if world > 1 or a.engine == "dist":
        from paper_1810_08403_b200 import dist

        for k, v in (("MASTER_ADDR", "127.0.0.1"), ("MASTER_PORT", "29533"), ("RANK", "0"),
                     ("WORLD_SIZE", "1"), ("LOCAL_RANK", "0")):
            os.environ.setdefault(k, v)
        return dist.bench_main(a, cfg, METRIC, config_of(cfg, a, world),
                               {"Clocks": Clocks, "measured_peaks": measured_peaks})
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    V, E, F, H, C = cfg["V"], cfg["E"], cfg["F"], cfg["H"], cfg["C"]
    t0 = time.perf_counter()
    g = (sg.rmat_graph if cfg["graph"] == "rmat" else sg.uniform_graph)(V, E, seed=0)
    t_gen = time.perf_counter() - t0
    grid = sg.ChunkGrid(g, V, split_edges=a.split_edges, gcn_weights=(cfg["model"] == "gcn"))
    t_grid = time.perf_counter() - t0 - t_gen
    build = sg.gcn_model if cfg["model"] == "gcn" else sg.ggcn_model
    m = build(grid, [F, H, C])
    # host features in the device layout ([V, ld], 16-B padded rows): one contiguous H2D
    X_host = torch.from_numpy(sg.synthetic_features(V, F, seed=1, ld=(F + 3) // 4 * 4)).pin_memory()
    lab_host = torch.from_numpy(np.random.default_rng(3).integers(0, C, V)).pin_memory()
    m.load_features(X_host)
    m.load_labels(lab_host)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(a.warmup):
        m.train_step(a.lr)
    torch.cuda.synchronize()
    m.check_status()

    # ---- timed region: K epochs, device-timed with CUDA events, L2 flushed between steps
    clocks = Clocks(local)
    clocks.start()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps)]
    m.prof = []
    stage_marks = []
    n0 = _lib.lib.sg_launch_count()
    torch.cuda.synchronize()
    for k in range(a.steps):
        flush.zero_()
        m.prof = []
        starts[k].record()
        m.train_step(a.lr)
        ends[k].record()
        stage_marks.append(m.prof)
    torch.cuda.synchronize()
    launches = _lib.lib.sg_launch_count() - n0
    m.check_status()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    stages = {}
    for marks in stage_marks:
        m.prof = marks
        for kname, v in m.stage_times().items():
            stages[kname] = stages.get(kname, 0.0) + v / a.steps
    m.prof = None
    t_step = float(np.mean(step_ms)) / 1e3
    value = E / t_step
    # the same K epochs back to back (no flush between them): the previous epoch's dirty L2
    # lines are then written back inside the timed region (reported beside the flushed number)
    bb0, bb1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    bb0.record()
    for _ in range(a.steps):
        m.train_step(a.lr)
    bb1.record()
    torch.cuda.synchronize()
    back_to_back_ms = bb0.elapsed_time(bb1) / a.steps

    # ---- roofline of the dominant kernel: layer-1 fused gather (stage L0.fwd.propagate)
    peak, peak_src = measured_peaks()
    k_ms = stages.get("L0.fwd.propagate")
    # G-GCN forward (GGCN_FWD_S): per edge index + [h | P] row; per destination the pointer,
    # Q read, aggregate and S written
    algo = gcn_pass_bytes(V, E, F) if cfg["model"] == "gcn" else \
        E * (4 + 2 * F * 4) + V * (4 + 3 * F * 4)
    achieved = algo / (k_ms / 1e3) / 1e9 if k_ms else None
    l2_ceiling = None  # measured L2->SM gather ceiling for 2.4-KB rows (tools/l2bw.cu)
    probe = os.path.join(ROOT, "profiles", "r01_l2_probe.txt")
    if os.path.exists(probe):
        vals = [json.loads(x)["GBps"] for x in open(probe) if x.startswith("{") and
                '"buffer_MB": 48,' in x and '"row_bytes": 2432' in x]
        l2_ceiling = max(vals) if vals else None
    traffic = None
    prof_json = os.path.join(ROOT, "profiles", "ncu_dram_bytes.json")
    if os.path.exists(prof_json):
        try:
            traffic = json.load(open(prof_json)).get(a.config, {}).get("L0.fwd.propagate")
        except Exception:
            traffic = None

    # ---- e2e through the public API with host buffers (H2D features+labels, D2H loss)
    e2e = None
    if not a.no_e2e:
        # every step: H2D of that step's features + labels from pinned host memory (staged
        # on a copy stream while the previous step computes) and D2H of its loss
        n_e2e = max(20, a.steps)  # the first step's copy has nothing to overlap: amortised over n
        m.capture(a.lr)  # one CUDA-graph launch per epoch (forward, backward, SGD)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        m.prefetch_inputs(X_host, lab_host)
        for k in range(n_e2e):
            m.replay()
            if k + 1 < n_e2e:
                m.prefetch_inputs(X_host, lab_host)
            float(m.loss.item())
        t_e2e = (time.perf_counter() - t1) / n_e2e
        e2e = {"value": E / t_e2e, "unit": "edges/s",
               "h2d_bytes_per_step": int(X_host.numel() * 4 + lab_host.numel() * 8),
               "d2h_bytes_per_step": 4, "ms_per_step": t_e2e * 1e3,
               "steps": n_e2e,
               "note": "wall clock over n_e2e steps: per step, H2D of that step's features + labels "
                       "from pinned host memory (copy stream, straight into the feature buffer the "
                       "other of two captured epoch graphs reads), one CUDA-graph epoch, loss D2H; "
                       "the first step's copy is not overlapped"}

    # clocks sampled across the timed loops above (device-timed, back-to-back and e2e epochs)
    clk = clocks.stop()

    # ---- secondary: the same epoch with reorder_linear_gather (Y = h W, then propagate Y):
    # the same function re-associated (fp32-rounding-equal, not bitwise), gathers at the
    # narrower output widths.  Reported beside the headline, which keeps the reference's
    # stage order (the F-wide fused gather the roofline is judged on).
    reordered = None
    if cfg["model"] == "gcn" and not a.no_reorder:
        m2 = build(grid, [F, H, C], reorder=True)
        m2.load_features(X_host)
        m2.load_labels(lab_host)
        for _ in range(a.warmup):
            m2.train_step(a.lr)
        torch.cuda.synchronize()
        m2.check_status()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(a.steps)]
        marks2 = []
        for k in range(a.steps):
            flush.zero_()
            m2.prof = []
            ev[k][0].record()
            m2.train_step(a.lr)
            ev[k][1].record()
            marks2.append(m2.prof)
        torch.cuda.synchronize()
        ms2 = float(np.mean([s_.elapsed_time(e_) for s_, e_ in ev]))
        st2 = {}
        for mk in marks2:
            m2.prof = mk
            for kname, v in m2.stage_times().items():
                st2[kname] = st2.get(kname, 0.0) + v / a.steps
        reordered = {"ms_per_step": ms2, "value": E / (ms2 / 1e3), "unit": "edges/s",
                     "layers_reordered": [bool(L.reorder) for L in m2.layers],
                     "stages_ms": {k: round(v, 4) for k, v in st2.items()},
                     "note": "optimizer pass reorder_linear_gather: ReLU((A h) W) computed as "
                             "ReLU(A (h W)); loss/gradients within fp32 tolerance of the reference "
                             "order (tests/test_gpu_kernels.py::test_reordered_gcn_epoch_vs_oracle)"}
        del m2

    # ---- CPU baseline (oracle port) on a bounded sample, rank 0 only
    cpu = None
    if not a.no_cpu_baseline and rank == 0:
        n = a.cpu_sample_edges or CPU_SAMPLE_EDGES[a.config]
        args = cpu_sample(cfg, n, use_native_inputs=True)
        t = cpu_epoch(cfg, args)
        cpu = {"value": n / t, "unit": "edges/s", "cores": cpu_threads(), "kind": "port",
               "sample": f"one epoch on the first {n} edges of the same edge stream over all "
                         f"{V} vertices (numpy oracle port of tensor.py); {t:.1f} s",
               "extrapolated_epoch_ms": E / (n / t) * 1e3}

    line = {
        "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_of(cfg, a, world),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                     "kernel": "L0.fwd.propagate (sg_propagate %s, F=%d)" % (
                         "GCN" if cfg["model"] == "gcn" else "GGCN_FWD_S", F),
                     "algorithmic_bytes_per_launch": algo, "launch_ms": k_ms, "peak_source": peak_src,
                     "note": "frac > 1: the algorithmic bytes count one source row per edge, but "
                             "R-MAT's hot rows are re-served from L1/L2 (canonical CSC: sources "
                             "ascending within a destination); DRAM bytes per launch are in "
                             "'traffic' (ncu); l2_ceiling_gbs = measured L2->SM ceiling for random "
                             "2.4-KB row gathers (tools/l2bw.cu)",
                     "share_of_step": (k_ms / (t_step * 1e3)) if k_ms else None,
                     "launch_list": "profiles/r01_launches_bench_steps.txt (ncu share of the same "
                                    "kernel over 5 epochs of this workload)",
                     "l2_ceiling_gbs": l2_ceiling,
                     "frac_of_l2_ceiling": (achieved / l2_ceiling) if (achieved and l2_ceiling) else None},
        "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": int(launches),
        "ms_per_step_back_to_back": back_to_back_ms,
        "reordered_apply_vertex": reordered,
        "clocks": clk,
        "stages_ms": {k: round(v, 4) for k, v in stages.items()},
        "scatter_gather_edges_per_s": (E / (k_ms / 1e3)) if k_ms else None,
        "setup_s": {"graph_gen": round(t_gen, 2), "partition_upload": round(t_grid, 2)},
        "step_ms_all": [round(x, 3) for x in step_ms],
    }
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    cfg = CONFIGS[a.config]
    if a.gpus != dist_env()[2]:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={dist_env()[2]}: launch N > 1 ranks with "
                         f"python -m torch.distributed.run --nproc-per-node {a.gpus} bench.py --gpus {a.gpus}")
    if a.impl == "reference":
        return run_reference(a, cfg)
    return run_ours(a, cfg)


if __name__ == "__main__":
    main()
