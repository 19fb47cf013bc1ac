"""Scatter/Gather microbenchmark sweep (BASELINE.json configs[4]).

    python tools/sweep.py [--quick] > profiles/r01_sweep.jsonl

Uniform random graphs with V = 2^22 vertices (V reduced so E = V*deg <= 2^28), average
degree 4..512; feature widths 16..1024; Gather(sum) = sg_propagate(PASS) over the CSC
index, Gather(max) = sg_segment_max (the primitive, int64 argmax) and sg_max_gather (the MP-GCN
fused max gather, int32 argmax positions); fp32 and bf16 rows.  Every point times the
kernel with CUDA events (median of 5 after 2 warm-ups, L2 flushed before each) and
reports algorithmic bytes / time against MEASURED_PEAKS.json's HBM bandwidth.  Points
whose source matrix V*F*s is below 4x the L2 size are flagged `l2_resident`.
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1810_08403_b200 as sg  # noqa: E402
from paper_1810_08403_b200 import _lib  # noqa: E402
from paper_1810_08403_b200 import kernels as K  # noqa: E402


def peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    return json.load(open(p))["hbm_gbs"] if os.path.exists(p) else 6650.0


def timed(fn, flush, reps=5):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        flush.zero_()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    a = ap.parse_args()
    degs = [4, 16, 64, 256] if a.quick else [4, 8, 16, 32, 64, 128, 256, 512]
    widths = [16, 128, 1024] if a.quick else [16, 32, 64, 128, 256, 512, 1024]
    dev = torch.device("cuda")
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    hbm = peak()
    for deg in degs:
        V = min(1 << 22, (1 << 28) // deg)
        E = V * deg
        t0 = time.perf_counter()
        g = sg.uniform_graph(V, E, seed=deg)
        grid = sg.ChunkGrid(g, V, gcn_weights=False, device=dev)
        pi = grid.csc[(0, 0)]
        setup = time.perf_counter() - t0
        for F in widths:
            for dt, s in ((torch.float32, 4), (torch.bfloat16, 2)):
                if V * F * s > 24 << 30:
                    continue
                ld = (F + 7) // 8 * 8
                X = torch.rand((V, ld), device=dev).to(dt)[:, :F]
                out = torch.empty((V, ld), device=dev, dtype=dt)[:, :F]
                ms = timed(lambda: K.propagate(pi, _lib.PROP_PASS, X, out, F), flush)
                byt = E * (4 + F * s) + V * (4 + F * s)
                rec = dict(reduction="sum", dtype=str(dt).split(".")[-1], F=F, avg_degree=deg, V=V,
                           E=E, ms=ms, algo_bytes=byt, gbs=byt / ms / 1e6, hbm_frac=byt / ms / 1e6 / hbm,
                           edges_per_s=E / ms * 1e3, l2_resident=V * F * s < 4 * l2,
                           setup_s=round(setup, 1))
                print(json.dumps(rec), flush=True)
                if dt == torch.float32:
                    arg = torch.empty((V, F), dtype=torch.int64, device=dev)
                    xm = X.contiguous() if X.stride(0) % 4 else X

                    def run_max():
                        _lib.check(_lib.lib.sg_segment_max(
                            K.dtype_code(xm), pi.ptr.data_ptr(), pi.idx.data_ptr(), V, xm.data_ptr(),
                            xm.stride(0), out.data_ptr(), out.stride(0), arg.data_ptr(), F, F, 0.0,
                            _lib.stream_handle()))

                    ms = timed(run_max, flush)
                    byt = E * (4 + F * s) + V * (4 + F * (s + 8))
                    rec.update(reduction="max", ms=ms, algo_bytes=byt, gbs=byt / ms / 1e6,
                               hbm_frac=byt / ms / 1e6 / hbm, edges_per_s=E / ms * 1e3)
                    print(json.dumps(rec), flush=True)
                    # the hot path's fused max gather (K7, MP-GCN): int32 argmax positions
                    arg32 = torch.empty((V, F), dtype=torch.int32, device=dev)
                    ms = timed(lambda: K.max_gather(pi, xm, out, arg32, F), flush)
                    byt = E * (4 + F * s) + V * (4 + F * (s + 4))
                    rec.update(reduction="max_fused", ms=ms, algo_bytes=byt, gbs=byt / ms / 1e6,
                               hbm_frac=byt / ms / 1e6 / hbm, edges_per_s=E / ms * 1e3)
                    print(json.dumps(rec), flush=True)
                    del arg32
                del X, out
        del grid, g, pi
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
