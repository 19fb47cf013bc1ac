"""Time the ApplyVertex GEMM shapes of the Reddit-shaped GCN epoch (CUDA events, L2-cold).

    python tools/gemm_bench.py [--prec tc|f32] [--iters 20] [--only NAME]

Prints one line per shape: ms, effective TFLOP/s (2MNK per pass; 3xTF32 issues 3 tensor
passes), and HBM GB/s of the operand+result bytes.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1810_08403_b200 import _lib  # noqa: E402
from paper_1810_08403_b200 import kernels as K  # noqa: E402

V, F, H, C = 232965, 602, 128, 41
SHAPES = {  # name: (M, N, K, trans_a, trans_b, relu)
    "L0.fwd z=aW": (V, H, F, 0, 0, 1),
    "L0.bwd dW=a^T dz": (F, H, V, 1, 0, 0),
    "L1.fwd z=aW": (V, C, H, 0, 0, 0),
    "L1.bwd dW=a^T dz": (H, C, V, 1, 0, 0),
    "L1.bwd da=dz W^T": (V, H, C, 0, 1, 0),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--prec", default="tc")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--only", default=None)
    a = ap.parse_args()
    prec = _lib.GEMM_TF32X3 if a.prec == "tc" else _lib.GEMM_F32
    dev = torch.device("cuda")
    ws = K.Workspace(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def pad(r, c):
        return (torch.rand((r, (c + 3) // 4 * 4), device=dev) - 0.5)[:, :c]
    for name, (M, N, Kd, ta, tb, relu) in SHAPES.items():
        if a.only and a.only not in name:
            continue
        A = pad(*((Kd, M) if ta else (M, Kd)))  # 16-B aligned rows, as the engine allocates
        B = pad(*((N, Kd) if tb else (Kd, N)))
        Cm = pad(M, N)
        D = pad(M, N) if relu else None
        for _ in range(3):
            K.gemm(A, B, Cm, trans_a=bool(ta), trans_b=bool(tb), relu_out=D, prec=prec, ws=ws)
        ts = []
        for _ in range(a.iters):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            K.gemm(A, B, Cm, trans_a=bool(ta), trans_b=bool(tb), relu_out=D, prec=prec, ws=ws)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ts.sort()
        ms = ts[len(ts) // 2]
        fl = 2.0 * M * N * Kd
        by = 4.0 * (M * Kd + Kd * N + M * N * (2 if relu else 1))
        print(f"{name:20s} M={M:7d} N={N:4d} K={Kd:7d}  {ms:7.3f} ms  {fl / ms / 1e9:7.1f} TFLOP/s "
              f"(x3 passes {3 * fl / ms / 1e9:7.1f})  {by / ms / 1e6:7.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
