"""Probe the tcgen05 GEMM operand layouts with one-hot inputs (GPU debugging aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1810_08403_b200 import _lib, kernels as K

def run(M, N, Kd, ta, tb):
    r = np.random.default_rng(0)
    A = r.uniform(-1, 1, (Kd, M) if ta else (M, Kd)).astype(np.float32)
    B = r.uniform(-1, 1, (N, Kd) if tb else (Kd, N)).astype(np.float32)
    C = torch.zeros((M, N), device="cuda")
    K.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), C, trans_a=bool(ta), trans_b=bool(tb), prec=_lib.GEMM_TF32X3)
    torch.cuda.synchronize()
    ref = (A.T if ta else A).astype(np.float64) @ (B.T if tb else B).astype(np.float64)
    got = C.cpu().numpy()
    print(f"M={M} N={N} K={Kd} ta={ta} tb={tb}: max|got|={np.abs(got).max():.3g} max|ref|={np.abs(ref).max():.3g} relerr={np.linalg.norm(got-ref)/np.linalg.norm(ref):.3g}")
    return A, B, got

for args in [(128, 64, 32, 0, 1), (128, 64, 32, 0, 0), (128, 64, 32, 1, 1), (128, 64, 32, 1, 0), (128,128,32,0,1), (128,128,32,0,0)]:
    run(*args)
# one-hot probe for MN-major B: A = e_k selector, C[m, n] = B[m % 32, n]
M, N, Kd = 128, 64, 32
A = np.zeros((M, Kd), np.float32); A[np.arange(M), np.arange(M) % Kd] = 1
B = (np.arange(Kd)[:, None] * 100 + np.arange(N)[None, :]).astype(np.float32)
C = torch.zeros((M, N), device="cuda")
K.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), C, prec=_lib.GEMM_TF32X3)
got = C.cpu().numpy()
print("probe rows 0..5, cols 0..8 (expect k*100+n):")
print(got[:6, :9])
print(got[32:34, :9])
