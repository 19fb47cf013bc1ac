// tcgen05 / TMEM tensor-core GEMM paths (SG_GEMM_TF32X3, SG_GEMM_BF16) -- see below.
#include <cuda_runtime.h>

#include "common.h"

int64_t sg_gemm_tc_workspace_bytes(int64_t M, int64_t N, int64_t K, int prec) {
  (void)M; (void)N; (void)K; (void)prec;
  return 0;
}

int sg_gemm_tc(int prec, int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const float* A,
               int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int epilogue,
               float* D, int64_t ldd, void* workspace, int64_t workspace_bytes, cudaStream_t st) {
  SG_FAIL(SG_EINVAL, "tensor-core GEMM precision %d not built yet", prec);
}
