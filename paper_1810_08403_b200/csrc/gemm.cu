// ApplyVertex dense GEMM (K8), matmul of tensor.py:306-319, row-major:
//   C[M,N] = op(A)[M,K] . op(B)[K,N]  (+ optional D = relu(C), tensor.py:207)
//
// SG_GEMM_F32 is a SIMT fp32 kernel (128x128x16 CTA tile, 8x8 per thread,
// register-staged double buffering); it is the exact-fp32 reference path.  The
// tensor-core paths (tcgen05 / TMEM) live in gemm_tc.cu.  K-splitting writes
// fp32 partials to the caller's workspace and reduces them in a fixed order,
// so every GEMM is deterministic.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.h"

namespace {

constexpr int BM = 128, BN = 128, BK = 16, TM = 8, TN = 8, NTHR = 256;

struct GemmArgs {
  const float* A;
  const float* B;
  float* C;
  float* D;
  int64_t lda, ldb, ldc, ldd;
  int64_t M, N, K;
  int64_t k_chunk;
  int trans_a, trans_b, epilogue;
  float* partial;  // [splits][M][N] when split-K
  int32_t* nonfinite;
};

__device__ __forceinline__ float ldA(const GemmArgs& p, int64_t m, int64_t k) {
  if (m >= p.M || k >= p.K) return 0.f;
  return p.trans_a ? __ldg(p.A + k * p.lda + m) : __ldg(p.A + m * p.lda + k);
}
__device__ __forceinline__ float ldB(const GemmArgs& p, int64_t k, int64_t n) {
  if (n >= p.N || k >= p.K) return 0.f;
  return p.trans_b ? __ldg(p.B + n * p.ldb + k) : __ldg(p.B + k * p.ldb + n);
}

__global__ void __launch_bounds__(NTHR) sgemm_kernel(const GemmArgs p) {
  __shared__ float As[2][BK][BM + 4];
  __shared__ float Bs[2][BK][BN + 4];
  const int tid = threadIdx.x;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int64_t kb = (int64_t)blockIdx.z * p.k_chunk;
  const int64_t ke = std::min(p.K, kb + p.k_chunk);
  const int tx = tid % 16, ty = tid / 16;

  // per-thread load coordinates (8 elements each of A and B per K tile)
  float ra[8], rb[8];
  auto load_tile = [&](int64_t k0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int mm, kk;
      if (p.trans_a) { mm = tid % 128; kk = tid / 128 + 2 * i; }
      else { kk = tid % 16; mm = tid / 16 + 16 * i; }
      ra[i] = (k0 + kk < ke) ? ldA(p, m0 + mm, k0 + kk) : 0.f;
      int nn, kk2;
      if (p.trans_b) { kk2 = tid % 16; nn = tid / 16 + 16 * i; }
      else { nn = tid % 128; kk2 = tid / 128 + 2 * i; }
      rb[i] = (k0 + kk2 < ke) ? ldB(p, k0 + kk2, n0 + nn) : 0.f;
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int mm, kk;
      if (p.trans_a) { mm = tid % 128; kk = tid / 128 + 2 * i; }
      else { kk = tid % 16; mm = tid / 16 + 16 * i; }
      As[buf][kk][mm] = ra[i];
      int nn, kk2;
      if (p.trans_b) { kk2 = tid % 16; nn = tid / 16 + 16 * i; }
      else { nn = tid % 128; kk2 = tid / 128 + 2 * i; }
      Bs[buf][kk2][nn] = rb[i];
    }
  };

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.f;

  int buf = 0;
  load_tile(kb);
  store_tile(0);
  __syncthreads();
  for (int64_t k0 = kb; k0 < ke; k0 += BK) {
    const bool more = k0 + BK < ke;
    if (more) load_tile(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM / 4; ++i) {
        float4 v = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4 + i * 64]);
        a[i * 4 + 0] = v.x; a[i * 4 + 1] = v.y; a[i * 4 + 2] = v.z; a[i * 4 + 3] = v.w;
      }
#pragma unroll
      for (int j = 0; j < TN / 4; ++j) {
        float4 v = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4 + j * 64]);
        b[j * 4 + 0] = v.x; b[j * 4 + 1] = v.y; b[j * 4 + 2] = v.z; b[j * 4 + 3] = v.w;
      }
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    if (more) {
      store_tile(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }

  // epilogue: rows ty*4 + {0..3} + {0, 64}, cols tx*4 + {0..3} + {0, 64}
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int64_t m = m0 + ty * 4 + (i % 4) + (i / 4) * 64;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int64_t n = n0 + tx * 4 + (j % 4) + (j / 4) * 64;
      if (n >= p.N) continue;
      const float v = acc[i][j];
      if (p.partial) {
        p.partial[((int64_t)blockIdx.z * p.M + m) * p.N + n] = v;
      } else {
        p.C[m * p.ldc + n] = v;
        if (p.epilogue == SG_EPI_RELU_DUAL) p.D[m * p.ldd + n] = sg::relu_np(v);
        if (p.nonfinite && !isfinite(v)) atomicOr(p.nonfinite, 1);
      }
    }
  }
}

__global__ void splitk_reduce_kernel(const float* partial, int splits, int64_t M, int64_t N,
                                     float* C, int64_t ldc, float* D, int64_t ldd, int epilogue,
                                     int32_t* nonfinite) {
  const int64_t total = M * N;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += partial[(int64_t)z * total + t];  // fixed order
    const int64_t m = t / N, n = t % N;
    C[m * ldc + n] = s;
    if (epilogue == SG_EPI_RELU_DUAL) D[m * ldd + n] = sg::relu_np(s);
    if (nonfinite && !isfinite(s)) atomicOr(nonfinite, 1);
  }
}

int choose_splits(int64_t M, int64_t N, int64_t K) {
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int64_t target = 2 * 148;
  if (tiles >= target || K < 4 * 256) return 1;
  int64_t s = (target + tiles - 1) / tiles;
  s = std::min<int64_t>(s, K / 256);
  return (int)std::max<int64_t>(1, std::min<int64_t>(s, 64));
}

}  // namespace

int sg_gemm_tc(int prec, int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const float* A,
               int64_t lda, const float* B, int64_t ldb, void* C, int64_t ldc, int c_bf16, int epilogue,
               void* D, int64_t ldd, int d_bf16, int32_t* nonfinite, void* workspace,
               int64_t workspace_bytes, cudaStream_t st);
int64_t sg_gemm_tc_workspace_bytes(int64_t M, int64_t N, int64_t K, int prec);
int64_t sg_gemm_bf16_workspace_bytes(int64_t M, int64_t N, int64_t K);
int sg_gemm_bf16_run(const sg_gemm_desc* d, cudaStream_t st);

namespace {

// the fp32 paths (SIMT / 3xTF32) behind sg_gemm and sg_gemm_ex
int gemm_f32(int prec, int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const float* A,
             int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int epilogue, float* D,
             int64_t ldd, int32_t* nonfinite, void* workspace, int64_t workspace_bytes, cudaStream_t st);

}  // namespace

extern "C" {

int64_t sg_gemm_workspace_bytes(int64_t M, int64_t N, int64_t K, int prec) {
  if (prec == SG_GEMM_BF16) return sg_gemm_bf16_workspace_bytes(M, N, K);
  if (prec != SG_GEMM_F32) return sg_gemm_tc_workspace_bytes(M, N, K, prec);
  const int s = choose_splits(M, N, K);
  return s > 1 ? (int64_t)s * M * N * 4 : 0;
}

int sg_gemm(int prec, int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const float* A,
            int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int epilogue, float* D,
            int64_t ldd, void* workspace, int64_t workspace_bytes, void* stream) {
  sg_gemm_desc d;
  d.prec = prec; d.trans_a = trans_a; d.trans_b = trans_b; d.epilogue = epilogue;
  d.M = M; d.N = N; d.K = K;
  d.A = A; d.lda = lda; d.B = B; d.ldb = ldb;
  d.C = C; d.ldc = ldc; d.c_dtype = SG_F32;
  d.D = D; d.ldd = ldd; d.d_dtype = SG_F32;
  d.nonfinite = nullptr;
  d.workspace = workspace; d.workspace_bytes = workspace_bytes;
  return sg_gemm_ex(&d, stream);
}

int sg_gemm_ex(const sg_gemm_desc* d, void* stream) {
  SG_REQUIRE(d, SG_EINVAL, "gemm: null descriptor");
  SG_REQUIRE(d->M >= 0 && d->N >= 0 && d->K >= 0, SG_ESHAPE, "gemm: negative extent");
  SG_REQUIRE(d->epilogue != SG_EPI_RELU_DUAL || d->D, SG_EINVAL, "gemm: RELU_DUAL needs D");
  SG_REQUIRE(d->prec == SG_GEMM_F32 || d->prec == SG_GEMM_TF32X3 || d->prec == SG_GEMM_BF16, SG_EINVAL,
             "gemm: unknown precision %d", d->prec);
  if (d->M == 0 || d->N == 0) return SG_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (d->prec == SG_GEMM_BF16) return sg_gemm_bf16_run(d, st);
  if (d->prec == SG_GEMM_TF32X3)  // fp32 operands; C / D may be bf16 (TMA path), C may be NULL
    return sg_gemm_tc(d->prec, d->trans_a, d->trans_b, d->M, d->N, d->K, (const float*)d->A, d->lda,
                      (const float*)d->B, d->ldb, d->C, d->ldc, d->c_dtype == SG_BF16, d->epilogue, d->D,
                      d->ldd, d->d_dtype == SG_BF16, d->nonfinite, d->workspace, d->workspace_bytes, st);
  SG_REQUIRE(d->c_dtype == SG_F32 && d->d_dtype == SG_F32 && d->C, SG_EINVAL,
             "gemm: SG_GEMM_F32 writes fp32 C (and D)");
  return gemm_f32(d->prec, d->trans_a, d->trans_b, d->M, d->N, d->K, (const float*)d->A, d->lda,
                  (const float*)d->B, d->ldb, (float*)d->C, d->ldc, d->epilogue, (float*)d->D, d->ldd,
                  d->nonfinite, d->workspace, d->workspace_bytes, st);
}

}  // extern "C"

namespace {

int gemm_f32(int prec, int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const float* A,
             int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int epilogue, float* D,
             int64_t ldd, int32_t* nonfinite, void* workspace, int64_t workspace_bytes, cudaStream_t st) {
  if (prec != SG_GEMM_F32)
    return sg_gemm_tc(prec, trans_a, trans_b, M, N, K, A, lda, B, ldb, C, ldc, 0, epilogue, D, ldd, 0,
                      nonfinite, workspace, workspace_bytes, st);
  const int splits = choose_splits(M, N, K);
  GemmArgs p;
  p.A = A; p.B = B; p.C = C; p.D = D;
  p.lda = lda; p.ldb = ldb; p.ldc = ldc; p.ldd = ldd;
  p.M = M; p.N = N; p.K = K;
  p.trans_a = trans_a; p.trans_b = trans_b; p.epilogue = epilogue;
  p.partial = nullptr;
  p.nonfinite = nonfinite;
  int64_t kc = (K + splits - 1) / splits;
  kc = (kc + BK - 1) / BK * BK;
  p.k_chunk = std::max<int64_t>(kc, BK);
  const int gz = (int)((K + p.k_chunk - 1) / p.k_chunk);
  if (gz > 1) {
    SG_REQUIRE(workspace && workspace_bytes >= (int64_t)gz * M * N * 4, SG_EBUDGET,
               "gemm split-K workspace too small");
    p.partial = (float*)workspace;
    p.nonfinite = nullptr;  // checked by the reduction
  }
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)std::max(gz, 1));
  if (K == 0) {
    // C = 0
    cudaError_t e = cudaMemset2DAsync(C, ldc * 4, 0, N * 4, M, st);
    if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "gemm memset: %s", cudaGetErrorString(e));
    if (epilogue == SG_EPI_RELU_DUAL) cudaMemset2DAsync(D, ldd * 4, 0, N * 4, M, st);
    return SG_OK;
  }
  sgemm_kernel<<<grid, NTHR, 0, st>>>(p);
  sg::count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "sgemm launch: %s", cudaGetErrorString(e));
  if (gz > 1) {
    const int64_t total = M * N;
    int g = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    splitk_reduce_kernel<<<g, 256, 0, st>>>(p.partial, gz, M, N, C, ldc, D, ldd, epilogue, nonfinite);
    sg::count_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "split-k reduce: %s", cudaGetErrorString(e));
  }
  return SG_OK;
}

}  // namespace

