// ApplyVertex GEMM in bf16 (SG_GEMM_BF16): tcgen05 kind::f16 with bf16 operands and fp32
// accumulation in TMEM (matmul, tensor.py:306-319; the north star's "bf16 ApplyVertex").
//
// C[M,N] = op(A)[M,K] . op(B)[K,N], A/B bf16 in HBM, C and D = relu(C) written as fp32 or
// bf16 (rounded once from the fp32 accumulator).  Per CTA (128 x BN output tile, K in blocks
// of 64 = one 128-B swizzle row of bf16), warp-specialised:
//   warp 4 (one thread)  TMA producer: cp.async.bulk.tensor loads straight into the UMMA
//                        canonical layouts -- K-contiguous operands as K-major SWIZZLE_128B
//                        ({64 k, rows} boxes), MN-contiguous operands (a^T and dz in
//                        dW = a^T dz, W in z = a W) as MN-major SWIZZLE_128B ({64 mn, 64 k}
//                        boxes, 8 KB apart) -- nothing is transposed or converted anywhere;
//   warp 5 (one thread)  TMEM allocator + UMMA issuer (4 x K=16 per stage), tcgen05.commit
//                        releases the stage to the producer;
//   warps 0-3            epilogue: tcgen05.ld of TMEM lanes 32w..32w+31, fp32 -> C / D with
//                        the strict-mode non-finite vote fused in.
// Split-K (dW, K = |V|) writes fixed-order fp32 partials, reduced deterministically.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>

#include "common.h"
#include "sm100.cuh"

namespace {

constexpr int BM = 128, BK = 64;
constexpr int kTmaWarp = 4, kMmaWarp = 5;
constexpr int kThreads = 192;

template <int BN>
struct BCfg {
  static constexpr int A_TILE = BM * BK * 2;  // 16 KB
  static constexpr int B_TILE = BN * BK * 2;
  static constexpr int STAGE = A_TILE + B_TILE;
  static constexpr int STAGES = (192 * 1024) / STAGE < 8 ? (192 * 1024) / STAGE : 8;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
};

struct BArgs {
  void* C;
  void* D;
  float* partial;
  int32_t* nonfinite;
  int64_t ldc, ldd;
  int64_t M, N;
  int kb_per_split, n_kb;
  int epilogue;
  int c_bf16, d_bf16;
  int vec_c, vec_d;  // 4-element vector stores allowed (ld % 4 == 0, base aligned)
};

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm100::smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(sm100::smem_u32(bar))
      : "memory");
}

// D[tmem] (+)= A[smem] * B[smem], kind::f16 (bf16 in, fp32 accumulate), one thread
__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// kind::f16 instruction descriptor: c_format F32 [4,6), a/b_format BF16 = 1 [7,10)/[10,13),
// a/b major [15]/[16] (1 = MN), N >> 3 [17,23), M >> 4 [24,29)
constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// one operand tile of R rows x 64 k: K-major = one box {64 k, R rows}; MN-major = R/64 boxes
// {64 mn, 64 k} of 8 KB each
template <bool MN, int R>
__device__ __forceinline__ void load_operand(const CUtensorMap* map, uint32_t dst, int64_t mn0, int64_t k0,
                                             uint64_t* bar) {
  if constexpr (!MN) {
    tma_load_2d(dst, map, (int)k0, (int)mn0, bar);
  } else {
#pragma unroll
    for (int j = 0; j < R / 64; ++j) tma_load_2d(dst + j * 8192, map, (int)(mn0 + 64 * j), (int)k0, bar);
  }
}

// UMMA descriptor of k-step kk (16 bf16) of a tile.  K-major SW128: 128-B rows of 64 k,
// 8-row groups 1 KB apart (SBO), a k-step advances 32 B inside the swizzled row.  MN-major
// SW128: 128-B rows of 64 mn per k, 8-k groups 1 KB apart (SBO), 64-mn blocks 8 KB apart
// (LBO), a k-step of 16 rows advances 2 KB.
template <bool MN>
__device__ __forceinline__ uint64_t op_desc(uint32_t base, int kk) {
  if constexpr (!MN) return sm100::smem_desc(base + kk * 32, 16, 1024, sm100::kLayoutSW128);
  return sm100::smem_desc(base + kk * 2048, 8192, 1024, sm100::kLayoutSW128);
}

template <bool A_MN, bool B_MN, int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_bf16_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                     const BArgs p) {
  using C = BCfg<BN>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t raw0 = sm100::smem_u32(smem_raw);
  const uint32_t base = (raw0 + 1023u) & ~1023u;
  unsigned char* base_ptr = smem_raw + (base - raw0);
  uint64_t* full = reinterpret_cast<uint64_t*>(base_ptr + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* done = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int kb0 = blockIdx.z * p.kb_per_split;
  const int nkb = min(p.n_kb, kb0 + p.kb_per_split) - kb0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      sm100::mbar_init(full + s, 1);
      sm100::mbar_init(empty + s, 1);
    }
    sm100::mbar_init(done, 1);
    sm100::fence_mbar_init();
  }
  if (warp == kMmaWarp) sm100::tmem_alloc<C::TMEM_COLS>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == kTmaWarp) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapB)) : "memory");
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        const uint32_t use = i / C::STAGES;
        sm100::mbar_wait(empty + s, (use & 1) ^ 1);
        const uint32_t st = base + s * C::STAGE;
        const int64_t k0 = (int64_t)(kb0 + i) * BK;
        mbar_expect_tx(full + s, C::A_TILE + C::B_TILE);
        load_operand<A_MN, BM>(&mapA, st, m0, k0, full + s);
        load_operand<B_MN, BN>(&mapB, st + C::A_TILE, n0, k0, full + s);
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16(BM, BN, A_MN, B_MN);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        const uint32_t use = i / C::STAGES;
        sm100::mbar_wait(full + s, use & 1);
        sm100::tc_fence_after();
        const uint32_t a_t = base + s * C::STAGE, b_t = a_t + C::A_TILE;
#pragma unroll
        for (int kk = 0; kk < BK / 16; ++kk)
          umma_f16(tmem, op_desc<A_MN>(a_t, kk), op_desc<B_MN>(b_t, kk), idesc, (i > 0 || kk > 0) ? 1u : 0u);
        sm100::umma_commit(empty + s);
      }
      sm100::umma_commit(done);
    }
    __syncwarp();
  } else {
    // ---------------- epilogue: warp w drains TMEM lanes 32w..32w+31 (its rows), all BN columns
    sm100::mbar_wait(done, 0);
    sm100::tc_fence_after();
    const int64_t row = m0 + warp * 32 + lane;
    const bool split = p.partial != nullptr;
    const bool relu = !split && p.epilogue == SG_EPI_RELU_DUAL;
    const bool vec_c = split ? (p.N % 4 == 0) : p.vec_c;
    const bool vec_d = p.vec_d;
    bool bad = false;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
      float v[16];
      sm100::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c0, v);
      if (row < p.M) {
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          const int64_t col = n0 + c0 + j;
          if (col >= p.N) continue;
          const int nvalid = p.N - col < 4 ? (int)(p.N - col) : 4;
          if (split) {
            sm100::store4(p.partial + (int64_t)blockIdx.z * p.M * p.N, false, row * p.N + col, v + j, nvalid, vec_c);
            continue;
          }
          for (int q = 0; q < nvalid; ++q) bad |= !isfinite(v[j + q]);
          if (p.C) sm100::store4(p.C, p.c_bf16, row * p.ldc + col, v + j, nvalid, vec_c);
          if (relu) {
            float r[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) r[q] = sg::relu_np(v[j + q]);
            sm100::store4(p.D, p.d_bf16, row * p.ldd + col, r, nvalid, vec_d);
          }
        }
      }
    }
    if (p.nonfinite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(p.nonfinite, 1);
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) sm100::tmem_dealloc<C::TMEM_COLS>(tmem);
}

__global__ void bf16_splitk_reduce(const float* partial, int splits, int64_t M, int64_t N, void* Cv, int64_t ldc,
                                   int c_bf16, void* Dv, int64_t ldd, int d_bf16, int epilogue, int32_t* flag) {
  const int64_t total = M * N;
  bool bad = false;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += partial[(int64_t)z * total + t];  // fixed order
    const int64_t m = t / N, n = t % N;
    bad |= !isfinite(s);
    if (Cv) {
      if (c_bf16) static_cast<__nv_bfloat16*>(Cv)[m * ldc + n] = __float2bfloat16_rn(s);
      else static_cast<float*>(Cv)[m * ldc + n] = s;
    }
    if (epilogue == SG_EPI_RELU_DUAL) {
      const float r = sg::relu_np(s);
      if (d_bf16) static_cast<__nv_bfloat16*>(Dv)[m * ldd + n] = __float2bfloat16_rn(r);
      else static_cast<float*>(Dv)[m * ldd + n] = r;
    }
  }
  if (flag && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// 2-D bf16 tensor map over a row-major [rows, cols] matrix (leading dimension ld elements),
// box {64 cols, box_rows}, 128-B swizzle
bool make_map(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64u, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <bool A_MN, bool B_MN, int BN>
cudaError_t launch(const CUtensorMap& ma, const CUtensorMap& mb, const BArgs& p, dim3 grid, cudaStream_t st) {
  auto k = gemm_bf16_kernel<A_MN, B_MN, BN>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, BCfg<BN>::SMEM);
    configured = true;
  }
  k<<<grid, kThreads, BCfg<BN>::SMEM, st>>>(ma, mb, p);
  sg::count_launch();
  return cudaGetLastError();
}

template <int BN>
cudaError_t dispatch(bool a_mn, bool b_mn, const CUtensorMap& ma, const CUtensorMap& mb, const BArgs& p,
                     dim3 grid, cudaStream_t st) {
  if (!a_mn && !b_mn) return launch<false, false, BN>(ma, mb, p, grid, st);
  if (!a_mn && b_mn) return launch<false, true, BN>(ma, mb, p, grid, st);
  if (a_mn && !b_mn) return launch<true, false, BN>(ma, mb, p, grid, st);
  return launch<true, true, BN>(ma, mb, p, grid, st);
}

int pick_bn(int64_t N) { return N <= 64 ? 64 : 128; }

}  // namespace

int bf16_splits(int64_t M, int64_t N, int64_t K) {
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + pick_bn(N) - 1) / pick_bn(N));
  const int64_t nkb = (K + BK - 1) / BK;
  if (tiles >= 148 || nkb < 16) return 1;
  int64_t s = std::min<int64_t>((2 * 148 + tiles - 1) / tiles, nkb / 8);
  return (int)std::max<int64_t>(1, std::min<int64_t>(s, 64));
}

int64_t sg_gemm_bf16_workspace_bytes(int64_t M, int64_t N, int64_t K) {
  const int s = bf16_splits(M, N, K);
  return s > 1 ? (int64_t)s * M * N * 4 : 0;
}

int sg_gemm_bf16_run(const sg_gemm_desc* d, cudaStream_t st) {
  const int64_t M = d->M, N = d->N, K = d->K;
  SG_REQUIRE(d->C || d->epilogue == SG_EPI_RELU_DUAL, SG_EINVAL, "bf16 gemm: C may be NULL only with RELU_DUAL");
  const bool c_bf16 = d->c_dtype == SG_BF16, d_bf16 = d->d_dtype == SG_BF16;
  if (K == 0) {
    // C = 0, D = relu(0) = 0
    if (d->C) cudaMemset2DAsync(d->C, d->ldc * (c_bf16 ? 2 : 4), 0, N * (c_bf16 ? 2 : 4), M, st);
    if (d->epilogue == SG_EPI_RELU_DUAL) cudaMemset2DAsync(d->D, d->ldd * (d_bf16 ? 2 : 4), 0, N * (d_bf16 ? 2 : 4), M, st);
    return SG_OK;
  }
  SG_REQUIRE(d->A && d->B, SG_EINVAL, "bf16 gemm: null operand");
  SG_REQUIRE((d->lda % 8) == 0 && (d->ldb % 8) == 0 && ((uintptr_t)d->A % 16) == 0 && ((uintptr_t)d->B % 16) == 0,
             SG_EINVAL, "bf16 gemm: operands need ld %% 8 == 0 and 16-B aligned bases (lda %lld, ldb %lld)",
             (long long)d->lda, (long long)d->ldb);
  SG_REQUIRE(M <= 0x7fffffff && N <= 0x7fffffff && K <= 0x7fffffff, SG_ESHAPE, "bf16 gemm: extent > 2^31");
  const bool a_mn = d->trans_a != 0, b_mn = d->trans_b == 0;
  const int BN = pick_bn(N);
  CUtensorMap ma, mb;
  // A: K-major = stored [M, K] (box 64 k x 128 rows); MN-major = stored [K, M] (box 64 m x 64 k)
  const bool ok_a = a_mn ? make_map(&ma, d->A, K, M, d->lda, 64) : make_map(&ma, d->A, M, K, d->lda, BM);
  const bool ok_b = b_mn ? make_map(&mb, d->B, K, N, d->ldb, 64) : make_map(&mb, d->B, N, K, d->ldb, BN);
  SG_REQUIRE(ok_a && ok_b, SG_ECUDA, "bf16 gemm: tensor map encode failed");
  BArgs p;
  p.C = d->C; p.D = d->D; p.nonfinite = d->nonfinite;
  p.ldc = d->ldc; p.ldd = d->ldd; p.M = M; p.N = N;
  p.epilogue = d->epilogue;
  p.c_bf16 = c_bf16; p.d_bf16 = d_bf16;
  p.n_kb = (int)((K + BK - 1) / BK);
  int splits = bf16_splits(M, N, K);
  p.kb_per_split = (p.n_kb + splits - 1) / splits;
  const int gz = (p.n_kb + p.kb_per_split - 1) / p.kb_per_split;
  p.partial = nullptr;
  if (gz > 1) {
    SG_REQUIRE(d->workspace && d->workspace_bytes >= (int64_t)gz * M * N * 4, SG_EBUDGET,
               "bf16 gemm split-K workspace too small");
    p.partial = (float*)d->workspace;
  }
  // 4-element vector stores need ld % 4 == 0 and 16-B (fp32) / 8-B (bf16) aligned bases
  p.vec_c = d->C && (d->ldc % 4 == 0) && ((uintptr_t)d->C % (c_bf16 ? 8 : 16) == 0);
  p.vec_d = d->D && (d->ldd % 4 == 0) && ((uintptr_t)d->D % (d_bf16 ? 8 : 16) == 0);
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)gz);
  cudaError_t e = BN == 64 ? dispatch<64>(a_mn, b_mn, ma, mb, p, grid, st) : dispatch<128>(a_mn, b_mn, ma, mb, p, grid, st);
  if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "bf16 gemm launch: %s", cudaGetErrorString(e));
  if (gz > 1) {
    const int64_t total = M * N;
    int g = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    bf16_splitk_reduce<<<g, 256, 0, st>>>(p.partial, gz, M, N, d->C, d->ldc, c_bf16, d->D, d->ldd, d_bf16,
                                          d->epilogue, d->nonfinite);
    sg::count_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "bf16 split-k reduce: %s", cudaGetErrorString(e));
  }
  return SG_OK;
}
