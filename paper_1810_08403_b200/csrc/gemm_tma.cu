// ApplyVertex GEMM, TMA-fed variant (the default tensor-core path when the operands are
// 16-B aligned): C[M,N] = op(A) . op(B), fp32 in HBM, 3xTF32 on tcgen05 (matmul,
// tensor.py:306-319).
//
// Per CTA (128 x BN output tile, K in blocks of 32), warp-specialised:
//   warp 8 (one thread)  TMA producer: cp.async.bulk.tensor loads of the RAW fp32 tiles
//                        straight into the UMMA canonical layouts -- K-contiguous operands
//                        as K-major SWIZZLE_128B, MN-contiguous operands (a^T in dW = a^T dz,
//                        W in z = a W) as MN-major SWIZZLE_128B_BASE32B (the only MN-major
//                        tf32 layout), 32 x 32 boxes -- so no operand is transposed anywhere;
//   warps 0-7            converters: hi = rna_tf32(x) in place and lo = rna_tf32(x - hi)
//                        into a lo tile of the same layout (sm100.cuh split3: round-to-nearest
//                        split, 4x tighter than reading the raw container as truncated tf32);
//                        then the epilogue (TMEM -> global);
//   warp 9 (one thread)  TMEM allocator + UMMA issuer: hi*hi + hi*lo + lo*hi per k-step,
//                        tcgen05.commit releases the stage to the producer.
// Stage ring: [raw A | raw B | lo A | lo B]; barriers raw-full (TMA tx bytes), full
// (converters), empty (UMMA commit).  Split-K writes fixed-order partials like gemm_tc.cu.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "common.h"
#include "sm100.cuh"

namespace {

constexpr int BM = 128, BK = 32;
// 8 converter warps instead of 4: the five Reddit-epoch GEMMs 1.31 -> 1.14 ms (the round-to-nearest
// split writes both planes; profiles/r02_gemm_convert_probe.txt)
#ifndef SG_GEMM_CONV_WARPS
#define SG_GEMM_CONV_WARPS 8
#endif
constexpr int kConvWarps = SG_GEMM_CONV_WARPS;   // 4 or 8 converter / epilogue warps
constexpr int kConvThreads = kConvWarps * 32;
constexpr int kTmaWarp = kConvWarps, kMmaWarp = kConvWarps + 1;
constexpr int kThreads = (kConvWarps + 2) * 32;

template <int BN>
struct TCfg {
  static constexpr int A_TILE = BM * BK * 4;
  static constexpr int B_TILE = BN * BK * 4;
  static constexpr int STAGE = 2 * (A_TILE + B_TILE);  // raw + lo planes
  static constexpr int STAGES = (200 * 1024) / STAGE < 6 ? (200 * 1024) / STAGE : 6;
  static constexpr int SMEM = STAGES * STAGE + 1024 + 256;
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
};

struct TmaArgs {
  void* C;  // fp32 or bf16 (c_bf16); may be NULL with RELU_DUAL
  void* D;  // fp32 or bf16 (d_bf16)
  float* partial;
  int64_t ldc, ldd;
  int64_t M, N;
  int kb_per_split, n_kb;
  int epilogue;
  int vec_c, vec_d;
  int c_bf16, d_bf16;
  int32_t* nonfinite;  // strict-mode flag (tensor.py:161-163), checked in the epilogue
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

// one operand tile of R rows x 32 k: K-major = one box {32 k, R rows}; MN-major = R/32
// boxes {32 mn, 32 k} of 4 KB each
template <bool MN, int R>
__device__ __forceinline__ void load_operand(const CUtensorMap* map, uint32_t dst, int64_t mn0,
                                             int64_t k0, uint64_t* bar) {
  if constexpr (!MN) {
    tma_load_2d(dst, map, (int)k0, (int)mn0, bar);
  } else {
#pragma unroll
    for (int j = 0; j < R / 32; ++j) tma_load_2d(dst + j * 4096, map, (int)(mn0 + 32 * j), (int)k0, bar);
  }
}

// the UMMA descriptor of k-step kk (8 tf32 = 32 B of k) of a tile
template <bool MN>
__device__ __forceinline__ uint64_t op_desc(uint32_t base, int kk) {
  if constexpr (!MN) return sm100::smem_desc(base + kk * 32, 16, 1024, sm100::kLayoutSW128);
  // MN-major SW128_BASE32B: 128-B rows of 32 mn per k, 4-row swizzle groups (SBO 512 B),
  // 32-mn blocks 4 KB apart (LBO); a k-step of 8 rows advances 1 KB
  return sm100::smem_desc(base + kk * 1024, 4096, 512, sm100::kLayoutSW128Base32B);
}

template <int BYTES>
__device__ __forceinline__ void convert_plane(uint32_t raw, uint32_t lo, int t) {
  constexpr int N4 = BYTES / 16;
#pragma unroll 4
  for (int i = t; i < N4; i += kConvThreads) {
    float4 x;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(x.x), "=f"(x.y), "=f"(x.z), "=f"(x.w)
                 : "r"(raw + i * 16));
    float4 h, l;
    sm100::split3(x.x, h.x, l.x);
    sm100::split3(x.y, h.y, l.y);
    sm100::split3(x.z, h.z, l.z);
    sm100::split3(x.w, h.w, l.w);
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(raw + i * 16), "f"(h.x), "f"(h.y),
                 "f"(h.z), "f"(h.w)
                 : "memory");
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(lo + i * 16), "f"(l.x), "f"(l.y),
                 "f"(l.z), "f"(l.w)
                 : "memory");
  }
}

template <bool A_MN, bool B_MN, int BN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tma_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                    const TmaArgs p) {
  using C = TCfg<BN>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t raw0 = sm100::smem_u32(smem_raw);
  const uint32_t base = (raw0 + 1023u) & ~1023u;
  unsigned char* base_ptr = smem_raw + (base - raw0);
  uint64_t* rawfull = reinterpret_cast<uint64_t*>(base_ptr + C::STAGES * C::STAGE);
  uint64_t* full = rawfull + C::STAGES;
  uint64_t* empty = full + C::STAGES;
  uint64_t* done = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int kb0 = blockIdx.z * p.kb_per_split;
  const int nkb = min(p.n_kb, kb0 + p.kb_per_split) - kb0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      sm100::mbar_init(rawfull + s, 1);
      sm100::mbar_init(full + s, kConvThreads);
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
        mbar_expect_tx(rawfull + s, C::A_TILE + C::B_TILE);
        load_operand<A_MN, BM>(&mapA, st, m0, k0, rawfull + s);
        load_operand<B_MN, BN>(&mapB, st + C::A_TILE, n0, k0, rawfull + s);
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    if (lane == 0) {
      constexpr uint32_t idesc = sm100::idesc_tf32(BM, BN, A_MN, B_MN);
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        const uint32_t use = i / C::STAGES;
        sm100::mbar_wait(full + s, use & 1);
        sm100::tc_fence_after();
        const uint32_t st = base + s * C::STAGE;
        const uint32_t a_hi = st, b_hi = st + C::A_TILE;
        const uint32_t a_lo = st + C::A_TILE + C::B_TILE, b_lo = a_lo + C::A_TILE;
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          const uint64_t ah = op_desc<A_MN>(a_hi, kk), al = op_desc<A_MN>(a_lo, kk);
          const uint64_t bh = op_desc<B_MN>(b_hi, kk), bl = op_desc<B_MN>(b_lo, kk);
          sm100::umma_tf32(tmem, ah, bh, idesc, (i > 0 || kk > 0) ? 1u : 0u);
          sm100::umma_tf32(tmem, ah, bl, idesc, 1u);
          sm100::umma_tf32(tmem, al, bh, idesc, 1u);
        }
        sm100::umma_commit(empty + s);
      }
      sm100::umma_commit(done);
    }
    __syncwarp();
  } else {
    // ---------------- converters (warps 0-3)
    const int t = threadIdx.x;
    for (int i = 0; i < nkb; ++i) {
      const int s = i % C::STAGES;
      const uint32_t use = i / C::STAGES;
      sm100::mbar_wait(rawfull + s, use & 1);
      const uint32_t st = base + s * C::STAGE;
      convert_plane<C::A_TILE>(st, st + C::A_TILE + C::B_TILE, t);
      convert_plane<C::B_TILE>(st + C::A_TILE, st + 2 * C::A_TILE + C::B_TILE, t);
      sm100::fence_proxy_async_smem();
      sm100::mbar_arrive(full + s);
    }
    // ---------------- epilogue: warp w drains TMEM lanes 32(w%4)..+31 (its rows); with 8 warps
    // warps w and w+4 take the two halves of the BN columns
    sm100::mbar_wait(done, 0);
    sm100::tc_fence_after();
    const int lq = warp & 3;
    const int64_t row = m0 + lq * 32 + lane;
    float* part = p.partial ? p.partial + (int64_t)blockIdx.z * p.M * p.N : nullptr;
    const bool relu = !p.partial && p.epilogue == SG_EPI_RELU_DUAL;
    bool bad = false;
    constexpr int CW = kConvWarps == 8 ? BN / 2 : BN;
    const int cbeg = kConvWarps == 8 ? (warp >> 2) * CW : 0;
#pragma unroll 1
    for (int c0 = cbeg; c0 < cbeg + CW; c0 += 16) {
      float v[16];
      sm100::tmem_ld16(tmem + ((uint32_t)(lq * 32) << 16) + c0, v);
      if (row < p.M) {
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          const int64_t col = n0 + c0 + j;
          if (col >= p.N) continue;
          const int nvalid = p.N - col < 4 ? (int)(p.N - col) : 4;
          if (part) {  // split-K partial: fp32, reduced in a fixed order afterwards
            sm100::store4(part, false, row * p.N + col, v + j, nvalid, p.N % 4 == 0);
            continue;
          }
          for (int q = 0; q < nvalid; ++q) bad |= !isfinite(v[j + q]);
          if (p.C) sm100::store4(p.C, p.c_bf16, row * p.ldc + col, v + j, nvalid, p.vec_c);
          if (relu) {
            float r[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) r[q] = sg::relu_np(v[j + q]);
            sm100::store4(p.D, p.d_bf16, row * p.ldd + col, r, nvalid, p.vec_d);
          }
        }
      }
    }
    if (p.nonfinite && bad) atomicOr(p.nonfinite, 1);
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) sm100::tmem_dealloc<C::TMEM_COLS>(tmem);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    if (e == cudaSuccess && q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    if (getenv("SG_DEBUG")) fprintf(stderr, "sg_gemm_tma: entry point err=%d q=%d\n", (int)e, (int)q);
  }
  return fn;
}

// 2-D fp32 tensor map over a row-major [rows, cols] matrix with leading dimension ld;
// box = {32 (cols), box_rows}; swizzle 128B (K-major tiles) or 128B_ATOM_32B (MN-major).
bool make_map(CUtensorMap* map, const float* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
              bool mn_major) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {32u, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE,
                  mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <bool A_MN, bool B_MN, int BN>
cudaError_t launch_tma(const CUtensorMap& ma, const CUtensorMap& mb, const TmaArgs& p, dim3 grid,
                       cudaStream_t st) {
  auto k = gemm_tma_kernel<A_MN, B_MN, BN>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, TCfg<BN>::SMEM);
    configured = true;
  }
  k<<<grid, kThreads, TCfg<BN>::SMEM, st>>>(ma, mb, p);
  sg::count_launch();
  return cudaGetLastError();
}

template <int BN>
cudaError_t dispatch_tma(bool a_mn, bool b_mn, const CUtensorMap& ma, const CUtensorMap& mb,
                         const TmaArgs& p, dim3 grid, cudaStream_t st) {
  if (!a_mn && !b_mn) return launch_tma<false, false, BN>(ma, mb, p, grid, st);
  if (!a_mn && b_mn) return launch_tma<false, true, BN>(ma, mb, p, grid, st);
  if (a_mn && !b_mn) return launch_tma<true, false, BN>(ma, mb, p, grid, st);
  return launch_tma<true, true, BN>(ma, mb, p, grid, st);
}

bool tma_disabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SG_GEMM_TMA");
    v = (e && e[0] == '0') ? 1 : 0;
  }
  return v == 1;
}

}  // namespace

// Returns 1 if the TMA path launched (C/D written or partials + reduce pending in *partial
// handled by the caller), 0 if the operands do not meet TMA constraints (caller falls back).
int sg_gemm_tma_try(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                    const float* B, int64_t ldb, void* C, int64_t ldc, int c_bf16, int epilogue, void* D,
                    int64_t ldd, int d_bf16, int32_t* nonfinite, float* partial, int kb_per_split, int n_kb,
                    int gz, cudaStream_t st, cudaError_t* err) {
  if (tma_disabled()) return 0;
  if ((lda % 4) || (ldb % 4) || ((uintptr_t)A % 16) || ((uintptr_t)B % 16)) return 0;
  if (M > 0x7fffffff || N > 0x7fffffff || K > 0x7fffffff) return 0;
  const bool a_mn = trans_a != 0, b_mn = trans_b == 0;
  const int BN = N <= 64 ? 64 : 128;
  CUtensorMap ma, mb;
  // A: K-major = stored [M, K] (box 32 k x 128 rows); MN-major = stored [K, M] (box 32 m x 32 k)
  const bool ok_a = a_mn ? make_map(&ma, A, K, M, lda, 32, true) : make_map(&ma, A, M, K, lda, BM, false);
  const bool ok_b = b_mn ? make_map(&mb, B, K, N, ldb, 32, true) : make_map(&mb, B, N, K, ldb, BN, false);
  if (getenv("SG_DEBUG")) fprintf(stderr, "sg_gemm_tma: maps a=%d b=%d encode=%p\n", ok_a, ok_b, (void*)encode_fn());
  if (!ok_a || !ok_b) return 0;
  TmaArgs p;
  p.C = C; p.D = D; p.partial = gz > 1 ? partial : nullptr;
  p.ldc = ldc; p.ldd = ldd; p.M = M; p.N = N;
  p.kb_per_split = kb_per_split; p.n_kb = n_kb;
  p.epilogue = epilogue;
  p.nonfinite = nonfinite;
  p.c_bf16 = c_bf16;
  p.d_bf16 = d_bf16;
  p.vec_c = C != nullptr && (ldc % 4 == 0) && ((uintptr_t)C % (c_bf16 ? 8 : 16) == 0);
  p.vec_d = D != nullptr && (ldd % 4 == 0) && ((uintptr_t)D % (d_bf16 ? 8 : 16) == 0);
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)gz);
  *err = BN == 64 ? dispatch_tma<64>(a_mn, b_mn, ma, mb, p, grid, st)
                  : dispatch_tma<128>(a_mn, b_mn, ma, mb, p, grid, st);
  return 1;
}
