// ApplyVertex GEMM on the 5th-generation tensor cores (tcgen05 + TMEM), fp32 in/out.
//
// C[M,N] = op(A)[M,K] . op(B)[K,N] (matmul, tensor.py:306-319), every operand
// fp32 in HBM.  Precision SG_GEMM_TF32X3 ("3xTF32"): each fp32 tile is split on
// the fly into hi = rna_tf32(x) and lo = rna_tf32(x - hi) (sm100.cuh split3), and
// the tensor core accumulates hi*hi + hi*lo + lo*hi in fp32 TMEM -- ~1e-6
// relative error, inside the 1e-4 fp32 parity bar that a single TF32 pass misses
// (SURVEY.md §7 "fp32 parity of the GEMM").
//
// CTA = 128 x BN output tile, K in blocks of 32, STAGES-deep shared-memory ring:
//   warps 0-7  load A/B tiles with coalesced 128-bit LDG, split hi/lo and store them
//              in the UMMA canonical K-major SWIZZLE_128B layout (operands stored
//              MN-contiguous in HBM, e.g. a^T in dW = a^T dz, are transposed 4x4 in
//              registers on the way, never in memory); after the K loop they drain
//              the TMEM accumulator with tcgen05.ld (epilogue).
//   warp 8     allocates TMEM and is the single-thread tcgen05.mma issuer; each
//              stage is released back to the loaders by tcgen05.commit -> mbarrier.
// Long-K products (dW = a^T dz, K = |V|) are split over K; fp32 partials are
// reduced in a fixed order, so results are deterministic.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.h"
#include "sm100.cuh"

namespace {

constexpr int BM = 128, BK = 32;
constexpr int kLoadThreads = 256;                 // 8 loader / epilogue warps
constexpr int kMmaWarp = kLoadThreads / 32;       // warp 8: TMEM allocator + UMMA issuer
constexpr int kThreads = kLoadThreads + 32;

template <int BN>
struct Cfg {
  static constexpr int STAGES = BN >= 128 ? 3 : 4;
  static constexpr int A_TILE = BM * BK * 4;  // bytes, fp32
  static constexpr int B_TILE = BN * BK * 4;
  static constexpr int STAGE = 2 * A_TILE + 2 * B_TILE;  // hi + lo planes
  static constexpr int SMEM = STAGES * STAGE + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int TMEM_COLS = BN < 32 ? 32 : BN;
};

struct TcArgs {
  const float* A;
  const float* B;
  float* C;
  float* D;
  float* partial;
  int64_t lda, ldb, ldc, ldd;
  int64_t M, N, K;
  int kb_per_split, n_kb;
  int epilogue;
  int vec_a, vec_b, vec_c, vec_d;
  int32_t* nonfinite;  // strict-mode flag (tensor.py:161-163), checked in the epilogue
};

__device__ __forceinline__ void split_tf32(float4 x, float4& hi, float4& lo) {
  sm100::split3(x.x, hi.x, lo.x);
  sm100::split3(x.y, hi.y, lo.y);
  sm100::split3(x.z, hi.z, lo.z);
  sm100::split3(x.w, hi.w, lo.w);
}

__device__ __forceinline__ float4 ld4(const float* base, int64_t ld, int64_t r, int64_t c, int64_t R,
                                      int64_t Cn, bool vec) {
  // element (r, c..c+3) of a row-major [R, Cn] matrix, zero outside
  if (r >= R) return make_float4(0.f, 0.f, 0.f, 0.f);
  const float* p = base + r * ld + c;
  if (vec && c + 3 < Cn) return __ldg(reinterpret_cast<const float4*>(p));
  float4 v;
  v.x = c + 0 < Cn ? __ldg(p + 0) : 0.f;
  v.y = c + 1 < Cn ? __ldg(p + 1) : 0.f;
  v.z = c + 2 < Cn ? __ldg(p + 2) : 0.f;
  v.w = c + 3 < Cn ? __ldg(p + 3) : 0.f;
  return v;
}

__device__ __forceinline__ void sts128(uint32_t addr, float4 v) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// Load + split one operand tile (R rows of the operand x 32 k) into hi/lo planes, stored
// in the K-major SWIZZLE_128B canonical layout: atom = 8 rows x 128 B, the 16-B chunk c
// of row r at chunk c ^ (r & 7), row-group stride (SBO) 1024 B.
// byte offset of the 16-B chunk holding (row, k..k+3) in a K-major SWIZZLE_128B tile
__device__ __forceinline__ uint32_t kmajor_off(int row, int kc) {
  return (row >> 3) * 1024 + (row & 7) * 128 + ((kc ^ (row & 7)) << 4);
}

__device__ __forceinline__ void store_split(uint32_t hi_base, uint32_t lo_base, uint32_t off, float4 v) {
  float4 hi, lo;
  split_tf32(v, hi, lo);
  sts128(hi_base + off, hi);
  sts128(lo_base + off, lo);
}

// One operand tile (R rows of the operand x 32 k) held in registers between its global
// load and its split/store, so the next stage's loads are in flight while this stage is
// written to shared memory (register double buffering in the loader loop).
template <bool MN_MAJOR, int R>
struct TileRegs {
  // K-major: one 16-B chunk (row, 4 k) per slot; MN-major: one 4x4 (4 k x 4 rows) block
  static constexpr int PER_K = R * BK / 4 / kLoadThreads;
  static constexpr int BLOCKS = (R / 4) * (BK / 4);
  static constexpr int PER_MN = (BLOCKS + kLoadThreads - 1) / kLoadThreads;
  static constexpr int N4 = MN_MAJOR ? PER_MN * 4 : PER_K;
  float4 v[N4];

  // MN-major block -> (mb, kb).  Thread bits: b0 = mb & 1 (two threads cover a full 32-B
  // sector of a k-row), b1-b2 = kb & 3, rest = mb >> 1 | kb >> 2.  For a fixed q the 32
  // swizzled STS.128 of a warp then hit 8 distinct 16-B bank groups (4 wavefronts, no
  // conflicts): chunk = kb ^ (row & 7) with row & 7 = (mb & 1) * 4 + q.
  __device__ __forceinline__ static void mn_coords(int idx, int& mb, int& kb) {
    const int rest = idx >> 3;
    mb = (rest % (R / 8)) * 2 + (idx & 1);
    kb = ((idx >> 1) & 3) + 4 * (rest / (R / 8));
  }

  __device__ __forceinline__ void load(const float* X, int64_t ld, int64_t mn0, int64_t k0,
                                       int64_t MNmax, int64_t Kmax, bool vec, int t) {
    if constexpr (!MN_MAJOR) {
#pragma unroll
      for (int i = 0; i < PER_K; ++i) {
        const int idx = t + kLoadThreads * i;
        v[i] = ld4(X, ld, mn0 + idx / 8, k0 + (idx % 8) * 4, MNmax, Kmax, vec);
      }
    } else {
#pragma unroll
      for (int i = 0; i < PER_MN; ++i) {
        const int idx = t + kLoadThreads * i;
        if (BLOCKS % kLoadThreads != 0 && idx >= BLOCKS) continue;
        int mb, kb;
        mn_coords(idx, mb, kb);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t k = k0 + kb * 4 + q;
          v[i * 4 + q] = k < Kmax ? ld4(X, ld, k, mn0 + mb * 4, Kmax, MNmax, vec)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    }
  }

  // split hi/lo and store in the K-major SWIZZLE_128B canonical layout (operands stored
  // MN-contiguous in HBM are transposed 4x4 in registers: the shared-memory operand is
  // always K-major, no operand is ever transposed in HBM)
  __device__ __forceinline__ void store(uint32_t hi_base, uint32_t lo_base, int t) const {
    if constexpr (!MN_MAJOR) {
#pragma unroll
      for (int i = 0; i < PER_K; ++i) {
        const int idx = t + kLoadThreads * i;
        store_split(hi_base, lo_base, kmajor_off(idx / 8, idx % 8), v[i]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < PER_MN; ++i) {
        const int idx = t + kLoadThreads * i;
        if (BLOCKS % kLoadThreads != 0 && idx >= BLOCKS) continue;
        int mb, kb;
        mn_coords(idx, mb, kb);
        const float4* b = v + i * 4;
        store_split(hi_base, lo_base, kmajor_off(mb * 4 + 0, kb), make_float4(b[0].x, b[1].x, b[2].x, b[3].x));
        store_split(hi_base, lo_base, kmajor_off(mb * 4 + 1, kb), make_float4(b[0].y, b[1].y, b[2].y, b[3].y));
        store_split(hi_base, lo_base, kmajor_off(mb * 4 + 2, kb), make_float4(b[0].z, b[1].z, b[2].z, b[3].z));
        store_split(hi_base, lo_base, kmajor_off(mb * 4 + 3, kb), make_float4(b[0].w, b[1].w, b[2].w, b[3].w));
      }
    }
  }
};

// one tf32 UMMA consumes K = 8 = 32 B of each K-major row: advance the start address
__device__ __forceinline__ uint64_t tile_desc(uint32_t base, int kk) {
  return sm100::smem_desc(base + kk * 32, 16, 1024, sm100::kLayoutSW128);
}

template <bool A_MN, bool B_MN, int BN>
__global__ void __launch_bounds__(kThreads, 1) gemm_tf32x3_kernel(const TcArgs p) {
  using C = Cfg<BN>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte alignment for the SWIZZLE_128B atoms
  const uint32_t raw = sm100::smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char* base_ptr = smem_raw + (base - raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(base_ptr + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* done = empty + C::STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int kb0 = blockIdx.z * p.kb_per_split;
  const int kb1 = min(p.n_kb, kb0 + p.kb_per_split);
  const int nkb = kb1 - kb0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      sm100::mbar_init(full + s, kLoadThreads);
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

  if (warp < kMmaWarp) {
    // ---------------- loaders: LDG -> split hi/lo -> swizzled STS, one stage ahead
    const int t = threadIdx.x;
    TileRegs<A_MN, BM> ra[2];
    TileRegs<B_MN, BN> rb[2];
    if (nkb > 0) {
      ra[0].load(p.A, p.lda, m0, (int64_t)kb0 * BK, p.M, p.K, p.vec_a, t);
      rb[0].load(p.B, p.ldb, n0, (int64_t)kb0 * BK, p.N, p.K, p.vec_b, t);
    }
#pragma unroll 1
    for (int i = 0; i < nkb; i += 2) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {  // static register-set index (no dynamic indexing)
        const int ii = i + h;
        if (ii >= nkb) break;
        if (ii + 1 < nkb) {
          const int64_t kn = (int64_t)(kb0 + ii + 1) * BK;
          ra[h ^ 1].load(p.A, p.lda, m0, kn, p.M, p.K, p.vec_a, t);
          rb[h ^ 1].load(p.B, p.ldb, n0, kn, p.N, p.K, p.vec_b, t);
        }
        const int s = ii % C::STAGES;
        const uint32_t use = ii / C::STAGES;
        sm100::mbar_wait(empty + s, (use & 1) ^ 1);
        const uint32_t st = base + s * C::STAGE;
        ra[h].store(st, st + C::A_TILE, t);
        rb[h].store(st + 2 * C::A_TILE, st + 2 * C::A_TILE + C::B_TILE, t);
        sm100::fence_proxy_async_smem();
        sm100::mbar_arrive(full + s);
      }
    }
    // ---------------- epilogue: TMEM -> registers -> global
    sm100::mbar_wait(done, 0);
    sm100::tc_fence_after();
    // warp w reads TMEM lane quarter w % 4 (its rows) and column half w / 4
    const int quarter = warp & 3, half = warp >> 2;
    const int64_t row = m0 + quarter * 32 + lane;
    // each thread owns 16 consecutive columns of one row: 4 x 16-B stores (full sectors)
    float* dst = p.partial ? p.partial + (int64_t)blockIdx.z * p.M * p.N : p.C;
    const int64_t ldo = p.partial ? p.N : p.ldc;
    const bool relu = !p.partial && p.epilogue == SG_EPI_RELU_DUAL;
    const bool vec_o = p.partial ? (p.N % 4 == 0) : p.vec_c;
#pragma unroll 1
    for (int c0 = half * (BN / 2); c0 < (half + 1) * (BN / 2); c0 += 16) {
      float v[16];
      sm100::tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + c0, v);
      if (row < p.M) {
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          const int64_t col = n0 + c0 + j;
          if (vec_o && col + 3 < p.N) {
            *reinterpret_cast<float4*>(dst + row * ldo + col) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (col + q < p.N) dst[row * ldo + col + q] = v[j + q];
          }
          if (!p.partial && p.nonfinite) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (col + q < p.N && !isfinite(v[j + q])) atomicOr(p.nonfinite, 1);
          }
          if (relu) {
            if (p.vec_d && col + 3 < p.N) {
              *reinterpret_cast<float4*>(p.D + row * p.ldd + col) =
                  make_float4(sg::relu_np(v[j]), sg::relu_np(v[j + 1]), sg::relu_np(v[j + 2]), sg::relu_np(v[j + 3]));
            } else {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (col + q < p.N) p.D[row * p.ldd + col + q] = sg::relu_np(v[j + q]);
            }
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ---------------- single-thread UMMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = sm100::idesc_tf32(BM, BN, false, false);  // smem always K-major
      for (int i = 0; i < nkb; ++i) {
        const int s = i % C::STAGES;
        const uint32_t use = i / C::STAGES;
        sm100::mbar_wait(full + s, use & 1);
        sm100::tc_fence_after();
        const uint32_t st = base + s * C::STAGE;
        const uint32_t a_hi = st, a_lo = st + C::A_TILE;
        const uint32_t b_hi = st + 2 * C::A_TILE, b_lo = b_hi + C::B_TILE;
#pragma unroll
        for (int kk = 0; kk < BK / 8; ++kk) {
          const uint64_t ah = tile_desc(a_hi, kk), al = tile_desc(a_lo, kk);
          const uint64_t bh = tile_desc(b_hi, kk), bl = tile_desc(b_lo, kk);
          sm100::umma_tf32(tmem, ah, bh, idesc, (i > 0 || kk > 0) ? 1u : 0u);
          sm100::umma_tf32(tmem, ah, bl, idesc, 1u);
          sm100::umma_tf32(tmem, al, bh, idesc, 1u);
        }
        sm100::umma_commit(empty + s);  // frees the stage when these MMAs are done
      }
      sm100::umma_commit(done);
    }
    __syncwarp();
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) sm100::tmem_dealloc<C::TMEM_COLS>(tmem);
}

__global__ void tc_splitk_reduce(const float* partial, int splits, int64_t M, int64_t N, void* C,
                                 int64_t ldc, int c_bf16, void* D, int64_t ldd, int d_bf16, int epilogue,
                                 int32_t* nonfinite) {
  const int64_t total = M * N;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    for (int z = 0; z < splits; ++z) s += partial[(int64_t)z * total + t];  // fixed order
    const int64_t m = t / N, n = t % N;
    if (C) sm100::store4(C, c_bf16, m * ldc + n, &s, 1, false);
    if (epilogue == SG_EPI_RELU_DUAL) {
      const float r = sg::relu_np(s);
      sm100::store4(D, d_bf16, m * ldd + n, &r, 1, false);
    }
    if (nonfinite && !isfinite(s)) atomicOr(nonfinite, 1);
  }
}

int pick_bn(int64_t N) { return N <= 64 ? 64 : 128; }

int tc_splits(int64_t M, int64_t N, int64_t K) {
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + pick_bn(N) - 1) / pick_bn(N));
  const int64_t nkb = (K + BK - 1) / BK;
  if (tiles >= 148 || nkb < 16) return 1;
  int64_t s = std::min<int64_t>((2 * 148 + tiles - 1) / tiles, nkb / 8);
  return (int)std::max<int64_t>(1, std::min<int64_t>(s, 64));
}

template <bool A_MN, bool B_MN, int BN>
cudaError_t launch_tc(const TcArgs& p, dim3 grid, cudaStream_t st) {
  auto k = gemm_tf32x3_kernel<A_MN, B_MN, BN>;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::SMEM);
    configured = true;
  }
  k<<<grid, kThreads, Cfg<BN>::SMEM, st>>>(p);
  sg::count_launch();
  return cudaGetLastError();
}

template <int BN>
cudaError_t dispatch_major(bool a_mn, bool b_mn, const TcArgs& p, dim3 grid, cudaStream_t st) {
  if (!a_mn && !b_mn) return launch_tc<false, false, BN>(p, grid, st);
  if (!a_mn && b_mn) return launch_tc<false, true, BN>(p, grid, st);
  if (a_mn && !b_mn) return launch_tc<true, false, BN>(p, grid, st);
  return launch_tc<true, true, BN>(p, grid, st);
}

}  // namespace

int sg_gemm_tma_try(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const float* A, int64_t lda,
                    const float* B, int64_t ldb, void* C, int64_t ldc, int c_bf16, int epilogue, void* D,
                    int64_t ldd, int d_bf16, int32_t* nonfinite, float* partial, int kb_per_split, int n_kb,
                    int gz, cudaStream_t st, cudaError_t* err);

int64_t sg_gemm_tc_workspace_bytes(int64_t M, int64_t N, int64_t K, int prec) {
  (void)prec;
  const int s = tc_splits(M, N, K);
  return s > 1 ? (int64_t)s * M * N * 4 : 0;
}

int sg_gemm_tc(int prec, int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, const float* A,
               int64_t lda, const float* B, int64_t ldb, void* Cv, int64_t ldc, int c_bf16, int epilogue,
               void* Dv, int64_t ldd, int d_bf16, int32_t* nonfinite, void* workspace,
               int64_t workspace_bytes, cudaStream_t st) {
  SG_REQUIRE(prec == SG_GEMM_TF32X3, SG_EINVAL, "tensor-core GEMM precision %d not supported", prec);
  if (K == 0) {
    if (Cv) cudaMemset2DAsync(Cv, ldc * (c_bf16 ? 2 : 4), 0, N * (c_bf16 ? 2 : 4), M, st);
    if (epilogue == SG_EPI_RELU_DUAL) cudaMemset2DAsync(Dv, ldd * (d_bf16 ? 2 : 4), 0, N * (d_bf16 ? 2 : 4), M, st);
    return SG_OK;
  }
  // the LDG-fed fallback kernel writes fp32 C (and D) only
  const bool plain = Cv != nullptr && !c_bf16 && !d_bf16;
  float* C = static_cast<float*>(Cv);
  float* D = static_cast<float*>(Dv);
  // K-major when the reduction dim is contiguous: A stored [M,K] (!trans_a), B stored [N,K] (trans_b)
  const bool a_mn = trans_a != 0, b_mn = trans_b == 0;
  TcArgs p;
  p.A = A; p.B = B; p.C = C; p.D = D;
  p.lda = lda; p.ldb = ldb; p.ldc = ldc; p.ldd = ldd;
  p.M = M; p.N = N; p.K = K;
  p.epilogue = epilogue;
  p.nonfinite = nonfinite;
  p.vec_a = (lda % 4 == 0) && ((uintptr_t)A % 16 == 0);
  p.vec_b = (ldb % 4 == 0) && ((uintptr_t)B % 16 == 0);
  p.vec_c = (ldc % 4 == 0) && ((uintptr_t)C % 16 == 0);
  p.vec_d = D != nullptr && (ldd % 4 == 0) && ((uintptr_t)D % 16 == 0);
  p.n_kb = (int)((K + BK - 1) / BK);
  const int splits = tc_splits(M, N, K);
  p.kb_per_split = (p.n_kb + splits - 1) / splits;
  const int gz = (p.n_kb + p.kb_per_split - 1) / p.kb_per_split;
  p.partial = nullptr;
  if (gz > 1) {
    SG_REQUIRE(workspace && workspace_bytes >= (int64_t)gz * M * N * 4, SG_EBUDGET,
               "tensor-core GEMM split-K workspace too small");
    p.partial = (float*)workspace;
  }
  const int BN = pick_bn(N);
  dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)gz);
  cudaError_t e = cudaSuccess;
  // TMA-fed kernel (gemm_tma.cu) when the operands meet the tensor-map constraints;
  // otherwise the LDG-fed kernel above (any alignment)
  if (!sg_gemm_tma_try(trans_a, trans_b, M, N, K, A, lda, B, ldb, Cv, ldc, c_bf16, epilogue, Dv, ldd, d_bf16,
                       nonfinite, p.partial, p.kb_per_split, p.n_kb, gz, st, &e)) {
    SG_REQUIRE(plain, SG_EINVAL, "tensor-core GEMM: bf16 or absent C needs 16-B aligned operands (TMA path)");
    e = BN == 64 ? dispatch_major<64>(a_mn, b_mn, p, grid, st) : dispatch_major<128>(a_mn, b_mn, p, grid, st);
  }
  if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "tcgen05 gemm launch: %s", cudaGetErrorString(e));
  if (gz > 1) {
    const int64_t total = M * N;
    int g = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
    tc_splitk_reduce<<<g, 256, 0, st>>>(p.partial, gz, M, N, Cv, ldc, c_bf16, Dv, ldd, d_bf16, epilogue,
                                        nonfinite);
    sg::count_launch();
    e = cudaGetLastError();
    if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "split-k reduce: %s", cudaGetErrorString(e));
  }
  return SG_OK;
}
