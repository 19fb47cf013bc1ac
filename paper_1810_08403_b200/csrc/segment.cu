// Unfused Scatter / Gather(max) primitives and the device segment sort (K1, K2, K7).
//
//  * sg_take_rows      -- Scatter, take_rows (tensor.py:424-436)
//  * sg_segment_max    -- Gather(max) + argmax (tensor.py:453-484)
//  * sg_segment_sort   -- stable segment index (ptr, perm) so that segment_sum /
//                         take_rows backward (np.add.at, tensor.py:433, :445) run
//                         as an ordered sg_propagate(PASS) pass.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include "common.h"
#include "vecio.cuh"

namespace {
using sg::VecIO;

// source rows in flight per lane in the fused max gather and its backward: hub rows (R-MAT:
// ~800K edges) are walked by one team, so the kernel time is that row's load-latency chain
#ifndef SG_MAX_DEPTH
#define SG_MAX_DEPTH 12
#endif
constexpr int kMaxDepth = SG_MAX_DEPTH;

template <int DT, int W>
__global__ void take_rows_kernel(const void* X, int64_t ldx, int64_t n_src, const int64_t* idx,
                                 int64_t n, void* out, int64_t ldo, int F, int32_t* err) {
  using IO = VecIO<DT, W>;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int Fv = (F + W - 1) / W;
  for (int64_t k = warp; k < n; k += nwarps) {
    int64_t s = idx[k];
    if (s < 0 || s >= n_src) {
      if (lane == 0) atomicOr(err, 1);
      continue;
    }
    for (int cv = lane; cv < Fv; cv += 32) {
      float v[W];
      IO::ld_nc(X, s * ldx + (int64_t)cv * W, v);
      IO::st(out, k * ldo + (int64_t)cv * W, v, min(W, F - cv * W));
    }
  }
}

// TEAM lanes per segment (narrow rows pack 32/TEAM segments per warp), lanes over column
// vectors; 4 source rows loaded before any is compared (4 reads in flight per lane); strict
// '>' so the first (lowest position) maximum wins; -inf init; empty segment -> empty_fill,
// argmax -1.  argmax = idx[e] (the gathered row, tensor.py:467-469 with rows pre-gathered).
template <int DT, int W, int TEAM>
__global__ void __launch_bounds__(256) segmax_kernel(const int64_t* __restrict__ ptr,
                                                     const int32_t* __restrict__ idx, int64_t n_rows,
                                                     const void* X, int64_t ldx, void* out, int64_t ldo,
                                                     int64_t* arg, int64_t lda, int F, float fill) {
  using IO = VecIO<DT, W>;
  constexpr int RPW = 32 / TEAM;
  const int lane = threadIdx.x & 31, tl = lane % TEAM;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nteams = (((int64_t)gridDim.x * blockDim.x) >> 5) * RPW;
  const int Fv = (F + W - 1) / W;
  for (int64_t r = warp * RPW + lane / TEAM; r < n_rows; r += nteams) {
    const int64_t e0 = __ldg(ptr + r), e1 = __ldg(ptr + r + 1);
    for (int cv = tl; cv < Fv; cv += TEAM) {
      float best[W];
      int64_t barg[W];
#pragma unroll
      for (int k = 0; k < W; ++k) {
        best[k] = -INFINITY;
        barg[k] = -1;
      }
      int64_t e = e0;
      for (; e + 4 <= e1; e += 4) {
        int64_t s[4];
        float v[4][W];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          s[u] = __ldg(idx + e + u);
          IO::ld_nc(X, s[u] * ldx + (int64_t)cv * W, v[u]);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int k = 0; k < W; ++k)
            if (v[u][k] > best[k]) {
              best[k] = v[u][k];
              barg[k] = s[u];
            }
      }
      for (; e < e1; ++e) {
        const int64_t sv = __ldg(idx + e);
        float v[W];
        IO::ld_nc(X, sv * ldx + (int64_t)cv * W, v);
#pragma unroll
        for (int k = 0; k < W; ++k)
          if (v[k] > best[k]) {
            best[k] = v[k];
            barg[k] = sv;
          }
      }
      const int nvalid = min(W, F - cv * W);
#pragma unroll
      for (int k = 0; k < W; ++k) {
        if (barg[k] < 0) best[k] = fill;
        if (k < nvalid) arg[r * lda + (int64_t)cv * W + k] = barg[k];
      }
      IO::st(out, r * ldo + (int64_t)cv * W, best, nvalid);
    }
  }
}

template <int DT>
__global__ void segmax_bwd_kernel(const void* g, int64_t ldg, const int64_t* arg, int64_t lda,
                                  int64_t n_rows, void* gx, int64_t ldx, int F) {
  using IO = VecIO<DT, 1>;
  const int64_t total = n_rows * (int64_t)F;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / F, f = t % F;
    const int64_t a = arg[r * lda + f];
    if (a < 0) continue;
    float v;
    IO::ld_nc(g, r * ldg + f, &v);
    IO::st(gx, a * ldx + f, &v, 1);  // each (row, col) has at most one argmax owner
  }
}

__global__ void seg_keys_kernel(const int64_t* seg, int64_t n, int64_t n_seg, int32_t* keys,
                                int32_t* vals, int32_t* err) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (int64_t)gridDim.x * blockDim.x) {
    int64_t s = seg[k];
    if (s < 0 || s >= n_seg) {
      atomicOr(err, 1);
      s = 0;
    }
    keys[k] = (int32_t)s;
    vals[k] = (int32_t)k;
  }
}

// ptr[s] = number of sorted keys < s (lower bound), ptr[n_seg] = n.
__global__ void seg_ptr_kernel(const int32_t* sorted, int64_t n, int64_t n_seg, int64_t* ptr) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s <= n_seg;
       s += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (sorted[mid] < s) lo = mid + 1;
      else hi = mid;
    }
    ptr[s] = (s == n_seg) ? n : lo;
  }
}

inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
inline bool aligned(const void* p, int b) { return ((uintptr_t)p % b) == 0; }

int end_bit_for(int64_t n_seg) {
  int b = 1;
  while ((int64_t(1) << b) < n_seg) ++b;
  return b;
}

size_t cub_temp_bytes(int64_t n, int64_t n_seg) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, (const int32_t*)nullptr, (int32_t*)nullptr,
                                  (const int32_t*)nullptr, (int32_t*)nullptr, (int)n, 0,
                                  end_bit_for(n_seg));
  return bytes;
}

int grid_for(int64_t work, int per_block) {
  int64_t g = (work + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 32));
}

// Fused Gather(max) over a CSC index (MP-GCN): out[u] = max over the
// in-edges of Y[src] with the position of the first maximum recorded as the argmax
// ("ties broken by lowest CSC edge index"); empty rows -> fill, argmax -1.
//
// Positions are global: base + in-chunk CSC position, base = the chunk's offset in the
// source-interval-major flattening of the 2D grid, so for a destination interval the
// chunks C_0j, C_1j, ... (visited in that order, `accumulate` carrying the running
// max/argmax in out/arg) produce exactly segment_max over the flattened edge list.
// `finalize` applies the empty fill on the last chunk of the chain.
//
// TEAM lanes per destination row (narrow pooled widths pack 32/TEAM rows per warp);
// 4 source rows are loaded before any is compared so 4 row reads are in flight per lane.
template <int W, int TEAM>
__global__ void __launch_bounds__(256) maxgather_kernel(
    const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx, int64_t n_rows,
    const float* __restrict__ Y, int64_t ldy, float* __restrict__ out, int64_t ldo,
    int32_t* __restrict__ arg, int64_t lda, int F, float fill, int64_t base, int accumulate,
    int finalize) {
  constexpr int RPW = 32 / TEAM;
  const int lane = threadIdx.x & 31, tl = lane % TEAM;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nteams = (((int64_t)gridDim.x * blockDim.x) >> 5) * RPW;
  const int Fv = (F + W - 1) / W;
  for (int64_t r = warp * RPW + lane / TEAM; r < n_rows; r += nteams) {
    const int64_t e0 = __ldg(ptr + r), e1 = __ldg(ptr + r + 1);
    for (int cv = tl; cv < Fv; cv += TEAM) {
      const int c0 = cv * W;
      float best[W];
      int32_t barg[W];
#pragma unroll
      for (int k = 0; k < W; ++k) {
        best[k] = -INFINITY;
        barg[k] = -1;
        if (accumulate && c0 + k < F) {
          barg[k] = arg[r * lda + c0 + k];
          if (barg[k] >= 0) best[k] = out[r * ldo + c0 + k];
        }
      }
      int64_t e = e0;
      for (; e + kMaxDepth <= e1; e += kMaxDepth) {
        float v[kMaxDepth][W];
#pragma unroll
        for (int u = 0; u < kMaxDepth; ++u) {
          const float* row = Y + (int64_t)__ldg(idx + e + u) * ldy + c0;
          if (W == 4) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(row));
            v[u][0] = q.x; v[u][1 % W] = q.y; v[u][2 % W] = q.z; v[u][3 % W] = q.w;
          } else {
            v[u][0] = __ldg(row);
          }
        }
#pragma unroll
        for (int u = 0; u < kMaxDepth; ++u)
#pragma unroll
          for (int k = 0; k < W; ++k)
            if (v[u][k] > best[k]) {  // strict '>' : the lowest position wins (tensor.py:467)
              best[k] = v[u][k];
              barg[k] = (int32_t)(base + e + u);
            }
      }
      for (; e < e1; ++e) {
        const float* row = Y + (int64_t)__ldg(idx + e) * ldy + c0;
        float v[W];
        if (W == 4) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(row));
          v[0] = q.x; v[1 % W] = q.y; v[2 % W] = q.z; v[3 % W] = q.w;
        } else {
          v[0] = __ldg(row);
        }
#pragma unroll
        for (int k = 0; k < W; ++k)
          if (v[k] > best[k]) {
            best[k] = v[k];
            barg[k] = (int32_t)(base + e);
          }
      }
#pragma unroll
      for (int k = 0; k < W; ++k) {
        if (c0 + k < F) {
          out[r * ldo + c0 + k] = (finalize && barg[k] < 0) ? fill : best[k];
          arg[r * lda + c0 + k] = barg[k];
        }
      }
    }
  }
}

// Backward of the fused max gather over the transposed (CSR) index: dY[v] = sum over
// out-edges k of v, in CSR order (= the forward edge-list order, tensor.py:431-434), of
// dA[dst_k] where the destination's argmax is this edge (pos_base + pos_k = its global
// position), else +0.0 -- exactly tensor.py:473-482 followed by take_rows' backward.
// `accumulate` continues the sum of the previous chunk of the same source interval
// (chunks C_i0, C_i1, ... in that order).  No atomics.
template <int W, int TEAM>
__global__ void __launch_bounds__(256) maxgather_bwd_kernel(
    const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx, const int32_t* __restrict__ pos,
    int64_t n_rows, const float* __restrict__ G, int64_t ldg, const int32_t* __restrict__ arg,
    int64_t lda, float* __restrict__ out, int64_t ldo, int F, const float* __restrict__ mask,
    int64_t ldm, int64_t pos_base, int accumulate) {
  constexpr int RPW = 32 / TEAM;
  const int lane = threadIdx.x & 31, tl = lane % TEAM;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nteams = (((int64_t)gridDim.x * blockDim.x) >> 5) * RPW;
  const int Fv = (F + W - 1) / W;
  for (int64_t r = warp * RPW + lane / TEAM; r < n_rows; r += nteams) {
    const int64_t e0 = __ldg(ptr + r), e1 = __ldg(ptr + r + 1);
    for (int cv = tl; cv < Fv; cv += TEAM) {
      const int c0 = cv * W;
      float acc[W];
#pragma unroll
      for (int k = 0; k < W; ++k) acc[k] = (accumulate && c0 + k < F) ? out[r * ldo + c0 + k] : 0.f;
      int64_t e = e0;
      for (; e + kMaxDepth <= e1; e += kMaxDepth) {  // kMaxDepth edges' rows in flight (G + arg)
        float g[kMaxDepth][W];
        int32_t a[kMaxDepth][W], p[kMaxDepth];
#pragma unroll
        for (int u = 0; u < kMaxDepth; ++u) {
          const int64_t d = __ldg(idx + e + u);
          p[u] = (int32_t)(pos_base + __ldg(pos + e + u));
          if (W == 4) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(G + d * ldg + c0));
            const int4 t = __ldg(reinterpret_cast<const int4*>(arg + d * lda + c0));
            g[u][0] = q.x; g[u][1 % W] = q.y; g[u][2 % W] = q.z; g[u][3 % W] = q.w;
            a[u][0] = t.x; a[u][1 % W] = t.y; a[u][2 % W] = t.z; a[u][3 % W] = t.w;
          } else {
            g[u][0] = __ldg(G + d * ldg + c0);
            a[u][0] = __ldg(arg + d * lda + c0);
          }
        }
#pragma unroll
        for (int u = 0; u < kMaxDepth; ++u)
#pragma unroll
          for (int k = 0; k < W; ++k) acc[k] = __fadd_rn(acc[k], a[u][k] == p[u] ? g[u][k] : 0.f);
      }
      for (; e < e1; ++e) {
        const int64_t d = __ldg(idx + e);
        const int32_t pp = (int32_t)(pos_base + __ldg(pos + e));
#pragma unroll
        for (int k = 0; k < W; ++k) {
          const int c = min(c0 + k, F - 1);
          acc[k] = __fadd_rn(acc[k], __ldg(arg + d * lda + c) == pp ? __ldg(G + d * ldg + c) : 0.f);
        }
      }
#pragma unroll
      for (int k = 0; k < W; ++k) {
        if (c0 + k < F) {
          float v = acc[k];
          if (mask) v = __fmul_rn(v, __ldg(mask + r * ldm + c0 + k) > 0.f ? 1.f : 0.f);
          out[r * ldo + c0 + k] = v;
        }
      }
    }
  }
}

// ---------------------------------------------------------------- plan-driven max gather
// Hub-heavy passes (R-MAT: rows of ~10^5-10^6 edges) cannot be left to one team per row: the
// kernel would last as long as the heaviest row.  These variants consume the pass's work plan
// (sg_item / sg_split, as sg_propagate): warps pull items from an atomic queue; a split item
// is one subgroup of <= T edges of a heavy row whose partial lands in the workspace, and the
// last subgroup to finish combines the partials in subgroup order.
//  * forward: max and argmax are exact, so the split result equals the sequential one bit for
//    bit (partials are combined lowest position first with strict '>');
//  * backward: a sum, so a split row follows the subgroup rule of every propagation pass
//    (oracle/saga.py:seq_sum_rows).
// split rows: partials combined by a second launch (1) or by the last subgroup's warp (0).
// MP-GCN step on the 28.6M-edge R-MAT graph (tools/mp_time.py, profiles/r02_max_split_ab.txt):
// backward passes 1.73 / 1.97 -> 1.64 / 1.83 ms with the launch, forward passes 1.26 / 1.19 ->
// 1.34 / 1.29 ms -- so the backward (a sum over subgroups) uses it and the forward keeps the
// in-pass max/argmax combine
#ifndef SG_MAX_SPLIT_FWD
#define SG_MAX_SPLIT_FWD 0
#endif
#ifndef SG_MAX_SPLIT_BWD
#define SG_MAX_SPLIT_BWD 1
#endif
struct MaxPlan {
  const int64_t* ptr;
  const int32_t* idx;
  const int32_t* pos;    // bwd: CSC position per CSR edge
  const sg_item* items;
  const sg_split* splits;
  int32_t n_items;
  int32_t n_splits;
  int32_t* queue;
  int32_t* counters;
  float* pval;           // [n_slots][pld]
  int32_t* parg;         // [n_slots][pld] (fwd)
  int64_t pld;
  const float* Y;        // fwd: gathered rows; bwd: dA rows
  int64_t ldy;
  float* out;
  int64_t ldo;
  int32_t* arg;          // fwd: out argmax; bwd: argmax of the destinations
  int64_t* arg64;        // fwd (segment_max primitive): argmax written as the gathered row idx[pos]
  int64_t lda;
  const float* mask;
  int64_t ldm;
  int F;
  float fill;
  int64_t base;
  int accumulate, finalize;
};

template <int W>
__device__ __forceinline__ void ld_vec(const float* p, float (&v)[W]) {
  if constexpr (W == 4) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = q.x; v[1 % W] = q.y; v[2 % W] = q.z; v[3 % W] = q.w;
  } else {
    v[0] = __ldg(p);
  }
}

template <int W>
__device__ __forceinline__ void ld_ivec(const int32_t* p, int32_t (&v)[W]) {
  if constexpr (W == 4) {
    const int4 q = __ldg(reinterpret_cast<const int4*>(p));
    v[0] = q.x; v[1 % W] = q.y; v[2 % W] = q.z; v[3 % W] = q.w;
  } else {
    v[0] = __ldg(p);
  }
}

template <int W>
__global__ void __launch_bounds__(256) maxgather_plan_kernel(const MaxPlan a) {
  const int lane = threadIdx.x & 31;
  const int Fv = (a.F + W - 1) / W;
  for (;;) {
    int it = 0;
    if (lane == 0) it = atomicAdd(a.queue, 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= a.n_items) break;
    const sg_item item = a.items[it];
    const bool split = item.split >= 0;
    for (int r = item.row_begin; r < item.row_end; ++r) {
      const int64_t e0 = split ? item.e_begin : __ldg(a.ptr + r);
      const int64_t e1 = split ? item.e_end : __ldg(a.ptr + r + 1);
      for (int cv = lane; cv < Fv; cv += 32) {
        const int c0 = cv * W;
        float best[W];
        int32_t barg[W];
#pragma unroll
        for (int k = 0; k < W; ++k) {
          best[k] = -INFINITY;
          barg[k] = -1;
          if (!split && a.accumulate && c0 + k < a.F) {
            barg[k] = a.arg[r * a.lda + c0 + k];
            if (barg[k] >= 0) best[k] = a.out[r * a.ldo + c0 + k];
          }
        }
        int64_t e = e0;
        for (; e + kMaxDepth <= e1; e += kMaxDepth) {
          float v[kMaxDepth][W];
#pragma unroll
          for (int u = 0; u < kMaxDepth; ++u) ld_vec<W>(a.Y + (int64_t)__ldg(a.idx + e + u) * a.ldy + c0, v[u]);
#pragma unroll
          for (int u = 0; u < kMaxDepth; ++u)
#pragma unroll
            for (int k = 0; k < W; ++k)
              if (v[u][k] > best[k]) {
                best[k] = v[u][k];
                barg[k] = (int32_t)(a.base + e + u);
              }
        }
        for (; e < e1; ++e) {
          float v[W];
          ld_vec<W>(a.Y + (int64_t)__ldg(a.idx + e) * a.ldy + c0, v);
#pragma unroll
          for (int k = 0; k < W; ++k)
            if (v[k] > best[k]) {
              best[k] = v[k];
              barg[k] = (int32_t)(a.base + e);
            }
        }
        if (!split) {
#pragma unroll
          for (int k = 0; k < W; ++k)
            if (c0 + k < a.F) {
              a.out[r * a.ldo + c0 + k] = (a.finalize && barg[k] < 0) ? a.fill : best[k];
              if (a.arg64)
                a.arg64[r * a.lda + c0 + k] = barg[k] >= 0 ? (int64_t)__ldg(a.idx + barg[k]) : -1;
              else
                a.arg[r * a.lda + c0 + k] = barg[k];
            }
        } else {
          const int64_t slot = a.splits[item.split].slot0 + item.sub;
#pragma unroll
          for (int k = 0; k < W; ++k)
            if (c0 + k < a.F) {
              __stcg(a.pval + slot * a.pld + c0 + k, best[k]);
              __stcg(a.parg + slot * a.pld + c0 + k, barg[k]);
            }
        }
      }
    }
#if !SG_MAX_SPLIT_FWD
    if (split) {
      const sg_split sp = a.splits[item.split];
      __threadfence();
      __syncwarp();
      int ticket = 0;
      if (lane == 0) ticket = atomicAdd(a.counters + item.split, 1);
      ticket = __shfl_sync(0xffffffffu, ticket, 0);
      if (ticket == sp.n_sub - 1) {
        __threadfence();
        const int64_t r = sp.row;
        for (int c = lane; c < a.F; c += 32) {
          float best = -INFINITY;
          int32_t barg = -1;
          if (a.accumulate) {
            barg = a.arg[r * a.lda + c];
            if (barg >= 0) best = a.out[r * a.ldo + c];
          }
          for (int q = 0; q < sp.n_sub; ++q) {  // ascending positions: strict '>' keeps the first
            const float v = __ldcg(a.pval + (sp.slot0 + q) * a.pld + c);
            const int32_t g = __ldcg(a.parg + (sp.slot0 + q) * a.pld + c);
            if (g >= 0 && v > best) {
              best = v;
              barg = g;
            }
          }
          a.out[r * a.ldo + c] = (a.finalize && barg < 0) ? a.fill : best;
          if (a.arg64)
            a.arg64[r * a.lda + c] = barg >= 0 ? (int64_t)__ldg(a.idx + barg) : -1;
          else
            a.arg[r * a.lda + c] = barg;
        }
        if (lane == 0) a.counters[item.split] = 0;
      }
    }
#endif
  }
}

template <int W>
__global__ void __launch_bounds__(256) maxgather_bwd_plan_kernel(const MaxPlan a) {
  const int lane = threadIdx.x & 31;
  const int Fv = (a.F + W - 1) / W;
  for (;;) {
    int it = 0;
    if (lane == 0) it = atomicAdd(a.queue, 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= a.n_items) break;
    const sg_item item = a.items[it];
    const bool split = item.split >= 0;
    for (int r = item.row_begin; r < item.row_end; ++r) {
      const int64_t e0 = split ? item.e_begin : __ldg(a.ptr + r);
      const int64_t e1 = split ? item.e_end : __ldg(a.ptr + r + 1);
      for (int cv = lane; cv < Fv; cv += 32) {
        const int c0 = cv * W;
        float acc[W];
#pragma unroll
        for (int k = 0; k < W; ++k)
          acc[k] = (!split && a.accumulate && c0 + k < a.F) ? a.out[r * a.ldo + c0 + k] : 0.f;
        int64_t e = e0;
        for (; e + kMaxDepth <= e1; e += kMaxDepth) {
          float g[kMaxDepth][W];
          int32_t t[kMaxDepth][W], p[kMaxDepth];
#pragma unroll
          for (int u = 0; u < kMaxDepth; ++u) {
            const int64_t d = __ldg(a.idx + e + u);
            p[u] = (int32_t)(a.base + __ldg(a.pos + e + u));
            ld_vec<W>(a.Y + d * a.ldy + c0, g[u]);
            ld_ivec<W>(a.arg + d * a.lda + c0, t[u]);
          }
#pragma unroll
          for (int u = 0; u < kMaxDepth; ++u)
#pragma unroll
            for (int k = 0; k < W; ++k) acc[k] = __fadd_rn(acc[k], t[u][k] == p[u] ? g[u][k] : 0.f);
        }
        for (; e < e1; ++e) {
          const int64_t d = __ldg(a.idx + e);
          const int32_t pp = (int32_t)(a.base + __ldg(a.pos + e));
          float g[W];
          int32_t t[W];
          ld_vec<W>(a.Y + d * a.ldy + c0, g);
          ld_ivec<W>(a.arg + d * a.lda + c0, t);
#pragma unroll
          for (int k = 0; k < W; ++k) acc[k] = __fadd_rn(acc[k], t[k] == pp ? g[k] : 0.f);
        }
        if (!split) {
#pragma unroll
          for (int k = 0; k < W; ++k)
            if (c0 + k < a.F) {
              float v = acc[k];
              if (a.mask) v = __fmul_rn(v, __ldg(a.mask + r * a.ldm + c0 + k) > 0.f ? 1.f : 0.f);
              a.out[r * a.ldo + c0 + k] = v;
            }
        } else {
          const int64_t slot = a.splits[item.split].slot0 + item.sub;
#pragma unroll
          for (int k = 0; k < W; ++k)
            if (c0 + k < a.F) __stcg(a.pval + slot * a.pld + c0 + k, acc[k]);
        }
      }
    }
#if !SG_MAX_SPLIT_BWD
    if (split) {
      const sg_split sp = a.splits[item.split];
      __threadfence();
      __syncwarp();
      int ticket = 0;
      if (lane == 0) ticket = atomicAdd(a.counters + item.split, 1);
      ticket = __shfl_sync(0xffffffffu, ticket, 0);
      if (ticket == sp.n_sub - 1) {
        __threadfence();
        const int64_t r = sp.row;
        for (int c = lane; c < a.F; c += 32) {
          float v = a.accumulate ? a.out[r * a.ldo + c] : 0.f;
          for (int q = 0; q < sp.n_sub; ++q) v = __fadd_rn(v, __ldcg(a.pval + (sp.slot0 + q) * a.pld + c));
          if (a.mask) v = __fmul_rn(v, __ldg(a.mask + r * a.ldm + c) > 0.f ? 1.f : 0.f);
          a.out[r * a.ldo + c] = v;
        }
        if (lane == 0) a.counters[item.split] = 0;
      }
    }
#endif
  }
}

// Split-row combine launches (SG_MAX_SPLIT_FWD / _BWD, as sg_propagate's combine_kernel): one
// thread per (split row, column), the row's partials read lowest subgroup first with U of them
// in flight.  Forward: strict '>' over ascending positions keeps the first maximum (bitwise the
// in-pass combine); backward: the subgroup sums added in subgroup order.
#if SG_MAX_SPLIT_FWD
__global__ void __launch_bounds__(256) maxgather_combine_kernel(const MaxPlan a, int tps) {
  constexpr int U = 8;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t sid = t / tps;
  const int c = (int)(t - sid * tps);
  if (sid >= a.n_splits || c >= a.F) return;
  const sg_split sp = a.splits[sid];
  const int64_t r = sp.row;
  float best = -INFINITY;
  int32_t barg = -1;
  if (a.accumulate) {
    barg = a.arg[r * a.lda + c];
    if (barg >= 0) best = a.out[r * a.ldo + c];
  }
  #pragma unroll 1
  for (int q = 0; q < sp.n_sub; q += U) {
    float v[U];
    int32_t g[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (q + u < sp.n_sub) {
        v[u] = __ldcg(a.pval + (sp.slot0 + q + u) * a.pld + c);
        g[u] = __ldcg(a.parg + (sp.slot0 + q + u) * a.pld + c);
      }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (q + u < sp.n_sub && g[u] >= 0 && v[u] > best) {
        best = v[u];
        barg = g[u];
      }
  }
  a.out[r * a.ldo + c] = (a.finalize && barg < 0) ? a.fill : best;
  if (a.arg64)
    a.arg64[r * a.lda + c] = barg >= 0 ? (int64_t)__ldg(a.idx + barg) : -1;
  else
    a.arg[r * a.lda + c] = barg;
}
#endif

__global__ void __launch_bounds__(256) maxgather_bwd_combine_kernel(const MaxPlan a, int tps) {
  constexpr int U = 16;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t sid = t / tps;
  const int c = (int)(t - sid * tps);
  if (sid >= a.n_splits || c >= a.F) return;
  const sg_split sp = a.splits[sid];
  const int64_t r = sp.row;
  float v = a.accumulate ? a.out[r * a.ldo + c] : 0.f;
  #pragma unroll 1
  for (int q = 0; q < sp.n_sub; q += U) {
    float x[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (q + u < sp.n_sub) x[u] = __ldcg(a.pval + (sp.slot0 + q + u) * a.pld + c);
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (q + u < sp.n_sub) v = __fadd_rn(v, x[u]);
  }
  if (a.mask) v = __fmul_rn(v, __ldg(a.mask + r * a.ldm + c) > 0.f ? 1.f : 0.f);
  a.out[r * a.ldo + c] = v;
}

int team_for(int Fv) {
  int t = 1;
  while (t < Fv && t < 32) t <<= 1;
  return t;
}

}  // namespace

extern "C" {

int sg_max_gather(const int64_t* ptr, const int32_t* idx, int64_t n_rows, const float* Y, int64_t ldy,
                  float* out, int64_t ldo, int32_t* argpos, int64_t lda, int64_t F, float empty_fill,
                  int64_t pos_base, int accumulate, int finalize, void* stream) {
  if (n_rows == 0 || F == 0) return SG_OK;
  SG_REQUIRE(ptr && idx && Y && out && argpos, SG_EINVAL, "max_gather: null pointer");
  const bool vec = (F % 4 == 0) && (ldy % 4 == 0) && aligned(Y, 16);
  const int team = team_for(vec ? (int)(F / 4) : (int)F);
  const int g = grid_for(n_rows * team, 256);
  cudaStream_t st = (cudaStream_t)stream;
#define SG_MG(Wv, T)                                                                        \
  maxgather_kernel<Wv, T><<<g, 256, 0, st>>>(ptr, idx, n_rows, Y, ldy, out, ldo, argpos, lda, \
                                             (int)F, empty_fill, pos_base, accumulate, finalize)
#define SG_MG_TEAMS(Wv)                         \
  switch (team) {                               \
    case 1: SG_MG(Wv, 1); break;                \
    case 2: SG_MG(Wv, 2); break;                \
    case 4: SG_MG(Wv, 4); break;                \
    case 8: SG_MG(Wv, 8); break;                \
    case 16: SG_MG(Wv, 16); break;              \
    default: SG_MG(Wv, 32); break;              \
  }
  if (vec) {
    SG_MG_TEAMS(4)
  } else {
    SG_MG_TEAMS(1)
  }
#undef SG_MG_TEAMS
#undef SG_MG
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "max_gather launch: %s", cudaGetErrorString(e));
  sg::count_launch(1);
  return SG_OK;
}

int sg_max_gather_bwd(const int64_t* ptr, const int32_t* idx, const int32_t* pos, int64_t n_rows,
                      const float* G, int64_t ldg, const int32_t* argpos, int64_t lda, float* out,
                      int64_t ldo, int64_t F, const float* mask, int64_t ldm, int64_t pos_base,
                      int accumulate, void* stream) {
  if (n_rows == 0 || F == 0) return SG_OK;
  SG_REQUIRE(ptr && idx && pos && G && argpos && out, SG_EINVAL, "max_gather_bwd: null pointer");
  const bool vec = (F % 4 == 0) && (ldg % 4 == 0) && (lda % 4 == 0) && aligned(G, 16) &&
                   aligned(argpos, 16);
  const int team = team_for(vec ? (int)(F / 4) : (int)F);
  const int g = grid_for(n_rows * team, 256);
  cudaStream_t st = (cudaStream_t)stream;
#define SG_MB(Wv, T)                                                                              \
  maxgather_bwd_kernel<Wv, T><<<g, 256, 0, st>>>(ptr, idx, pos, n_rows, G, ldg, argpos, lda, out, \
                                                 ldo, (int)F, mask, ldm, pos_base, accumulate)
#define SG_MB_TEAMS(Wv)                         \
  switch (team) {                               \
    case 1: SG_MB(Wv, 1); break;                \
    case 2: SG_MB(Wv, 2); break;                \
    case 4: SG_MB(Wv, 4); break;                \
    case 8: SG_MB(Wv, 8); break;                \
    case 16: SG_MB(Wv, 16); break;              \
    default: SG_MB(Wv, 32); break;              \
  }
  if (vec) {
    SG_MB_TEAMS(4)
  } else {
    SG_MB_TEAMS(1)
  }
#undef SG_MB_TEAMS
#undef SG_MB
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "max_gather_bwd launch: %s", cudaGetErrorString(e));
  sg::count_launch(1);
  return SG_OK;
}

int64_t sg_max_plan_workspace_bytes(int64_t n_splits, int64_t n_slots, int64_t F) {
  const int64_t pld = (F + 3) / 4 * 4;
  return 256 + (4 * std::max<int64_t>(n_splits, 1) + 255) / 256 * 256 + n_slots * pld * 8;
}

static int max_plan_launch(bool bwd, const int64_t* ptr, const int32_t* idx, const int32_t* pos,
                           const sg_item* items, int64_t n_items, const sg_split* splits, int64_t n_splits,
                           int64_t n_slots, const float* Y, int64_t ldy, float* out, int64_t ldo, int32_t* arg,
                           int64_t lda, const float* mask, int64_t ldm, int64_t F, float fill, int64_t base,
                           int accumulate, int finalize, void* ws, int64_t ws_bytes, void* stream,
                           int64_t* arg64 = nullptr) {
  if (n_items == 0 || F == 0) return SG_OK;
  SG_REQUIRE(ptr && idx && items && Y && out && (arg || arg64) && (!bwd || pos), SG_EINVAL,
             "max plan: null pointer");
  SG_REQUIRE(!arg64 || (!bwd && !accumulate), SG_EINVAL, "max plan: int64 argmax is forward-only");
  SG_REQUIRE(n_splits == 0 || splits, SG_EINVAL, "max plan: split records missing");
  SG_REQUIRE(ws && ws_bytes >= sg_max_plan_workspace_bytes(n_splits, n_slots, F), SG_EBUDGET,
             "max plan workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  char* w = static_cast<char*>(ws);
  const int64_t cbytes = (4 * std::max<int64_t>(n_splits, 1) + 255) / 256 * 256;
  const int64_t pld = (F + 3) / 4 * 4;
  MaxPlan a;
  a.ptr = ptr; a.idx = idx; a.pos = pos; a.items = items; a.splits = splits;
  a.n_items = (int32_t)n_items;
  a.n_splits = (int32_t)n_splits;
  a.queue = reinterpret_cast<int32_t*>(w);
  a.counters = reinterpret_cast<int32_t*>(w + 256);
  a.pval = reinterpret_cast<float*>(w + 256 + cbytes);
  a.parg = reinterpret_cast<int32_t*>(w + 256 + cbytes + n_slots * pld * 4);
  a.pld = pld;
  a.Y = Y; a.ldy = ldy; a.out = out; a.ldo = ldo; a.arg = arg; a.arg64 = arg64; a.lda = lda;
  a.mask = mask; a.ldm = ldm;
  a.F = (int)F; a.fill = fill; a.base = base; a.accumulate = accumulate; a.finalize = finalize;
  cudaError_t e = cudaMemsetAsync(w, 0, 256 + cbytes, st);
  if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "memset: %s", cudaGetErrorString(e));
  const bool vec = (F % 4 == 0) && (ldy % 4 == 0) && (lda % 4 == 0) && aligned(Y, 16) &&
                   (arg64 || aligned(arg, 16));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n_items + 7) / 8, (int64_t)sms * 8));
  if (bwd) {
    if (vec) maxgather_bwd_plan_kernel<4><<<grid, 256, 0, st>>>(a);
    else maxgather_bwd_plan_kernel<1><<<grid, 256, 0, st>>>(a);
  } else {
    if (vec) maxgather_plan_kernel<4><<<grid, 256, 0, st>>>(a);
    else maxgather_plan_kernel<1><<<grid, 256, 0, st>>>(a);
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "max plan launch: %s", cudaGetErrorString(e));
  sg::count_launch(1);
  if (n_splits > 0 && (bwd ? SG_MAX_SPLIT_BWD : SG_MAX_SPLIT_FWD)) {
    const int tps = (int)((F + 31) / 32 * 32);
    const int64_t blocks = (n_splits * tps + 255) / 256;
    if (bwd) maxgather_bwd_combine_kernel<<<(unsigned)blocks, 256, 0, st>>>(a, tps);
#if SG_MAX_SPLIT_FWD
    else maxgather_combine_kernel<<<(unsigned)blocks, 256, 0, st>>>(a, tps);
#endif
    e = cudaGetLastError();
    if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "max plan combine launch: %s", cudaGetErrorString(e));
    sg::count_launch(1);
  }
  return SG_OK;
}

int sg_max_gather_plan(const int64_t* ptr, const int32_t* idx, const sg_item* items, int64_t n_items,
                       const sg_split* splits, int64_t n_splits, int64_t n_slots, const float* Y, int64_t ldy,
                       float* out, int64_t ldo, int32_t* argpos, int64_t lda, int64_t F, float empty_fill,
                       int64_t pos_base, int accumulate, int finalize, void* workspace,
                       int64_t workspace_bytes, void* stream) {
  return max_plan_launch(false, ptr, idx, nullptr, items, n_items, splits, n_splits, n_slots, Y, ldy, out, ldo,
                         argpos, lda, nullptr, 0, F, empty_fill, pos_base, accumulate, finalize, workspace,
                         workspace_bytes, stream);
}

int sg_segment_max_plan(const int64_t* ptr, const int32_t* idx, const sg_item* items, int64_t n_items,
                        const sg_split* splits, int64_t n_splits, int64_t n_slots, const float* X, int64_t ldx,
                        float* out, int64_t ldo, int64_t* argmax, int64_t lda, int64_t F, float empty_fill,
                        void* workspace, int64_t workspace_bytes, void* stream) {
  return max_plan_launch(false, ptr, idx, nullptr, items, n_items, splits, n_splits, n_slots, X, ldx, out, ldo,
                         nullptr, lda, nullptr, 0, F, empty_fill, 0, 0, 1, workspace, workspace_bytes, stream,
                         argmax);
}

int sg_max_gather_bwd_plan(const int64_t* ptr, const int32_t* idx, const int32_t* pos, const sg_item* items,
                           int64_t n_items, const sg_split* splits, int64_t n_splits, int64_t n_slots,
                           const float* G, int64_t ldg, const int32_t* argpos, int64_t lda, float* out,
                           int64_t ldo, int64_t F, const float* mask, int64_t ldm, int64_t pos_base,
                           int accumulate, void* workspace, int64_t workspace_bytes, void* stream) {
  return max_plan_launch(true, ptr, idx, pos, items, n_items, splits, n_splits, n_slots, G, ldg, out, ldo,
                         const_cast<int32_t*>(argpos), lda, mask, ldm, F, 0.f, pos_base, accumulate, 0,
                         workspace, workspace_bytes, stream);
}

int sg_take_rows(int dtype, const void* X, int64_t ldx, int64_t n_src, const int64_t* idx,
                 int64_t n, void* out, int64_t ldo, int64_t F, int32_t* err_flag, void* stream) {
  if (n == 0 || F == 0) return SG_OK;
  SG_REQUIRE(X && idx && out && err_flag, SG_EINVAL, "take_rows: null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  const int g = grid_for(n * 32, 256);
  if (dtype == SG_F32) {
    if (ldx % 4 == 0 && ldo % 4 == 0 && aligned(X, 16) && aligned(out, 16))
      take_rows_kernel<SG_F32, 4><<<g, 256, 0, st>>>(X, ldx, n_src, idx, n, out, ldo, (int)F, err_flag);
    else
      take_rows_kernel<SG_F32, 1><<<g, 256, 0, st>>>(X, ldx, n_src, idx, n, out, ldo, (int)F, err_flag);
  } else {
    if (ldx % 8 == 0 && ldo % 8 == 0 && aligned(X, 16) && aligned(out, 16))
      take_rows_kernel<SG_BF16, 8><<<g, 256, 0, st>>>(X, ldx, n_src, idx, n, out, ldo, (int)F, err_flag);
    else
      take_rows_kernel<SG_BF16, 1><<<g, 256, 0, st>>>(X, ldx, n_src, idx, n, out, ldo, (int)F, err_flag);
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "take_rows launch: %s", cudaGetErrorString(e));
  sg::count_launch(1);
  return SG_OK;
}

int sg_segment_max(int dtype, const int64_t* ptr, const int32_t* idx, int64_t n_rows,
                   const void* X, int64_t ldx, void* out, int64_t ldo, int64_t* argmax,
                   int64_t lda, int64_t F, float empty_fill, void* stream) {
  if (n_rows == 0 || F == 0) return SG_OK;
  SG_REQUIRE(ptr && idx && X && out && argmax, SG_EINVAL, "segment_max: null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  const bool vec = dtype == SG_F32 && ldx % 4 == 0 && ldo % 4 == 0 && aligned(X, 16) && aligned(out, 16);
  const int team = team_for(vec ? (int)((F + 3) / 4) : (int)F);
  const int g = grid_for(n_rows * team, 256);
#define SG_SM(DTv, Wv, T) \
  segmax_kernel<DTv, Wv, T><<<g, 256, 0, st>>>(ptr, idx, n_rows, X, ldx, out, ldo, argmax, lda, (int)F, empty_fill)
#define SG_SM_TEAMS(DTv, Wv)       \
  switch (team) {                  \
    case 1: SG_SM(DTv, Wv, 1); break;   \
    case 2: SG_SM(DTv, Wv, 2); break;   \
    case 4: SG_SM(DTv, Wv, 4); break;   \
    case 8: SG_SM(DTv, Wv, 8); break;   \
    case 16: SG_SM(DTv, Wv, 16); break; \
    default: SG_SM(DTv, Wv, 32); break; \
  }
  if (vec) {
    SG_SM_TEAMS(SG_F32, 4)
  } else if (dtype == SG_F32) {
    SG_SM_TEAMS(SG_F32, 1)
  } else {
    SG_SM_TEAMS(SG_BF16, 1)
  }
#undef SG_SM_TEAMS
#undef SG_SM
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "segment_max launch: %s", cudaGetErrorString(e));
  sg::count_launch(1);
  return SG_OK;
}

int sg_segment_max_bwd(int dtype, const void* g, int64_t ldg, const int64_t* argmax, int64_t lda,
                       int64_t n_rows, void* gx, int64_t ldx, int64_t F, void* stream) {
  if (n_rows == 0 || F == 0) return SG_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int grid = grid_for(n_rows * F, 256);
  if (dtype == SG_F32)
    segmax_bwd_kernel<SG_F32><<<grid, 256, 0, st>>>(g, ldg, argmax, lda, n_rows, gx, ldx, (int)F);
  else
    segmax_bwd_kernel<SG_BF16><<<grid, 256, 0, st>>>(g, ldg, argmax, lda, n_rows, gx, ldx, (int)F);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "segment_max_bwd launch: %s", cudaGetErrorString(e));
  sg::count_launch(1);
  return SG_OK;
}

int64_t sg_sort_workspace_bytes(int64_t n, int64_t n_seg) {
  return 3 * align_up(4 * std::max<int64_t>(n, 1), 256) + align_up((int64_t)cub_temp_bytes(n, n_seg), 256) + 256;
}

int sg_segment_sort(const int64_t* seg, int64_t n, int64_t n_seg, int64_t* ptr, int32_t* perm,
                    int32_t* err_flag, void* workspace, int64_t workspace_bytes, void* stream) {
  SG_REQUIRE(n >= 0 && n <= INT32_MAX && n_seg >= 0 && n_seg <= INT32_MAX, SG_EINVAL,
             "segment_sort: sizes exceed int32");
  SG_REQUIRE(workspace_bytes >= sg_sort_workspace_bytes(n, n_seg), SG_EBUDGET,
             "segment_sort workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = (char*)workspace;
  const int64_t a = align_up(4 * std::max<int64_t>(n, 1), 256);
  int32_t* keys_in = (int32_t*)ws;
  int32_t* keys_out = (int32_t*)(ws + a);
  int32_t* vals_in = (int32_t*)(ws + 2 * a);
  void* temp = ws + 3 * a;
  size_t temp_bytes = cub_temp_bytes(n, n_seg);
  if (n > 0) {
    seg_keys_kernel<<<grid_for(n, 256), 256, 0, st>>>(seg, n, n_seg, keys_in, vals_in, err_flag);
    cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in,
                                                    perm, (int)n, 0, end_bit_for(n_seg), st);
    if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "radix sort: %s", cudaGetErrorString(e));
  }
  seg_ptr_kernel<<<grid_for(n_seg + 1, 256), 256, 0, st>>>(keys_out, n, n_seg, ptr);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "segment_sort: %s", cudaGetErrorString(e));
  sg::count_launch(2);
  return SG_OK;
}

}  // extern "C"
