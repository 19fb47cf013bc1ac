// Fused Scatter-ApplyEdge-Gather propagation kernels for sm_100a (K1-K7).
//
// One persistent-warp kernel template covers every SAGA-NN propagation pass on
// the hot path: GCN forward over CSC, GCN backward dual
// over the transposed (CSR) index with a fused ReLU-mask epilogue, passthrough
// segment_sum, and the three G-GCN gated passes.  Edge tensors never touch HBM:
// each warp walks the edges of its rows, loads source-feature rows with 128-bit
// loads (feature dimension across lanes -> coalesced), evaluates the ApplyEdge
// function in registers and accumulates in fp32 registers.
//
// Determinism / parity: per destination row the edge terms are added one by one
// in CSC (or CSR) order with IEEE round-to-nearest mul/add (this file is built
// with -fmad=false and uses explicit __f*_rn intrinsics), which is exactly the
// sequential np.add.at of segment_sum (tensor.py:445) and take_rows' backward
// (tensor.py:433).  Rows with more than T edges are split into consecutive
// subgroups: each subgroup's partial is summed from
// 0 into a workspace slot, and the last subgroup to finish (atomic ticket)
// combines the partials in subgroup order -- a fixed order, so results are
// identical run to run and to oracle/saga.py:seq_sum_rows.  No float atomics.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include "common.h"
#include "vecio.cuh"

namespace {
using sg::VecIO;

constexpr int kWarpsPerBlock = 8;
// Split rows (> T edges): the pass kernel only writes each subgroup's partial, and a second
// launch folds every split row's partials in subgroup order, one warp per (row, 32-vector column
// slice) with up to 16 partials' loads in flight (1, default); or the warp that finishes a row's
// last subgroup folds all of them, one partial per memory round trip, inside the pass (0).  At
// 8-way sharding the Reddit hub row has 800 subgroups (T = 1024): the in-pass fold kept one warp
// busy ~0.4 ms after the rest of the pass had drained (tools/dist_proxy.py, rank 0).
#ifndef SG_SPLIT_KERNEL
#define SG_SPLIT_KERNEL 1
#endif
// shared memory given to the hub-row cache (SG_HUB_KB overrides; the rest of the 256 KB
// L1/shared array stays L1 for the in-flight row loads)
// rows of >= 4 vectors per lane (F > 384 fp32): the cache measured slower on 1-vector
// rows (F = 128: 3.6 -> 5.0 ms, the hub branch breaks the 8-deep load batching)
constexpr int kHubMinVpl = 4;

int64_t hub_smem_bytes() {
  static int64_t v = -1;
  if (v < 0) {
    const char* e = getenv("SG_HUB_KB");
    v = (e ? atoll(e) : 64) * 1024;
  }
  return v;
}

// ------------------------------------------------------------------ modes
template <int MODE>
struct ModeT;

template <>
struct ModeT<SG_PROP_PASS> {
  static constexpr int NG = 1, NR = 0, NOUT = 1, GATE_ROW = -1;
  static constexpr bool USE_W = false;
  static __device__ __forceinline__ void term(const float* g0, const float*, const float*,
                                              const float*, float, float* t0, float*) {
    t0[0] = g0[0];
  }
};

template <>
struct ModeT<SG_PROP_GCN> {
  static constexpr int NG = 1, NR = 0, NOUT = 1, GATE_ROW = -1;
  static constexpr bool USE_W = true;
  // mul(take_rows(H, src), w): x * w (tensor.py:249); mul bwd g * w (tensor.py:263)
  static __device__ __forceinline__ void term(const float* g0, const float*, const float*,
                                              const float*, float w, float* t0, float*) {
    t0[0] = __fmul_rn(g0[0], w);
  }
};

using sg::add2_rn;

// Gate sigmoid.  The reference computes 1.0 / (1.0 + np.exp(-x)) (tensor.py:205); device exp
// is not bit-comparable with numpy's anyway, so the gate uses the SFU: eta = rcp(1 + 2^t)
// with t = -log2(e) * (P + Q) formed by ONE fma from the pre-scaled row operand
// (rs = -log2(e) * Q, scaled once per row in load_row_state).  ex2.approx / rcp.approx are
// within 2 ulp; 2^t -> inf gives eta = 0 and 2^t -> 0 gives 1 with no special-case path
// (the IEEE __frcp_rn's slow path cost 2x on saturated gates).
constexpr float kNegLog2e = -1.4426950408889634f;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// sigmoid(p + q) given p and qs = -log2(e) * q
__device__ __forceinline__ float gate(float p, float qs) {
  return rcp_approx(__fadd_rn(1.0f, ex2_approx(__fmaf_rn(p, kNegLog2e, qs))));
}

template <>
struct ModeT<SG_PROP_GGCN_FWD> {
  static constexpr int NG = 2, NR = 1, NOUT = 1, GATE_ROW = 0;
  static constexpr bool USE_W = false;
  // G = [h | P] row of v, R = Q row of u: eta = sigmoid(P[v] + Q[u]); t = eta * h[v]
  static __device__ __forceinline__ void term(const float* g0, const float* g1, const float* r0,
                                              const float*, float, float* t0, float*) {
    float eta = gate(g1[0], r0[0]);
    t0[0] = __fmul_rn(eta, g0[0]);
  }
};

template <>
struct ModeT<SG_PROP_GGCN_FWD_S> {
  static constexpr int NG = 2, NR = 1, NOUT = 2, GATE_ROW = 0;
  static constexpr bool USE_W = false;
  // the forward term plus S_e = (h[v] * eta) * (1 - eta): the destination-independent factor
  // of the backward dQ term ((dA[u] * h[v]) * eta) * (1 - eta), summed per destination now so
  // the backward needs no second CSC pass (dQ = dA (.) S)
  static __device__ __forceinline__ void term(const float* g0, const float* g1, const float* r0,
                                              const float*, float, float* t0, float* t1) {
    float eta = gate(g1[0], r0[0]);
    t0[0] = __fmul_rn(eta, g0[0]);
    t1[0] = __fmul_rn(__fmul_rn(g0[0], eta), __fsub_rn(1.0f, eta));
  }
};

template <>
struct ModeT<SG_PROP_GGCN_BWD_DST> {
  static constexpr int NG = 2, NR = 2, NOUT = 1, GATE_ROW = 1;
  static constexpr bool USE_W = false;
  // CSC row u.  G = [h | P] of v, R = [dA | Q] of u.
  // g_eta = dA[u] * h[v] (mul bwd, tensor.py:263); t = (g_eta * eta) * (1 - eta) (tensor.py:232)
  static __device__ __forceinline__ void term(const float* g0, const float* g1, const float* r0,
                                              const float* r1, float, float* t0, float*) {
    float eta = gate(g1[0], r1[0]);
    float ge = __fmul_rn(r0[0], g0[0]);
    t0[0] = __fmul_rn(__fmul_rn(ge, eta), __fsub_rn(1.0f, eta));
  }
};

template <>
struct ModeT<SG_PROP_GGCN_BWD_SRC> {
  static constexpr int NG = 2, NR = 2, NOUT = 2, GATE_ROW = 1;
  static constexpr bool USE_W = false;
  // CSR row v.  G = [dA | Q] of u, R = [h | P] of v (gate operand: the row's P, pre-scaled).
  // dP[v] += (dA[u]*h[v]*eta)*(1-eta);  dH[v] += dA[u] * eta  (g_hs = g * eta)
  static __device__ __forceinline__ void term(const float* g0, const float* g1, const float* r0,
                                              const float* r1, float, float* t0, float* t1) {
    float eta = gate(g1[0], r1[0]);
    float ge = __fmul_rn(g0[0], r0[0]);
    t0[0] = __fmul_rn(__fmul_rn(ge, eta), __fsub_rn(1.0f, eta));
    t1[0] = __fmul_rn(g0[0], eta);
  }
};

struct PropArgs {
  const int64_t* ptr;
  const int32_t* idx;
  const float* w;
  const sg_item* items;
  const sg_split* splits;
  float* partial;       // [NOUT][n_slots][pld] fp32
  int64_t pld, n_slots;
  int32_t* counters;    // [n_splits]
  int32_t n_splits;
  int32_t* queue;       // work-queue ticket
  const void* G;
  int64_t ldg, g_off;
  const void* R;
  int64_t ldr, r_off;
  void* out0;
  int64_t ld0;
  void* out1;
  int64_t ld1;
  const void* mask;
  int64_t ldm;
  int32_t n_items;
  int32_t Fv;        // vectors per row in this column slice
  int32_t Fcols;     // valid columns in this column slice
  int32_t accumulate;
  const int32_t* hub_rows;  // hub-row cache: idx < 0 means slot (idx & 0x7fffffff) in smem
  int32_t n_hub;
  // resident blocks per SM to launch for the wide single-operand kernels (0: all the kernel's
  // occupancy allows): passes without split rows (no hubs) cap at 3, see launch_one
  int32_t wide_blocks_cap;
};

template <int MODE, int DT, int W, int VPL, int LPR, int DEPTH, bool HUB = false>
struct Prop {
  using M = ModeT<MODE>;
  // DT = SG_BF16_F32OUT: bf16 inputs (G, R, mask) and fp32 outputs (out0 / out1)
  static constexpr int IDT = DT == SG_BF16_F32OUT ? SG_BF16 : DT;
  static constexpr int ODT = DT == SG_BF16_F32OUT ? SG_F32 : DT;
  using IO = VecIO<IDT, W>;
  using OIO = VecIO<ODT, W>;
  static constexpr int NG = M::NG, NR = M::NR, NOUT = M::NOUT;

  using Elem = typename IO::Elem;
  using Raw = typename IO::Raw;
  // run-length reuse of multi-edges (see step): single-operand rows of >= 2 vectors per lane.
  // One-vector rows (F <= 128 fp32) keep one load per edge: there the run bookkeeping cost
  // more than the loads it saved (Reddit F = 128 passes 3.6 -> 4.5 ms).
#ifndef SG_RUNS_MIN_VPL
#define SG_RUNS_MIN_VPL 2
#endif
  static constexpr bool kRuns = NG == 1 && VPL >= SG_RUNS_MIN_VPL;

  // Load the lane's slice of DEPTH gathered rows (raw 16-byte vectors in flight), then add
  // their terms in edge order.  FULL: all DEPTH edges valid (no per-edge predicates).
  // `gl` is G advanced to this lane's first column; only the last vector needs a bound check.
  // RUNS: entry d stands for a run of cnt[d] consecutive edges with the same (source, weight)
  // (multi-edges: R-MAT repeats 31% of the Reddit-shaped edges), so one row load serves the
  // whole run and its term is added cnt[d] times -- the same sequence of IEEE adds as one
  // load per edge, i.e. bitwise identical.
  template <bool FULL, bool RUNS>
  static __device__ __forceinline__ void step(const PropArgs& a, const Elem* gl, const Raw* hl,
                                              bool last_ok, const int (&s)[DEPTH],
                                              const float (&wv)[DEPTH], const int (&cnt)[DEPTH], int n,
                                              const float (&rs)[NR > 0 ? NR : 1][VPL][W],
                                              float (&acc)[NOUT][VPL][W]) {
    Raw g[DEPTH][NG][VPL];
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      if (HUB && (FULL || d < n) && s[d] < 0) {
        // hub row: served from this CTA's shared memory (same bits as the HBM row)
        const Raw* hrow = hl + (s[d] & 0x7fffffff) * a.Fv;
#pragma unroll
        for (int v = 0; v < VPL; ++v)
          if (v < VPL - 1 || last_ok) g[d][0][v] = hrow[v * LPR];
      } else if (FULL || d < n) {
        // 32x32->64 IMAD.WIDE row address; column offsets are immediates
        const Elem* row = gl + (uint64_t)(uint32_t)s[d] * (uint32_t)a.ldg;
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          if (v < VPL - 1 || last_ok) {
#pragma unroll
            for (int q = 0; q < NG; ++q)
              g[d][q][v] = IO::ld_raw(row + (q ? a.g_off : 0) + v * LPR * W);
          }
        }
      }
    }
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
      if (FULL || d < n) {
        // a run's terms are recomputed from the raw vectors still in registers (cheaper in
        // registers than keeping the fp32 terms of a whole row live)
        const int reps = RUNS ? cnt[d] : 1;
#pragma unroll 1
        for (int c = 0; c < reps; ++c) {
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            float x0[W], x1[W];
            IO::unpack(g[d][0][v], x0);
            IO::unpack(g[d][NG - 1][v], x1);
            if constexpr (W % 2 == 0) {
#pragma unroll
              for (int k = 0; k < W; k += 2) {
                float t0a, t1a = 0.f, t0b, t1b = 0.f;
                M::term(&x0[k], &x1[k], &rs[0][v][k], &rs[NR > 1 ? 1 : 0][v][k], wv[d], &t0a, &t1a);
                M::term(&x0[k + 1], &x1[k + 1], &rs[0][v][k + 1], &rs[NR > 1 ? 1 : 0][v][k + 1], wv[d],
                        &t0b, &t1b);
                add2_rn(acc[0][v][k], acc[0][v][k + 1], t0a, t0b);
                if (NOUT > 1) add2_rn(acc[NOUT - 1][v][k], acc[NOUT - 1][v][k + 1], t1a, t1b);
              }
            } else {
#pragma unroll
              for (int k = 0; k < W; ++k) {
                float t0, t1 = 0.f;
                M::term(&x0[k], &x1[k], &rs[0][v][k], &rs[NR > 1 ? 1 : 0][v][k], wv[d], &t0, &t1);
                acc[0][v][k] = __fadd_rn(acc[0][v][k], t0);
                if (NOUT > 1) acc[NOUT - 1][v][k] = __fadd_rn(acc[NOUT - 1][v][k], t1);
              }
            }
          }
        }
      }
    }
  }

  // Sequentially accumulate edges [e0, e1) of one row into acc (team-cooperative).
  static __device__ __forceinline__ void run_edges(const PropArgs& a, int64_t e0, int64_t e1,
                                                   const float (&rs)[NR > 0 ? NR : 1][VPL][W],
                                                   float (&acc)[NOUT][VPL][W], unsigned tmask,
                                                   int tl, const Raw* hs) {
    const Elem* gl = static_cast<const Elem*>(a.G) + tl * W;
    const Raw* hl = hs + tl;
    const bool last_ok = (VPL - 1) * LPR + tl < a.Fv;
    if constexpr (LPR == 32) {
      // warp-wide index window: 32 (src, w) pairs loaded coalesced, run-length encoded by
      // ballot (a lane heads a run unless it repeats the previous lane's (src, w)), the run
      // heads broadcast by shuffle DEPTH at a time; the next window is prefetched while this
      // one is consumed.  A run split by a window boundary is just two runs.
      int n_next = (int)min((int64_t)32, e1 - e0);
      int src_next = 0;
      float w_next = 0.f;
      if (tl < n_next) {
        src_next = __ldcs(a.idx + e0 + tl);
        if (M::USE_W) w_next = __ldcs(a.w + e0 + tl);
      }
      #pragma unroll 1
      for (int64_t eb = e0; eb < e1; eb += 32) {
        const int n = n_next;
        const int my_src = src_next;
        const float my_w = w_next;
        n_next = (int)min((int64_t)32, e1 - (eb + 32));
        if (tl < n_next) {
          src_next = __ldcs(a.idx + eb + 32 + tl);
          if (M::USE_W) w_next = __ldcs(a.w + eb + 32 + tl);
        }
        if constexpr (kRuns) {
          const int prev_src = __shfl_up_sync(0xffffffffu, my_src, 1);
          const float prev_w = __shfl_up_sync(0xffffffffu, my_w, 1);
          const bool head = tl < n && (tl == 0 || prev_src != my_src ||
                                       (M::USE_W && __float_as_int(prev_w) != __float_as_int(my_w)));
          unsigned heads = __ballot_sync(0xffffffffu, head);
          const unsigned later = heads & (0xfffffffeu << tl);  // heads after this lane
          const int my_cnt = (later ? __ffs(later) - 1 : n) - tl;
          int nu = __popc(heads);
          #pragma unroll 1
          for (; nu > 0; nu -= DEPTH) {
            int s[DEPTH], cnt[DEPTH];
            float wv[DEPTH];
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) {
              const int hl_d = heads ? __ffs(heads) - 1 : 0;
              heads &= heads - 1u;
              s[d] = __shfl_sync(0xffffffffu, my_src, hl_d);
              wv[d] = M::USE_W ? __shfl_sync(0xffffffffu, my_w, hl_d) : 0.f;
              cnt[d] = __shfl_sync(0xffffffffu, my_cnt, hl_d);
            }
            if (nu >= DEPTH)
              step<true, true>(a, gl, hl, last_ok, s, wv, cnt, DEPTH, rs, acc);
            else
              step<false, true>(a, gl, hl, last_ok, s, wv, cnt, nu, rs, acc);
          }
        } else {
          int d0 = 0;
          #pragma unroll 1
          for (; d0 + DEPTH <= n; d0 += DEPTH) {
            int s[DEPTH];
            float wv[DEPTH];
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) {
              s[d] = __shfl_sync(0xffffffffu, my_src, d0 + d);
              wv[d] = M::USE_W ? __shfl_sync(0xffffffffu, my_w, d0 + d) : 0.f;
            }
            step<true, false>(a, gl, hl, last_ok, s, wv, s, DEPTH, rs, acc);
          }
          if (d0 < n) {
            int s[DEPTH];
            float wv[DEPTH];
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) {
              s[d] = __shfl_sync(0xffffffffu, my_src, (d0 + d) & 31);
              wv[d] = M::USE_W ? __shfl_sync(0xffffffffu, my_w, (d0 + d) & 31) : 0.f;
            }
            step<false, false>(a, gl, hl, last_ok, s, wv, s, n - d0, rs, acc);
          }
        }
      }
    } else {
      // narrow rows (teams of LPR lanes, one row each): the team loads a window of WIN
      // (src, w) pairs coalesced -- WPL per lane -- and broadcasts them inside the team by
      // width-LPR shuffles; the next window is prefetched while this one is consumed, so
      // the index load latency no longer serialises with the row loads.
      constexpr int WIN = LPR > DEPTH ? LPR : DEPTH;
      constexpr int WPL = WIN / LPR;
      // every window slot is loaded by some team lane (a DEPTH of 6 with 4-lane teams would
      // leave slots 4-5 unloaded), and a multi-slot window is exactly one step
      static_assert(WIN % LPR == 0 && (WPL == 1 || WIN == DEPTH), "DEPTH must be a multiple of LPR");
      int src_next[WPL];
      float w_next[WPL];
      int n_next = (int)min((int64_t)WIN, e1 - e0);
#pragma unroll
      for (int q = 0; q < WPL; ++q) {
        const int k = q * LPR + tl;
        src_next[q] = k < n_next ? __ldcs(a.idx + e0 + k) : 0;
        w_next[q] = (M::USE_W && k < n_next) ? __ldcs(a.w + e0 + k) : 0.f;
      }
      #pragma unroll 1
      for (int64_t eb = e0; eb < e1; eb += WIN) {
        const int n = n_next;
        int my_src[WPL];
        float my_w[WPL];
#pragma unroll
        for (int q = 0; q < WPL; ++q) {
          my_src[q] = src_next[q];
          my_w[q] = w_next[q];
        }
        n_next = (int)min((int64_t)WIN, e1 - (eb + WIN));
#pragma unroll
        for (int q = 0; q < WPL; ++q) {
          const int k = q * LPR + tl;
          if (k < n_next) {
            src_next[q] = __ldcs(a.idx + eb + WIN + k);
            if (M::USE_W) w_next[q] = __ldcs(a.w + eb + WIN + k);
          }
        }
        if constexpr (WPL > 1) {
          // WIN == DEPTH: one step per window, edge d sits in slot d / LPR of lane d % LPR
          int s[DEPTH];
          float wv[DEPTH];
#pragma unroll
          for (int d = 0; d < DEPTH; ++d) {
            s[d] = __shfl_sync(tmask, my_src[d / LPR], d % LPR, LPR);
            wv[d] = M::USE_W ? __shfl_sync(tmask, my_w[d / LPR], d % LPR, LPR) : 0.f;
          }
          if (n == DEPTH)
            step<true, false>(a, gl, hl, last_ok, s, wv, s, DEPTH, rs, acc);
          else
            step<false, false>(a, gl, hl, last_ok, s, wv, s, n, rs, acc);
        } else {
          int d0 = 0;
          #pragma unroll 1
          for (; d0 + DEPTH <= n; d0 += DEPTH) {
            int s[DEPTH];
            float wv[DEPTH];
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) {
              s[d] = __shfl_sync(tmask, my_src[0], d0 + d, LPR);
              wv[d] = M::USE_W ? __shfl_sync(tmask, my_w[0], d0 + d, LPR) : 0.f;
            }
            step<true, false>(a, gl, hl, last_ok, s, wv, s, DEPTH, rs, acc);
          }
          if (d0 < n) {
            int s[DEPTH];
            float wv[DEPTH];
#pragma unroll
            for (int d = 0; d < DEPTH; ++d) {
              s[d] = __shfl_sync(tmask, my_src[0], (d0 + d) & (LPR - 1), LPR);
              wv[d] = M::USE_W ? __shfl_sync(tmask, my_w[0], (d0 + d) & (LPR - 1), LPR) : 0.f;
            }
            step<false, false>(a, gl, hl, last_ok, s, wv, s, n - d0, rs, acc);
          }
        }
      }
    }
  }

  static __device__ __forceinline__ void load_row_state(const PropArgs& a, int64_t r, int tl,
                                                        float (&rs)[NR > 0 ? NR : 1][VPL][W]) {
    if (NR == 0) return;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int cv = v * LPR + tl;
      if (cv < a.Fv) {
#pragma unroll
        for (int q = 0; q < NR; ++q) {
          IO::ld_cs(a.R, r * a.ldr + (q ? a.r_off : 0) + (int64_t)cv * W, rs[q][v]);
          if (q == M::GATE_ROW) {  // gate operand pre-scaled by -log2(e), once per row
#pragma unroll
            for (int k = 0; k < W; ++k) rs[q][v][k] = __fmul_rn(rs[q][v][k], kNegLog2e);
          }
        }
      }
    }
  }

  static __device__ __forceinline__ void init_acc(const PropArgs& a, int64_t r, int tl,
                                                  float (&acc)[NOUT][VPL][W], bool from_out) {
#pragma unroll
    for (int o = 0; o < NOUT; ++o)
#pragma unroll
      for (int v = 0; v < VPL; ++v)
#pragma unroll
        for (int k = 0; k < W; ++k) acc[o][v][k] = 0.f;
    if (!from_out) return;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int cv = v * LPR + tl;
      if (cv < a.Fv) {
        OIO::ld_cs(a.out0, r * a.ld0 + (int64_t)cv * W, acc[0][v]);
        if (NOUT > 1) OIO::ld_cs(a.out1, r * a.ld1 + (int64_t)cv * W, acc[NOUT - 1][v]);
      }
    }
  }

  static __device__ __forceinline__ void store_row(const PropArgs& a, int64_t r, int tl,
                                                   float (&acc)[NOUT][VPL][W]) {
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int cv = v * LPR + tl;
      if (cv < a.Fv) {
        const int nvalid = min(W, a.Fcols - cv * W);
        if (a.mask) {
          float m[W];
          IO::ld_cs(a.mask, r * a.ldm + (int64_t)cv * W, m);
#pragma unroll
          for (int k = 0; k < W; ++k)  // relu bwd: g * (x > 0.0)  (tensor.py:236)
            acc[0][v][k] = __fmul_rn(acc[0][v][k], m[k] > 0.f ? 1.f : 0.f);
        }
        OIO::st(a.out0, r * a.ld0 + (int64_t)cv * W, acc[0][v], nvalid);
        if (NOUT > 1) OIO::st(a.out1, r * a.ld1 + (int64_t)cv * W, acc[NOUT - 1][v], nvalid);
      }
    }
  }
};

// Resident blocks per SM to ask ptxas for: in-flight raw vectors (4 regs each) plus
// fp32 accumulators and row state decide the register budget (64 / 80 / 128 regs).
#ifndef SG_VPL1_BLOCKS
#define SG_VPL1_BLOCKS 2
#endif
// wide single-operand rows: 4 blocks/SM (64 registers, 56 B of spill) measured 4-5% faster than
// 3 (80 registers) on the Reddit layer-1 pass (11.99 -> 11.32-11.52 ms; 5 blocks: 19.2 ms, and
// 4 blocks without the in-register run detection: 13.8 ms; profiles/r02_occupancy_ab.txt)
#ifndef SG_WIDE_BLOCKS
#define SG_WIDE_BLOCKS 4
#endif
// bf16 rows of 3-4 vectors per lane at 3 blocks/SM (80 registers, 92 B of spill): Reddit bf16
// layer-1 pass 11.57 -> 10.51 ms (2 blocks with 4 rows in flight: 10.88; profiles/r02_occupancy_ab.txt)
#ifndef SG_BF16_WIDE_BLOCKS
#define SG_BF16_WIDE_BLOCKS 3
#endif
// bf16 rows of 65-128 columns (8-byte vectors, one per lane): 4 blocks/SM with 4 rows in flight
// (64 registers) instead of 2 blocks x 12: Reddit bf16 F = 128 passes 4.32 / 4.45 -> 3.34 / 3.44 ms
// (the fp32 one-vector rows measured the same at 2 x 8, 3 x 4 and 4 x 3; profiles/r02_occupancy_ab.txt)
#ifndef SG_BF16_HALF_BLOCKS
#define SG_BF16_HALF_BLOCKS 4
#endif
#ifndef SG_BF16_HALF_DEPTH
#define SG_BF16_HALF_DEPTH 4
#endif
template <int MODE, int DT, int W, int VPL, int DEPTH>
constexpr int prop_min_blocks() {
  if (DT != SG_F32 && W == 4 && VPL == 1 && ModeT<MODE>::NG == 1 && SG_BF16_HALF_BLOCKS > 0)
    return SG_BF16_HALF_BLOCKS;
  if (VPL == 1 && ModeT<MODE>::NG == 1 && SG_VPL1_BLOCKS != 2) return SG_VPL1_BLOCKS;
  // wide single-operand rows: one row in flight per warp at SG_WIDE_BLOCKS blocks/SM beat two
  // rows at 2 blocks/SM (F = 602 CSC pass 14.2-14.5 -> 13.1 ms at 3 blocks)
  if (VPL >= 5 && ModeT<MODE>::NG == 1 && SG_WIDE_BLOCKS > 0) return SG_WIDE_BLOCKS;
  // bf16 rows of 3-4 vectors per lane (8 bf16 per 16-B vector: F = 602 bf16 is 76 vectors)
  if (W == 8 && VPL >= 3 && ModeT<MODE>::NG == 1 && SG_BF16_WIDE_BLOCKS > 0) return SG_BF16_WIDE_BLOCKS;
  // per in-flight edge: raw vectors + 64-bit row pointer + shuffled (src, w)
  constexpr int regs = DEPTH * (ModeT<MODE>::NG * VPL * 4 + 4) +
                       (ModeT<MODE>::NOUT + ModeT<MODE>::NR) * VPL * W + 40;
  return regs <= 80 ? 3 : 2;
}

// HUB: the block first copies the pass's hub rows (most-referenced source rows, listed in
// a.hub_rows; their edges carry idx = slot | 0x80000000) into shared memory, so those
// gathers are served on-chip instead of through L2.  One block of NWB warps per SM.
template <int MODE, int DT, int W, int VPL, int LPR, int DEPTH, bool HUB = false, int NWB = kWarpsPerBlock>
__global__ void __launch_bounds__(NWB * 32, (HUB ? 1 : prop_min_blocks<MODE, DT, W, VPL, DEPTH>()))
    prop_kernel(const PropArgs a) {
  using K = Prop<MODE, DT, W, VPL, LPR, DEPTH, HUB>;
  using Raw = typename K::Raw;
  extern __shared__ __align__(16) unsigned char prop_smem[];
  const Raw* hs = reinterpret_cast<const Raw*>(prop_smem);
  if constexpr (HUB) {
    Raw* hw = reinterpret_cast<Raw*>(prop_smem);
    const int total = a.n_hub * a.Fv;
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
      const int r = i / a.Fv, c = i - r * a.Fv;
      hw[i] = K::IO::ld_raw(static_cast<const typename K::Elem*>(a.G) +
                            (int64_t)__ldg(a.hub_rows + r) * a.ldg + (int64_t)c * W);
    }
    __syncthreads();
  }
  constexpr int NOUT = K::NOUT;
  constexpr int NRr = K::NR > 0 ? K::NR : 1;
  constexpr int NT = 32 / LPR;
  const int lane = threadIdx.x & 31;
  const int team = lane / LPR, tl = lane % LPR;
  const unsigned tmask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (team * LPR));

  // Work distribution: every warp takes the next item from the global queue.  Split subgroups
  // are queued by first source (sg_host_plan_order), so the items in flight at any moment --
  // on all SMs -- gather overlapping source ranges and share them in L2 (Reddit L0: DRAM
  // 49 -> 38 GB, 12.8 -> 11.5 ms; a CTA-chunked queue that kept adjacent items on one SM to
  // share L1 measured slower, profiles/r02_sched_ab.txt).
  for (;;) {
    int it = 0;
    if (lane == 0) it = atomicAdd(a.queue, 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= a.n_items) break;
    const sg_item item = a.items[it];
    const bool split = item.split >= 0;
    // One inlined copy of the edge loop serves whole rows and split subgroups alike
    // (a single call site keeps ptxas register allocation spill-free).
    const int r_end = (split && team != 0) ? item.row_begin : item.row_end;
    // row extents are loaded one row ahead, so a short row's pointer load does not
    // serialise with its index and feature loads (low-degree graphs: ~4 edges per row)
    int64_t n0 = 0, n1 = 0;
    if (item.row_begin + team < r_end) {
      n0 = split ? item.e_begin : __ldg(a.ptr + item.row_begin + team);
      n1 = split ? item.e_end : __ldg(a.ptr + item.row_begin + team + 1);
    }
#pragma unroll 1
    for (int r = item.row_begin + team; r < r_end; r += NT) {
      float rs[NRr][VPL][W];
      float acc[NOUT][VPL][W];
      const int64_t e0 = n0, e1 = n1;
      if (!split && r + NT < r_end) {
        n0 = __ldg(a.ptr + r + NT);
        n1 = __ldg(a.ptr + r + NT + 1);
      }
      K::load_row_state(a, r, tl, rs);
      K::init_acc(a, r, tl, acc, a.accumulate != 0 && !split);
      K::run_edges(a, e0, e1, rs, acc, tmask, tl, hs);
      if (!split) {
        K::store_row(a, r, tl, acc);
      } else {
        const int64_t slot = a.splits[item.split].slot0 + item.sub;
#pragma unroll
        for (int o = 0; o < NOUT; ++o)
#pragma unroll
          for (int v = 0; v < VPL; ++v) {
            const int cv = v * LPR + tl;
            if (cv < a.Fv) {
              float* p = a.partial + ((int64_t)o * a.n_slots + slot) * a.pld + (int64_t)cv * W;
#pragma unroll
              for (int k = 0; k < W; ++k) __stcg(p + k, acc[o][v][k]);
            }
          }
      }
    }
#if !SG_SPLIT_KERNEL
    if (split) {
      const sg_split sp = a.splits[item.split];
      const int64_t r = item.row_begin;
      __threadfence();
      __syncwarp();
      int ticket = 0;
      if (lane == 0) ticket = atomicAdd(a.counters + item.split, 1);
      ticket = __shfl_sync(0xffffffffu, ticket, 0);
      if (ticket == sp.n_sub - 1) {
        __threadfence();
        if (team == 0) {
          float acc[NOUT][VPL][W];
          K::init_acc(a, r, tl, acc, a.accumulate != 0);
          #pragma unroll 1
          for (int s = 0; s < sp.n_sub; ++s) {
#pragma unroll
            for (int o = 0; o < NOUT; ++o)
#pragma unroll
              for (int v = 0; v < VPL; ++v) {
                const int cv = v * LPR + tl;
                if (cv < a.Fv) {
                  const float* p =
                      a.partial + ((int64_t)o * a.n_slots + sp.slot0 + s) * a.pld + (int64_t)cv * W;
#pragma unroll
                  for (int k = 0; k < W; ++k) acc[o][v][k] = __fadd_rn(acc[o][v][k], __ldcg(p + k));
                }
              }
          }
          K::store_row(a, r, tl, acc);
        }
        if (lane == 0) a.counters[item.split] = 0;
      }
    }
#endif
  }
}

// Fold of the split rows' subgroup partials (SG_SPLIT_KERNEL): warp w takes split w / ncs,
// column slice w % ncs (32 vectors of W columns, one per lane); acc = init (0, or the output row
// when accumulating a chunk chain), then acc += p_0, p_1, ... in subgroup order with U partials'
// loads in flight (U = 16 fp32 vectors) -- the same IEEE adds in the same order as the in-pass fold -- then the
// row epilogue (ReLU mask) and store.
template <int MODE, int DT, int W>
__global__ void __launch_bounds__(kWarpsPerBlock * 32) combine_kernel(const PropArgs a0, int ncs) {
  using K = Prop<MODE, DT, W, 1, 32, 1>;
  constexpr int NOUT = K::NOUT;
  // partials in flight per lane: ~SG_COMBINE_REGS registers of loads
#ifndef SG_COMBINE_REGS
#define SG_COMBINE_REGS 64
#endif
  constexpr int U0 = SG_COMBINE_REGS / (NOUT * W);
  constexpr int U = U0 > 16 ? 16 : (U0 < 2 ? 2 : U0);
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= (int64_t)a0.n_splits * ncs) return;
  const sg_split sp = a0.splits[warp / ncs];
  const int c0 = (int)(warp % ncs) * 32;  // first vector of this column slice
  PropArgs a = a0;
  using IE = typename K::IO::Elem;
  using OE = typename K::OIO::Elem;
  a.Fv = min(32, a0.Fv - c0);
  a.Fcols = a0.Fcols - c0 * W;
  a.out0 = static_cast<OE*>(a0.out0) + (int64_t)c0 * W;
  if (a0.out1) a.out1 = static_cast<OE*>(a0.out1) + (int64_t)c0 * W;
  if (a0.mask) a.mask = static_cast<const IE*>(a0.mask) + (int64_t)c0 * W;
  float acc[NOUT][1][W];
  K::init_acc(a, sp.row, lane, acc, a.accumulate != 0);
  if (lane < a.Fv) {
    const float* pb = a0.partial + sp.slot0 * a0.pld + (int64_t)(c0 + lane) * W;
    const int64_t ostride = a0.n_slots * a0.pld;
    #pragma unroll 1
    for (int s = 0; s < sp.n_sub; s += U) {
      float x[U][NOUT][W];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (s + u < sp.n_sub) {
#pragma unroll
          for (int o = 0; o < NOUT; ++o)
#pragma unroll
            for (int k = 0; k < W; ++k) x[u][o][k] = __ldcg(pb + o * ostride + (int64_t)(s + u) * a0.pld + k);
        }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (s + u < sp.n_sub) {
#pragma unroll
          for (int o = 0; o < NOUT; ++o)
#pragma unroll
            for (int k = 0; k < W; ++k) acc[o][0][k] = __fadd_rn(acc[o][0][k], x[u][o][k]);
        }
    }
  }
  K::store_row(a, sp.row, lane, acc);
}

template <int MODE, int DT, int W>
cudaError_t launch_combine(const PropArgs& a, cudaStream_t st) {
#if SG_SPLIT_KERNEL
  if (a.n_splits <= 0) return cudaSuccess;
  const int ncs = (a.Fv + 31) / 32;
  const int64_t warps = (int64_t)a.n_splits * ncs;
  const int64_t blocks = (warps + kWarpsPerBlock - 1) / kWarpsPerBlock;
  combine_kernel<MODE, DT, W><<<(unsigned)blocks, kWarpsPerBlock * 32, 0, st>>>(a, ncs);
  sg::count_launch();
  return cudaGetLastError();
#else
  (void)a; (void)st;
  return cudaSuccess;
#endif
}

// ------------------------------------------------------------------ dispatch
struct LaunchCfg {
  int W, VPL, LPR;
};

int mode_nout(int mode) { return (mode == SG_PROP_GGCN_BWD_SRC || mode == SG_PROP_GGCN_FWD_S) ? 2 : 1; }
int mode_ng(int mode) { return mode >= SG_PROP_GGCN_FWD ? 2 : 1; }

int g_sm_count = 0;

int sm_count() {
  if (!g_sm_count) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (g_sm_count <= 0) g_sm_count = 148;
  }
  return g_sm_count;
}

// hub-cache kernel: one block per SM holding the hub rows
template <int MODE, int DT, int W, int VPL, int LPR, int DEPTH, int NWB>
cudaError_t launch_hub(const PropArgs& a, cudaStream_t st) {
  auto hk = prop_kernel<MODE, DT, W, VPL, LPR, DEPTH, true, NWB>;
  const size_t smem = (size_t)a.n_hub * a.Fv * 16;
  static int hub_cfg = 0;
  if (!hub_cfg) {
    cudaFuncSetAttribute(hk, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    hub_cfg = 1;
  }
  int64_t want = ((int64_t)a.n_items + NWB - 1) / NWB;
  int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, sm_count()));
  hk<<<grid, NWB * 32, smem, st>>>(a);
  sg::count_launch();
  return cudaGetLastError();
}

template <int MODE, int DT, int W, int VPL, int LPR>
cudaError_t launch_one(const PropArgs& a, cudaStream_t st) {
  constexpr int NG = ModeT<MODE>::NG;
  // rows in flight per warp: ~8 vectors per lane (DEPTH 3 at VPL 5 spills and runs 50% slower)
#ifndef SG_DEPTH1
#define SG_DEPTH1 8
#endif
#ifndef SG_DEPTH_WIDE
#define SG_DEPTH_WIDE 1
#endif
#ifndef SG_DEPTH_MID
#define SG_DEPTH_MID 8
#endif
  // single-operand rows of 2-4 vectors per lane: ~4 vectors per lane in flight measured faster
  // than ~8 (F = 384: 9.1 -> 7.8-8.0 ms per Reddit pass); two-operand rows (G-GCN) keep ~8
#ifndef SG_DEPTH_MID1
#define SG_DEPTH_MID1 4
#endif
  // bf16 rows carry half the bytes per column: single-operand bf16 rows of 2-4 vectors per lane
  // keep ~6 vectors per lane in flight (F = 602 bf16: 2 rows of 3 vectors, the bytes of one fp32
  // row), and 8-byte bf16 vectors (W = 4, rows of 65-128 columns) keep 12 rows in flight (16 spill)
#ifndef SG_DEPTH_MID1_BF16
#define SG_DEPTH_MID1_BF16 6
#endif
  constexpr int MID1 = DT != SG_F32 ? SG_DEPTH_MID1_BF16 : SG_DEPTH_MID1;
  constexpr int DEPTH_MID = NG == 1 ? (MID1 / VPL > 0 ? MID1 / VPL : 1)
                                    : SG_DEPTH_MID / (VPL * NG);
#ifndef SG_DEPTH1_WARP
#define SG_DEPTH1_WARP SG_DEPTH1
#endif
  // one-vector rows: SG_DEPTH1 rows in flight per lane team; SG_DEPTH1_WARP for warp-wide rows
  constexpr int D1 = LPR == 32 ? SG_DEPTH1_WARP : SG_DEPTH1;
  constexpr int DEPTH1 = (DT != SG_F32 && W == 4 && NG == 1) ? SG_BF16_HALF_DEPTH : D1;
  constexpr int DEPTH = (VPL * NG) == 1 ? DEPTH1
                                        : ((VPL * NG) <= 4 ? DEPTH_MID : (NG > 1 ? 1 : SG_DEPTH_WIDE));
  if constexpr (LPR == 32 && NG == 1 && W > 1 && VPL >= kHubMinVpl) {
    if (a.n_hub > 0) {
      // hub-cache kernel: one block per SM holding the hub rows, as many warps as the
      // register budget allowed the default kernel (2-3 blocks of 8 warps)
      constexpr int NWB = kWarpsPerBlock * prop_min_blocks<MODE, DT, W, VPL, DEPTH>();
      const cudaError_t e = launch_hub<MODE, DT, W, VPL, LPR, DEPTH, NWB>(a, st);
      return e != cudaSuccess ? e : launch_combine<MODE, DT, W>(a, st);
    }
  }
  auto kern = prop_kernel<MODE, DT, W, VPL, LPR, DEPTH>;
  static int blocks_per_sm = 0;
  if (!blocks_per_sm) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, kern, kWarpsPerBlock * 32, 0);
    if (blocks_per_sm <= 0) blocks_per_sm = 1;
  }
  int64_t want = ((int64_t)a.n_items + kWarpsPerBlock - 1) / kWarpsPerBlock;
  int64_t cap = (int64_t)blocks_per_sm * sm_count();
  // Wide rows: 4 blocks/SM pays on hub-heavy passes (R-MAT Reddit L0 11.5 -> 11.0 ms), but on a
  // pass without heavy rows (uniform graph, avg degree 490 < T) the 32 warps/SM sweep a wider
  // window of the source-sorted rows than L2 holds (DRAM 42 -> 127 GB, 16.2 -> 23.9 ms), so
  // such passes launch 3 blocks/SM of the same kernel
  if (VPL >= 5 && NG == 1 && a.wide_blocks_cap > 0)
    cap = std::min<int64_t>(cap, (int64_t)std::min(blocks_per_sm, (int)a.wide_blocks_cap) * sm_count());
  int grid = (int)std::max<int64_t>(1, std::min(want, cap));
  kern<<<grid, kWarpsPerBlock * 32, 0, st>>>(a);
  sg::count_launch();
  const cudaError_t e = cudaGetLastError();
  return e != cudaSuccess ? e : launch_combine<MODE, DT, W>(a, st);
}

// Widest vectors-per-lane instantiated: register pressure grows as VPL * W * (NG + NOUT);
// wider rows are processed in column slices.
// widest single-slice row for the one-operand modes: VPL 6-8 spill at 128 registers, so
// rows wider than 5 vectors per lane (F > 640 fp32) run as several column slices
// (F = 768 / 1024 / 1100: 21.3 / 32.4 / 37.8 ms at VPL 8 -> 18.0 / 24.7 / 29.1 ms at VPL 5 on
// the Reddit graph; VPL 4 and 6 in between, profiles/r01_narrow_ab.txt)
#ifndef SG_VPL_MAX
#define SG_VPL_MAX 5
#endif
constexpr int vpl_max(int mode, int dt) {
  return (dt == SG_F32 && (mode == SG_PROP_PASS || mode == SG_PROP_GCN)) ? SG_VPL_MAX : 4;
}

template <int MODE, int DT, int W>
cudaError_t dispatch_vpl(const PropArgs& a, int LPR, int VPL, cudaStream_t st) {
  constexpr int VMAX = vpl_max(MODE, DT);
  if (LPR < 32) {
    if (VPL == 2) return launch_one<MODE, DT, W, 2, 16>(a, st);  // two rows per warp
    switch (LPR) {
      case 2: return launch_one<MODE, DT, W, 1, 2>(a, st);
      case 4: return launch_one<MODE, DT, W, 1, 4>(a, st);
      case 8: return launch_one<MODE, DT, W, 1, 8>(a, st);
      default: return launch_one<MODE, DT, W, 1, 16>(a, st);
    }
  }
  switch (VPL) {
    case 1: return launch_one<MODE, DT, W, 1, 32>(a, st);
    case 2: return launch_one<MODE, DT, W, 2, 32>(a, st);
    case 3: return launch_one<MODE, DT, W, 3, 32>(a, st);
    case 4: return launch_one<MODE, DT, W, 4, 32>(a, st);
    case 5: return launch_one<MODE, DT, W, (VMAX >= 5 ? 5 : 4), 32>(a, st);
    case 6: return launch_one<MODE, DT, W, (VMAX >= 6 ? 6 : 4), 32>(a, st);
    case 7: return launch_one<MODE, DT, W, (VMAX >= 7 ? 7 : 4), 32>(a, st);
    default: return launch_one<MODE, DT, W, (VMAX >= 8 ? 8 : 4), 32>(a, st);
  }
}

template <int MODE>
cudaError_t dispatch_mode(int dtype, bool vec, bool half_vec, const PropArgs& a, int LPR, int VPL,
                          cudaStream_t st) {
#ifdef SG_TUNE_GCN_ONLY  // fast register/spill iteration: build only the fp32 GCN kernels
  if (MODE != SG_PROP_GCN || dtype != SG_F32 || !vec) return cudaErrorNotSupported;
  return dispatch_vpl<SG_PROP_GCN, SG_F32, 4>(a, LPR, VPL, st);
#endif
  if (dtype == SG_F32)
    return vec ? dispatch_vpl<MODE, SG_F32, 4>(a, LPR, VPL, st)
               : dispatch_vpl<MODE, SG_F32, 1>(a, LPR, VPL, st);
  if (dtype == SG_BF16_F32OUT) {
    // bf16 rows in, fp32 out: the GCN / passthrough gathers of the bf16-storage model
    if constexpr (MODE == SG_PROP_PASS || MODE == SG_PROP_GCN) {
      if (vec && half_vec) return launch_one<MODE, SG_BF16_F32OUT, 4, 1, 32>(a, st);
      return vec ? dispatch_vpl<MODE, SG_BF16_F32OUT, 8>(a, LPR, VPL, st)
                 : dispatch_vpl<MODE, SG_BF16_F32OUT, 1>(a, LPR, VPL, st);
    }
    return cudaErrorNotSupported;
  }
  if (vec && half_vec) return launch_one<MODE, SG_BF16, 4, 1, 32>(a, st);  // bf16 rows 65-128 cols
  return vec ? dispatch_vpl<MODE, SG_BF16, 8>(a, LPR, VPL, st)
             : dispatch_vpl<MODE, SG_BF16, 1>(a, LPR, VPL, st);
}

inline bool aligned(const void* p, int bytes) { return p == nullptr || ((uintptr_t)p % bytes) == 0; }

inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

}  // namespace

extern "C" {

int sg_device_sm_count(int device, int* out) {
  cudaError_t e = cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "cudaDeviceGetAttribute: %s", cudaGetErrorString(e));
  return SG_OK;
}

int64_t sg_propagate_workspace_bytes(int64_t n_items, int64_t n_splits, int64_t n_slots, int64_t F,
                                     int mode) {
  (void)n_items;
  return 256 + align_up(4 * std::max<int64_t>(n_splits, 1), 256) +
         (int64_t)mode_nout(mode) * n_slots * align_up(std::max<int64_t>(F, 1), 8) * 4;
}

int sg_propagate(int mode, int dtype, const int64_t* ptr, const int32_t* idx, const float* w,
                 int64_t n_rows, const sg_item* items, int64_t n_items, const sg_split* splits,
                 int64_t n_splits, int64_t n_slots, const void* G, int64_t ldg, int64_t g_off,
                 const void* R, int64_t ldr, int64_t r_off, void* out0, int64_t ld0, void* out1,
                 int64_t ld1, const void* mask, int64_t ldm, int64_t F, int accumulate,
                 void* workspace, int64_t workspace_bytes, void* stream) {
  return sg_propagate_hub(mode, dtype, ptr, idx, w, n_rows, items, n_items, splits, n_splits, n_slots,
                          G, ldg, g_off, R, ldr, r_off, out0, ld0, out1, ld1, mask, ldm, F, accumulate,
                          nullptr, 0, workspace, workspace_bytes, stream);
}

int64_t sg_propagate_hub_capacity(int64_t F, int dtype) {
  if (dtype != SG_F32 && dtype != SG_BF16) return 0;  // (no hub cache for SG_BF16_F32OUT)
  const int VW = dtype == SG_F32 ? 4 : 8;
  const int64_t max_cols = (int64_t)32 * vpl_max(SG_PROP_GCN, dtype) * VW;
  const int64_t slice_cols = std::min<int64_t>(F, max_cols);
  const int64_t row_bytes = (slice_cols + VW - 1) / VW * 16;
  // every column slice must be wide enough for the hub kernel (the index is encoded)
  const int64_t last_cols = F % max_cols == 0 ? std::min(F, max_cols) : F % max_cols;
  if (last_cols <= (int64_t)32 * (kHubMinVpl - 1) * VW) return 0;
  return std::min<int64_t>(hub_smem_bytes() / row_bytes, INT32_MAX);
}

int sg_propagate_hub(int mode, int dtype, const int64_t* ptr, const int32_t* idx, const float* w,
                     int64_t n_rows, const sg_item* items, int64_t n_items, const sg_split* splits,
                     int64_t n_splits, int64_t n_slots, const void* G, int64_t ldg, int64_t g_off,
                     const void* R, int64_t ldr, int64_t r_off, void* out0, int64_t ld0, void* out1,
                     int64_t ld1, const void* mask, int64_t ldm, int64_t F, int accumulate,
                     const int32_t* hub_rows, int64_t n_hub, void* workspace, int64_t workspace_bytes,
                     void* stream) {
  SG_REQUIRE(mode >= SG_PROP_PASS && mode <= SG_PROP_GGCN_FWD_S, SG_EINVAL, "bad mode %d", mode);
  SG_REQUIRE(dtype == SG_F32 || dtype == SG_BF16 || dtype == SG_BF16_F32OUT, SG_EINVAL, "bad dtype %d", dtype);
  SG_REQUIRE(dtype != SG_BF16_F32OUT || mode <= SG_PROP_GCN, SG_EINVAL,
             "bf16-in / fp32-out is implemented for the PASS and GCN modes");
  SG_REQUIRE(dtype != SG_BF16_F32OUT || n_hub == 0, SG_EINVAL, "no hub cache for bf16-in / fp32-out");
  SG_REQUIRE(n_items >= 0 && n_items <= INT32_MAX, SG_EINVAL, "bad n_items");
  if (n_rows == 0 || F == 0 || n_items == 0) return SG_OK;
  SG_REQUIRE(ptr && idx && items && G && out0, SG_EINVAL, "null required pointer");
  SG_REQUIRE(mode != SG_PROP_GCN || w, SG_EINVAL, "GCN mode needs edge weights");
  SG_REQUIRE(mode < SG_PROP_GGCN_FWD || R, SG_EINVAL, "gated modes need row-side operand R");
  SG_REQUIRE((mode != SG_PROP_GGCN_BWD_SRC && mode != SG_PROP_GGCN_FWD_S) || out1, SG_EINVAL,
             "mode %d needs out1", mode);
  SG_REQUIRE(n_splits == 0 || splits, SG_EINVAL, "split records missing");
  const int64_t need = sg_propagate_workspace_bytes(n_items, n_splits, n_slots, F, mode);
  SG_REQUIRE(workspace && workspace_bytes >= need, SG_EBUDGET,
             "propagate workspace too small: %lld < %lld bytes", (long long)workspace_bytes,
             (long long)need);
  const int VW = dtype == SG_F32 ? 4 : 8;
  const int esz = dtype == SG_F32 ? 4 : 2;        // input (G, R, mask) element size
  const int oesz = dtype == SG_BF16 ? 2 : 4;      // output (out0, out1) element size
  const int OVW = dtype == SG_BF16_F32OUT ? 4 : VW;  // fp32 outputs: 16-B float4 rows suffice
  bool vec = (ldg % VW == 0) && (g_off % VW == 0) && (ld0 % OVW == 0) && aligned(G, 16) &&
             aligned(out0, 16);
  if (R) vec = vec && (ldr % VW == 0) && (r_off % VW == 0) && aligned(R, 16);
  if (out1) vec = vec && (ld1 % OVW == 0) && aligned(out1, 16);
  if (mask) vec = vec && (ldm % VW == 0) && aligned(mask, 16);
  // split subgroups are half the plan's items or more (R-MAT hubs): see the lane-team note below
  const bool hub_heavy = n_slots * 2 >= n_items;
  // bf16 rows of 65-128 columns on hub-heavy passes: 8-byte vectors (4 bf16), so all 32 lanes
  // of a warp work on a row (Reddit bf16 F = 128 passes 4.32 -> 3.34 ms); elsewhere 16-byte
  // vectors with two rows per warp (uniform graphs, degree >= 32: the 8-byte rows measured up
  // to 15% slower, profiles/r02_sweep_full_table.md)
  const bool half_vec = vec && dtype != SG_F32 && F > 64 && F <= 128 && n_hub == 0 && hub_heavy;
  const int W = vec ? (half_vec ? 4 : VW) : 1;
  cudaStream_t st = static_cast<cudaStream_t>(stream);

  char* ws = static_cast<char*>(workspace);
  int32_t* queue = reinterpret_cast<int32_t*>(ws);
  int32_t* counters = reinterpret_cast<int32_t*>(ws + 256);
  float* partial = reinterpret_cast<float*>(ws + 256 + align_up(4 * std::max<int64_t>(n_splits, 1), 256));
  const int64_t pld = align_up(F, 8);

  // column slices of at most 32 lanes x vpl_max vectors
  const int64_t slice_cols = (int64_t)32 * vpl_max(mode, dtype) * W;
  for (int64_t c0 = 0; c0 < F; c0 += slice_cols) {
    const int64_t cols = std::min(slice_cols, F - c0);
    const int Fv = (int)((cols + W - 1) / W);
    int LPR = 32, VPL = (Fv + 31) / 32;
    // Lane teams (one narrow row per team, 32/LPR rows per warp) pay off when items hold
    // many similar rows (uniform graphs: 2-4x, tools/sweep.py).  When split subgroups are
    // half the plan's items or more (R-MAT hubs: Reddit 56% of edges in rows > T), only
    // team 0 works on split items and heavy packed rows leave teams idle: one warp per row
    // measured 17% faster there (tools/narrow_ab.py), so teams are not used.
    if (Fv <= 16 && !hub_heavy) {
      LPR = 2;
      while (LPR < Fv) LPR *= 2;
      VPL = 1;
    }
    PropArgs a;
    a.ptr = ptr; a.idx = idx; a.w = w; a.items = items; a.splits = splits;
    a.partial = partial + c0; a.pld = pld; a.n_slots = n_slots;
    a.counters = counters; a.queue = queue; a.n_splits = (int32_t)n_splits;
    a.G = static_cast<const char*>(G) + c0 * esz; a.ldg = ldg; a.g_off = g_off;
    a.R = R ? static_cast<const char*>(R) + c0 * esz : nullptr; a.ldr = ldr; a.r_off = r_off;
    a.out0 = static_cast<char*>(out0) + c0 * oesz; a.ld0 = ld0;
    a.out1 = out1 ? static_cast<char*>(out1) + c0 * oesz : nullptr; a.ld1 = ld1;
    a.mask = mask ? static_cast<const char*>(mask) + c0 * esz : nullptr; a.ldm = ldm;
    a.n_items = (int32_t)n_items; a.Fv = Fv; a.Fcols = (int32_t)cols; a.accumulate = accumulate;
    a.hub_rows = hub_rows;
    a.n_hub = 0;
    a.wide_blocks_cap = hub_heavy ? 0 : 3;
    if (n_hub > 0) {
      // an index encoded for hubs must run the hub kernel (negative entries are slots)
      SG_REQUIRE(hub_rows && vec && mode <= SG_PROP_GCN && LPR == 32 && VPL >= kHubMinVpl &&
                     n_hub <= sg_propagate_hub_capacity(F, dtype),
                 SG_EINVAL, "hub cache not applicable (mode %d, F %lld, n_hub %lld)", mode, (long long)F,
                 (long long)n_hub);
      a.n_hub = (int32_t)n_hub;
    }
    cudaError_t e = cudaMemsetAsync(ws, 0, 256 + align_up(4 * std::max<int64_t>(n_splits, 1), 256), st);
    if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "memset: %s", cudaGetErrorString(e));
    switch (mode) {
      case SG_PROP_PASS: e = dispatch_mode<SG_PROP_PASS>(dtype, vec, half_vec, a, LPR, VPL, st); break;
      case SG_PROP_GCN: e = dispatch_mode<SG_PROP_GCN>(dtype, vec, half_vec, a, LPR, VPL, st); break;
      case SG_PROP_GGCN_FWD: e = dispatch_mode<SG_PROP_GGCN_FWD>(dtype, vec, half_vec, a, LPR, VPL, st); break;
      case SG_PROP_GGCN_BWD_DST: e = dispatch_mode<SG_PROP_GGCN_BWD_DST>(dtype, vec, half_vec, a, LPR, VPL, st); break;
      case SG_PROP_GGCN_FWD_S: e = dispatch_mode<SG_PROP_GGCN_FWD_S>(dtype, vec, half_vec, a, LPR, VPL, st); break;
      default: e = dispatch_mode<SG_PROP_GGCN_BWD_SRC>(dtype, vec, half_vec, a, LPR, VPL, st); break;
    }
    if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "propagate launch: %s", cudaGetErrorString(e));
  }
  return SG_OK;
}

}  // extern "C"
