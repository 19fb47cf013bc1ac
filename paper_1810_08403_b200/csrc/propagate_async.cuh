// Wide-row propagation with per-lane cp.async (LDGSTS) prefetch into a shared-memory ring.
//
// Included by propagate.cu (shares ModeT / PropArgs / VecIO / add2_rn).  ncu on the
// register path for F = 602 shows the pass is latency bound (long_scoreboard ~9.5 per
// issue at 16 warps/SM): each warp can only hold DEPTH = 2 rows (10 x 16 B per lane)
// of loads in registers.  Here every lane streams its own 16-B column vectors of the
// next S source rows into a private slice of a shared-memory ring with
// cp.async.cg (L1 bypass; no register cost, no cross-lane dependency -- a lane only
// ever reads the bytes it copied), so S rows are in flight per warp.  Accumulation
// order and every output are identical to prop_kernel (bitwise).
#pragma once

namespace cpa {

__device__ __forceinline__ void cp16(uint32_t dst, const void* src) {
  // .ca keeps L1 allocation: hub source rows are re-read by neighbouring warps
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}

}  // namespace cpa

constexpr int kAsyncWarps = 8;

template <int MODE, int DT, int VPL, int S>
__global__ void __launch_bounds__(kAsyncWarps * 32, 2) prop_async_kernel(const PropArgs a) {
  constexpr int W = DT == SG_F32 ? 4 : 8;
  using M = ModeT<MODE>;
  using IO = VecIO<DT, W>;
  using Elem = typename IO::Elem;
  static_assert(M::NG == 1 && M::NR == 0 && M::NOUT == 1, "async path: single-operand modes");
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // ring layout: [warp][slot][VPL][32 lanes] x 16 B -> conflict-free LDS/LDGSTS
  const uint32_t ring = static_cast<uint32_t>(__cvta_generic_to_shared(smem)) +
                        (uint32_t)warp * S * VPL * 512 + lane * 16;
  const Elem* G = static_cast<const Elem*>(a.G) + lane * W;
  const bool last_ok = (VPL - 1) * 32 + lane < a.Fv;

  for (;;) {
    int it = 0;
    if (lane == 0) it = atomicAdd(a.queue, 1);
    it = __shfl_sync(0xffffffffu, it, 0);
    if (it >= a.n_items) break;
    const sg_item item = a.items[it];
    const bool split = item.split >= 0;
    const int64_t eb = split ? item.e_begin : __ldg(a.ptr + item.row_begin);
    const int64_t ee = split ? item.e_end : __ldg(a.ptr + item.row_end);
    const int n = (int)(ee - eb);

    int src_cur = 0, src_nxt = 0;
    float w_cur = 0.f;
    if (lane < n) {
      src_cur = __ldcs(a.idx + eb + lane);
      if (M::USE_W) w_cur = __ldcs(a.w + eb + lane);
    }
    float w_nxt = 0.f;
    if (32 + lane < n) {
      src_nxt = __ldcs(a.idx + eb + 32 + lane);
      if (M::USE_W) w_nxt = __ldcs(a.w + eb + 32 + lane);
    }
    auto issue = [&](int s, uint32_t slot) {
      const Elem* row = G + (uint64_t)(uint32_t)s * (uint32_t)a.ldg;
#pragma unroll
      for (int v = 0; v < VPL; ++v)
        if (v < VPL - 1 || last_ok) cpa::cp16(slot + v * 512, row + v * 32 * W);
    };
    // prologue: S rows in flight (one commit group per edge, empty groups past the end)
#pragma unroll
    for (int d = 0; d < S; ++d) {
      const int s = __shfl_sync(0xffffffffu, src_cur, d);
      if (d < n) issue(s, ring + d * VPL * 512);
      cpa::commit();
    }

    int r = item.row_begin;
    int64_t rend = split ? ee : __ldg(a.ptr + r + 1);
    float acc[VPL][W];
    auto init_row = [&](int row) {
#pragma unroll
      for (int v = 0; v < VPL; ++v)
#pragma unroll
        for (int k = 0; k < W; ++k) acc[v][k] = 0.f;
      if (a.accumulate && !split) {
#pragma unroll
        for (int v = 0; v < VPL; ++v)
          if (v < VPL - 1 || last_ok)
            IO::ld_cs(a.out0, (int64_t)row * a.ld0 + (int64_t)(v * 32 + lane) * W, acc[v]);
      }
    };
    auto store_row = [&](int row) {
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        const int cv = v * 32 + lane;
        if (v < VPL - 1 || last_ok) {
          if (a.mask) {
            float m[W];
            IO::ld_cs(a.mask, (int64_t)row * a.ldm + (int64_t)cv * W, m);
#pragma unroll
            for (int k = 0; k < W; ++k) acc[v][k] = __fmul_rn(acc[v][k], m[k] > 0.f ? 1.f : 0.f);
          }
          IO::st(a.out0, (int64_t)row * a.ld0 + (int64_t)cv * W, acc[v], min(W, a.Fcols - cv * W));
        }
      }
    };
    init_row(r);

    int k = 0;  // ring slot of edge j
#pragma unroll 1
    for (int j = 0; j < n; ++j) {
      if (!split) {
        while (eb + j >= rend) {  // row boundary (also rows without edges)
          store_row(r);
          ++r;
          rend = __ldg(a.ptr + r + 1);
          init_row(r);
        }
      }
      const float wj = M::USE_W ? __shfl_sync(0xffffffffu, w_cur, j & 31) : 0.f;
      const int jn = j + S;
      const int s_cur = __shfl_sync(0xffffffffu, src_cur, jn & 31);
      const int s_nxt = __shfl_sync(0xffffffffu, src_nxt, jn & 31);
      cpa::wait<S - 1>();  // this lane's copies of edge j have landed
      const uint32_t slot = ring + k * VPL * 512;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        if (v < VPL - 1 || last_ok) {
          uint4 raw = cpa::lds128(slot + v * 512);
          float x[W];
          IO::unpack(*reinterpret_cast<typename IO::Raw*>(&raw), x);
#pragma unroll
          for (int q = 0; q < W; q += 2) {
            float t0, t1, u0, u1;
            M::term(&x[q], &x[q], nullptr, nullptr, wj, &t0, &t1);
            M::term(&x[q + 1], &x[q + 1], nullptr, nullptr, wj, &u0, &u1);
            add2_rn(acc[v][q], acc[v][q + 1], t0, u0);
          }
        }
      }
      // refill the slot just consumed with edge j + S (the math above has used its bytes)
      if (jn < n) issue(((j & ~31) + 32 > jn) ? s_cur : s_nxt, slot);
      cpa::commit();
      if (++k == S) k = 0;
      if ((j & 31) == 31) {  // slide the index windows
        src_cur = src_nxt;
        w_cur = w_nxt;
        const int nb = j + 33 + lane;
        src_nxt = 0;
        if (nb < n) {
          src_nxt = __ldcs(a.idx + eb + nb);
          if (M::USE_W) w_nxt = __ldcs(a.w + eb + nb);
        }
      }
    }
    cpa::wait<0>();

    if (!split) {
      store_row(r);
      for (++r; r < item.row_end; ++r) {
        init_row(r);
        store_row(r);
      }
      continue;
    }
    const sg_split sp = a.splits[item.split];
    const int64_t pslot = sp.slot0 + item.sub;
#pragma unroll
    for (int v = 0; v < VPL; ++v) {
      const int cv = v * 32 + lane;
      if (v < VPL - 1 || last_ok) {
        float* p = a.partial + pslot * a.pld + (int64_t)cv * W;
#pragma unroll
        for (int q = 0; q < W; ++q) __stcg(p + q, acc[v][q]);
      }
    }
    __threadfence();
    __syncwarp();
    int ticket = 0;
    if (lane == 0) ticket = atomicAdd(a.counters + item.split, 1);
    ticket = __shfl_sync(0xffffffffu, ticket, 0);
    if (ticket == sp.n_sub - 1) {
      __threadfence();
      const int row = sp.row;
#pragma unroll
      for (int v = 0; v < VPL; ++v)
#pragma unroll
        for (int q = 0; q < W; ++q) acc[v][q] = 0.f;
      if (a.accumulate) {
#pragma unroll
        for (int v = 0; v < VPL; ++v)
          if (v < VPL - 1 || last_ok)
            IO::ld_cs(a.out0, (int64_t)row * a.ld0 + (int64_t)(v * 32 + lane) * W, acc[v]);
      }
#pragma unroll 1
      for (int s = 0; s < sp.n_sub; ++s) {
#pragma unroll
        for (int v = 0; v < VPL; ++v) {
          const int cv = v * 32 + lane;
          if (v < VPL - 1 || last_ok) {
            const float* p = a.partial + (sp.slot0 + s) * a.pld + (int64_t)cv * W;
#pragma unroll
            for (int q = 0; q < W; ++q) acc[v][q] = __fadd_rn(acc[v][q], __ldcg(p + q));
          }
        }
      }
      store_row(row);
      if (lane == 0) a.counters[item.split] = 0;
    }
  }
}
