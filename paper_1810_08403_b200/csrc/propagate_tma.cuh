// Wide-row propagation with TMA bulk copies into a per-warp shared-memory ring.
//
// Included by propagate.cu (shares ModeT / PropArgs / VecIO).  For rows wider than
// one warp-vector (F > 128 fp32) the register path can only keep ~2 rows in flight
// per warp and the pass is latency bound (ncu: long_scoreboard).  Here lane 0 of
// each warp issues one cp.async.bulk (TMA, SASS UBLKCP) per gathered source row
// into a ring of S shared-memory slots, each completing on its own mbarrier, while
// the warp consumes older slots with LDS.128 -- S rows (>= 19 KB for F = 602) in
// flight per warp without spending registers.  Accumulation order, split/combine
// semantics and outputs are identical to prop_kernel (bitwise).
#pragma once

namespace tma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// arm the barrier for `bytes` of transaction and issue the bulk copy global -> shared
__device__ __forceinline__ void load_row(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr));
  return v;
}

}  // namespace tma

constexpr int kTmaWarps = 8;

template <int MODE, int DT, int VPL>
__global__ void __launch_bounds__(kTmaWarps * 32, 2)
    prop_tma_kernel(const PropArgs a, int S, uint32_t slot_bytes) {
  constexpr int W = DT == SG_F32 ? 4 : 8;
  using M = ModeT<MODE>;
  using IO = VecIO<DT, W>;
  using Elem = typename IO::Elem;
  static_assert(M::NG == 1 && M::NR == 0 && M::NOUT == 1, "TMA path: single-operand modes");
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * S;
  const uint32_t bar_bytes = (uint32_t)((kTmaWarps * S * 8 + 127) / 128 * 128);
  const uint32_t ring = tma::smem_u32(smem) + bar_bytes + (uint32_t)(warp * S) * slot_bytes;
  unsigned char* ring_ptr = smem + bar_bytes + (size_t)warp * S * slot_bytes;
  if (lane == 0) {
    for (int k = 0; k < S; ++k) tma::mbar_init(bars + k, 1);
    tma::fence_mbar_init();
  }
  __syncwarp();
  const Elem* G = static_cast<const Elem*>(a.G);
  const bool last_ok = (VPL - 1) * 32 + lane < a.Fv;
  // ring cursor of the next slot to consume and the mbarrier phase parity of that use
  uint32_t kslot = 0, phase = 0;

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

    // index windows: cur = edges [32*kw, 32*kw+32), nxt = the following 32
    int src_cur = 0, src_nxt = 0;
    float w_cur = 0.f, w_nxt = 0.f;
    if (lane < n) {
      src_cur = __ldcs(a.idx + eb + lane);
      if (M::USE_W) w_cur = __ldcs(a.w + eb + lane);
    }
    if (32 + lane < n) {
      src_nxt = __ldcs(a.idx + eb + 32 + lane);
      if (M::USE_W) w_nxt = __ldcs(a.w + eb + 32 + lane);
    }
    // prologue: fill the ring
    const int pro = min(S, n);
    {
      uint32_t k = kslot;
      for (int j = 0; j < pro; ++j) {
        const int s = __shfl_sync(0xffffffffu, src_cur, j);
        if (lane == 0)
          tma::load_row(ring_ptr + (size_t)k * slot_bytes,
                        G + (uint64_t)(uint32_t)s * (uint32_t)a.ldg, slot_bytes, bars + k);
        k = (k + 1 == (uint32_t)S) ? 0u : k + 1;
      }
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
          if (v < VPL - 1 || last_ok) IO::ld_cs(a.out0, (int64_t)row * a.ld0 + (int64_t)(v * 32 + lane) * W, acc[v]);
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

#pragma unroll 1
    for (int j = 0; j < n; ++j) {
      if (!split) {
        while (eb + j >= rend) {  // row boundary (also skips rows without edges)
          store_row(r);
          ++r;
          rend = __ldg(a.ptr + r + 1);
          init_row(r);
        }
      }
      const uint32_t k = kslot;
      const float wj = M::USE_W ? __shfl_sync(0xffffffffu, w_cur, j & 31) : 0.f;
      tma::mbar_wait(bars + k, phase);
      const uint32_t slot = ring + k * slot_bytes;
#pragma unroll
      for (int v = 0; v < VPL; ++v) {
        if (v < VPL - 1 || last_ok) {
          uint4 raw = tma::lds128(slot + (uint32_t)(v * 32 + lane) * 16);
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
      // WAR on the slot: every lane's LDS result has been consumed by the math above, so
      // after the warp barrier the async-proxy refill cannot overtake a read (the same
      // release pattern as an mbarrier "empty" arrive; a proxy fence here would be a
      // MEMBAR that waits for this lane's in-flight bulk copies).
      __syncwarp();
      const int jn = j + S;
      const int lane_n = jn & 31;
      const int s_cur = __shfl_sync(0xffffffffu, src_cur, lane_n);
      const int s_nxt = __shfl_sync(0xffffffffu, src_nxt, lane_n);
      if (jn < n && lane == 0) {
        const int s = ((j & ~31) + 32 > jn) ? s_cur : s_nxt;
        tma::load_row(ring_ptr + (size_t)k * slot_bytes, G + (uint64_t)(uint32_t)s * (uint32_t)a.ldg,
                      slot_bytes, bars + k);
      }
      if (++kslot == (uint32_t)S) {
        kslot = 0;
        phase ^= 1u;
      }
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

    if (!split) {
      store_row(r);
      for (++r; r < item.row_end; ++r) {  // trailing rows without edges
        init_row(r);
        store_row(r);
      }
      continue;
    }
    // split subgroup: partial -> workspace slot; the last finisher combines in order
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
          if (v < VPL - 1 || last_ok) IO::ld_cs(a.out0, (int64_t)row * a.ld0 + (int64_t)(v * 32 + lane) * W, acc[v]);
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
