// Source-staged gather for the sum passes (GCN / PASS modes, fp32): sg_propagate_staged.
//
// The row-per-warp kernel of propagate.cu loads one source row per (unique) edge through L2,
// and on the Reddit-shaped graph that L2 -> SM stream (~195 GB per F = 602 pass, 16 TB/s) is
// what bounds it.  Here a CTA owns a GROUP of pieces (destination rows, or T-edge subgroups
// of heavy rows -- the same subgroups as sg_host_plan) whose sources overlap (sg_host_stage_plan
// orders pieces by first source), and stages the group's merged source list into shared
// memory with TMA bulk copies, batch by batch, so a source row shared by several pieces of the
// group crosses L2 -> SM once (R-MAT: ~half the row loads for groups of 32 pieces).
//
// CTA = 4 producer warps + 16 consumer warps; consumer warp w owns piece w of the group, its
// lanes the row's 16-byte column vectors (as in the row-per-warp kernel).  2-3 shared-memory
// stages, each a batch of up to S source rows + up to EMAX entries + the per-piece entry
// offsets; full / empty mbarriers between the producers (cp.async 16-byte copies arriving on
// full[stage] as they complete) and the consumers.
//
// Order / parity: each piece's entries are its edges in index order (runs of equal consecutive
// (source, weight) carry a count and add their term count times: the same IEEE adds), batches
// ascend in source, so every row adds exactly the sequence of terms sg_propagate adds, with
// __fmul_rn / add.rn (-fmad=false).  Split subgroups write partial slots and the last finisher
// combines them in subgroup order from the same workspace layout: bitwise identical results.
#include <cuda_runtime.h>

#include "common.h"
#include "sm100.cuh"
#include "vecio.cuh"

namespace {

struct StageArgs {
  const sg_stage_piece* pieces;
  const int32_t* group_batch;
  const int64_t* batch_src_off;
  const int32_t* batch_src;
  const int64_t* batch_ent_off;
  const uint64_t* entries;
  const uint16_t* batch_pofs;
  int32_t n_groups, pofs_stride, S, EMAX;
  const float* G;
  int64_t ldg;
  float* out;
  int64_t ldo;
  const float* mask;
  int64_t ldm;
  int32_t Fv, Fcols, accumulate, use_w;
  float* partial;
  int64_t pld;
  int32_t* counters;
  int32_t* queue;
};

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sm100::smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          sm100::smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(sm100::smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sm100::smem_u32(dst)), "l"(src) : "memory");
}

// arrive on the mbarrier when all of this thread's prior cp.async copies have completed
// (.noinc: the arrival counts toward the barrier's expected count)
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sm100::smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void add4(float (&a)[4], const float (&t)[4]) {
  using sg::add2_rn;
  add2_rn(a[0], a[1], t[0], t[1]);
  add2_rn(a[2], a[3], t[2], t[3]);
}

constexpr int NPROD = 4;         // producer warps
constexpr int kStageWarps = 16;  // consumer warps = pieces per group

// per-stage metadata written by the producer
struct StageMeta {
  int32_t group, batch, first, last, n_ent;
  int32_t pad[3];
};

template <int VPL, int NW, int NST>
__global__ void __launch_bounds__((NW + NPROD) * 32, 1) staged_kernel(const StageArgs a) {
  static_assert(NST >= 2 && NST <= 4, "2-4 stages");
  constexpr int NCONS = NW;
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);             // [NST]
  uint64_t* empty = full + NST;                                     // [NST]
  StageMeta* meta = reinterpret_cast<StageMeta*>(smem + 64);       // [NST + 1] x 32 B
  const int row_bytes = a.Fv * 16;
  const int ent_bytes = a.EMAX * 8, pofs_bytes = a.pofs_stride * 2;
  const int stage_bytes = ((a.S * row_bytes + ent_bytes + pofs_bytes) + 127) / 128 * 128;
  unsigned char* stage0 = smem + 256;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      sm100::mbar_init(full + s, NPROD * 32 + 1);
      sm100::mbar_init(empty + s, NCONS);
    }
    sm100::fence_mbar_init();
  }
  __syncthreads();

  if (warp >= NCONS) {
    // ---------------------------------------------------------------- producer warps
    // cp.async (LDGSTS, 16 B per lane, L2-only) row copies: per-row TMA bulk copies measured
    // ~300-500 cycles each on the SM's TMA unit (the pass ran 3-13x slower), LDGSTS is 8 cycles
    // per warp op.  Each producer thread's copies arrive on full[stage] when they complete
    // (cp.async.mbarrier.arrive.noinc), plus one plain arrive after the metadata is written.
    const int pw = warp - NCONS, pt = threadIdx.x - NCONS * 32;
    int stage = 0;
    uint32_t phase = 0;
    for (;;) {
      int g = 0;
      if (pt == 0) g = atomicAdd(a.queue, 1);
      // broadcast the group id to the producer warps through the stage's metadata slot
      named_sync(15, NPROD * 32);
      if (pt == 0) meta[NST].group = g;
      named_sync(15, NPROD * 32);
      g = meta[NST].group;
      const bool done = g >= a.n_groups;
      const int b0 = done ? 0 : __ldg(a.group_batch + g), b1 = done ? 1 : __ldg(a.group_batch + g + 1);
      // batch offsets prefetched one batch ahead; the batch's source ids are loaded lane-
      // parallel (row pw + NPROD * k in lane k % 32 of register k / 32) before the empty wait,
      // so no global-load latency sits between two row copies
      int64_t s1n = 0, e1n = 0, s0 = 0, e0 = 0;
      if (!done) {
        s0 = __ldg(a.batch_src_off + b0);
        e0 = __ldg(a.batch_ent_off + b0);
        s1n = __ldg(a.batch_src_off + b0 + 1);
        e1n = __ldg(a.batch_ent_off + b0 + 1);
      }
      for (int b = b0; b < b1; ++b) {
        const int64_t s1 = s1n, e1 = e1n;
        if (!done && b + 1 < b1) {
          s1n = __ldg(a.batch_src_off + b + 2);
          e1n = __ldg(a.batch_ent_off + b + 2);
        }
        const int nrows = (int)(s1 - s0), nent = (int)(e1 - e0);
        int src0 = 0, src1 = 0;
        if (!done) {
          const int r0 = pw + NPROD * lane, r1 = pw + NPROD * (lane + 32);
          if (r0 < nrows) src0 = __ldg(a.batch_src + s0 + r0);
          if (r1 < nrows) src1 = __ldg(a.batch_src + s0 + r1);
        }
        sm100::mbar_wait(empty + stage, phase ^ 1u);
        unsigned char* st = stage0 + stage * stage_bytes;
        if (done) {
          if (pt == 0) meta[stage].group = -1;
        } else {
          if (pt == 0) meta[stage] = StageMeta{g, b, b == b0, b == b1 - 1, nent, {0, 0, 0}};
          const int my_rows = (nrows - pw + NPROD - 1) / NPROD;
          for (int k = 0; k < my_rows; ++k) {
            const int src = __shfl_sync(0xffffffffu, k < 32 ? src0 : src1, k & 31);
            const int r = pw + NPROD * k;
            const float4* gsrc = reinterpret_cast<const float4*>(a.G + (int64_t)src * a.ldg);
            float4* dst = reinterpret_cast<float4*>(st + r * row_bytes);
            for (int c = lane; c < a.Fv; c += 32) cp_async16(dst + c, gsrc + c);
          }
          unsigned char* ent = st + a.S * row_bytes;
          const float4* gent = reinterpret_cast<const float4*>(a.entries + e0);
          for (int c = pt; c < nent / 2; c += NPROD * 32) cp_async16(reinterpret_cast<float4*>(ent) + c, gent + c);
          const float4* gpo = reinterpret_cast<const float4*>(a.batch_pofs + (int64_t)b * a.pofs_stride);
          for (int c = pt; c < pofs_bytes / 16; c += NPROD * 32)
            cp_async16(reinterpret_cast<float4*>(ent + ent_bytes) + c, gpo + c);
        }
        cp_async_arrive_noinc(full + stage);
        if (pt == 0) sm100::mbar_arrive(full + stage);
        if (done) return;
        if (++stage == NST) {
          stage = 0;
          phase ^= 1u;
        }
        s0 = s1;
        e0 = e1;
      }
    }
  }

  // ------------------------------------------------------------------ consumer warps
  // warp w owns piece w of the group; lane l the 16-byte column vectors l, l + 32, ... (VPL)
  const bool last_ok = (VPL - 1) * 32 + lane < a.Fv;
  float acc[VPL][4];
  sg_stage_piece p{-1, -1, 0, 0};
  int stage = 0;
  uint32_t phase = 0;
  for (;;) {
    sm100::mbar_wait(full + stage, phase);
    const StageMeta m = meta[stage];
    if (m.group < 0) return;
    const unsigned char* st = stage0 + stage * stage_bytes;
    const float4* rows = reinterpret_cast<const float4*>(st) + lane;
    const uint64_t* ent = reinterpret_cast<const uint64_t*>(st + a.S * row_bytes);
    const uint16_t* pofs = reinterpret_cast<const uint16_t*>(st + a.S * row_bytes + ent_bytes);
    if (m.first) {
      p = a.pieces[(int64_t)m.group * NW + warp];
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        acc[k][0] = acc[k][1] = acc[k][2] = acc[k][3] = 0.f;
        if (a.accumulate && p.row >= 0 && p.split < 0 && (k < VPL - 1 || last_ok))
          sg::VecIO<SG_F32, 4>::ld_cs(a.out, (int64_t)p.row * a.ldo + (int64_t)(k * 32 + lane) * 4, acc[k]);
      }
    }
    int e = pofs[warp];
    const int e1 = pofs[warp + 1];
    // two entries in flight: all their row vectors are loaded before the ordered adds
    for (; e + 1 < e1; e += 2) {
      const uint64_t x0 = ent[e], x1 = ent[e + 1];
      const float4* r0 = rows + (int)(x0 & 0xffffu) * a.Fv;
      const float4* r1 = rows + (int)(x1 & 0xffffu) * a.Fv;
      float4 g0[VPL], g1[VPL];
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        if (k < VPL - 1 || last_ok) {
          g0[k] = r0[k * 32];
          g1[k] = r1[k * 32];
        }
      }
      const float w0 = a.use_w ? __uint_as_float((uint32_t)(x0 >> 32)) : 1.f;
      const float w1 = a.use_w ? __uint_as_float((uint32_t)(x1 >> 32)) : 1.f;
      const int c0 = (int)((x0 >> 16) & 0xffffu), c1 = (int)((x1 >> 16) & 0xffffu);
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        float t[4] = {g0[k].x, g0[k].y, g0[k].z, g0[k].w};
        if (a.use_w) {
#pragma unroll
          for (int c = 0; c < 4; ++c) t[c] = __fmul_rn(t[c], w0);
        }
        for (int c = 0; c < c0; ++c) add4(acc[k], t);
      }
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        float t[4] = {g1[k].x, g1[k].y, g1[k].z, g1[k].w};
        if (a.use_w) {
#pragma unroll
          for (int c = 0; c < 4; ++c) t[c] = __fmul_rn(t[c], w1);
        }
        for (int c = 0; c < c1; ++c) add4(acc[k], t);
      }
    }
    if (e < e1) {
      const uint64_t x0 = ent[e];
      const float4* r0 = rows + (int)(x0 & 0xffffu) * a.Fv;
      const float w0 = a.use_w ? __uint_as_float((uint32_t)(x0 >> 32)) : 1.f;
      const int c0 = (int)((x0 >> 16) & 0xffffu);
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
        if (k < VPL - 1 || last_ok) g = r0[k * 32];
        float t[4] = {g.x, g.y, g.z, g.w};
        if (a.use_w) {
#pragma unroll
          for (int c = 0; c < 4; ++c) t[c] = __fmul_rn(t[c], w0);
        }
        for (int c = 0; c < c0; ++c) add4(acc[k], t);
      }
    }
    __syncwarp();
    if (lane == 0) sm100::mbar_arrive(empty + stage);
    const bool last = m.last;
    if (++stage == NST) {
      stage = 0;
      phase ^= 1u;
    }
    if (!last || p.row < 0) continue;

    // ---------------------------------------------------------------- piece end: outputs
    if (p.split < 0) {
#pragma unroll
      for (int k = 0; k < VPL; ++k) {
        if (!(k < VPL - 1 || last_ok)) continue;
        const int v = k * 32 + lane;
        if (a.mask) {
          float mk[4];
          sg::VecIO<SG_F32, 4>::ld_cs(a.mask, (int64_t)p.row * a.ldm + (int64_t)v * 4, mk);
#pragma unroll
          for (int c = 0; c < 4; ++c) acc[k][c] = __fmul_rn(acc[k][c], mk[c] > 0.f ? 1.f : 0.f);
        }
        sg::VecIO<SG_F32, 4>::st(a.out, (int64_t)p.row * a.ldo + (int64_t)v * 4, acc[k], min(4, a.Fcols - v * 4));
      }
      continue;
    }
    // split subgroup: partial slot, the last finisher combines in subgroup order
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      if (!(k < VPL - 1 || last_ok)) continue;
      float* pp = a.partial + (int64_t)(p.slot0 + (p.sub_nsub >> 16)) * a.pld + (int64_t)(k * 32 + lane) * 4;
#pragma unroll
      for (int c = 0; c < 4; ++c) __stcg(pp + c, acc[k][c]);
    }
    __threadfence();
    __syncwarp();
    int ticket = 0;
    if (lane == 0) ticket = atomicAdd(a.counters + p.split, 1);
    ticket = __shfl_sync(0xffffffffu, ticket, 0);
    const int nsub = p.sub_nsub & 0xffff;
    if (ticket != nsub - 1) continue;
    __threadfence();
#pragma unroll
    for (int k = 0; k < VPL; ++k) {
      if (!(k < VPL - 1 || last_ok)) continue;
      const int v = k * 32 + lane;
      float s4[4] = {0.f, 0.f, 0.f, 0.f};
      if (a.accumulate) sg::VecIO<SG_F32, 4>::ld_cs(a.out, (int64_t)p.row * a.ldo + (int64_t)v * 4, s4);
      for (int s = 0; s < nsub; ++s) {
        const float* pp = a.partial + (int64_t)(p.slot0 + s) * a.pld + (int64_t)v * 4;
#pragma unroll
        for (int c = 0; c < 4; ++c) s4[c] = __fadd_rn(s4[c], __ldcg(pp + c));
      }
      if (a.mask) {
        float mk[4];
        sg::VecIO<SG_F32, 4>::ld_cs(a.mask, (int64_t)p.row * a.ldm + (int64_t)v * 4, mk);
#pragma unroll
        for (int c = 0; c < 4; ++c) s4[c] = __fmul_rn(s4[c], mk[c] > 0.f ? 1.f : 0.f);
      }
      sg::VecIO<SG_F32, 4>::st(a.out, (int64_t)p.row * a.ldo + (int64_t)v * 4, s4, min(4, a.Fcols - v * 4));
    }
    if (lane == 0) a.counters[p.split] = 0;
  }
}

int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

template <int VPL>
cudaError_t launch_staged(const StageArgs& a, cudaStream_t st, int n_sm, int nst) {
  constexpr int NW = kStageWarps;
  auto k = nst == 3 ? staged_kernel<VPL, NW, 3> : staged_kernel<VPL, NW, 2>;
  const int row_bytes = a.Fv * 16;
  const int64_t stage = align_up((int64_t)a.S * row_bytes + (int64_t)a.EMAX * 8 + a.pofs_stride * 2, 128);
  const size_t smem = 256 + nst * stage;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int grid = std::max(1, std::min(n_sm, a.n_groups));
  k<<<grid, (NW + NPROD) * 32, smem, st>>>(a);
  sg::count_launch();
  return cudaGetLastError();
}

}  // namespace

extern "C" {

int32_t sg_stage_group_pieces(int64_t F) { return F < 1 || F > 640 ? 0 : kStageWarps; }

int64_t sg_stage_smem_bytes(int32_t group_pieces, int32_t batch_rows, int32_t batch_entries, int64_t F,
                            int32_t stages) {
  const int64_t pstride = (group_pieces + 1 + 7) / 8 * 8;
  const int64_t row_bytes = (F + 3) / 4 * 16;
  const int64_t stage = align_up((int64_t)batch_rows * row_bytes + (int64_t)batch_entries * 8 + pstride * 2, 128);
  return 256 + stages * stage;
}

int sg_propagate_staged(int mode, const sg_stage_piece* pieces, const int32_t* group_batch, int64_t n_groups,
                        const int64_t* batch_src_off, const int32_t* batch_src, const int64_t* batch_ent_off,
                        const uint64_t* entries, const uint16_t* batch_pofs, int32_t group_pieces,
                        int32_t batch_rows, int32_t batch_entries, int32_t stages, int64_t n_splits,
                        int64_t n_slots, const float* G, int64_t ldg, float* out, int64_t ldo, const float* mask,
                        int64_t ldm, int64_t F, int accumulate, void* workspace, int64_t workspace_bytes,
                        void* stream) {
  SG_REQUIRE(stages == 2 || stages == 3, SG_EINVAL, "staged gather: 2 or 3 stages");
  SG_REQUIRE(mode == SG_PROP_PASS || mode == SG_PROP_GCN, SG_EINVAL, "staged gather: PASS / GCN modes only");
  SG_REQUIRE(n_groups >= 0 && n_groups <= INT32_MAX, SG_EINVAL, "staged gather: bad group count");
  if (n_groups == 0 || F == 0) return SG_OK;
  SG_REQUIRE(pieces && group_batch && batch_src_off && batch_src && batch_ent_off && entries && batch_pofs &&
                 G && out,
             SG_EINVAL, "staged gather: null pointer");
  SG_REQUIRE(ldg % 4 == 0 && ldo % 4 == 0 && (!mask || ldm % 4 == 0) && ((uintptr_t)G % 16) == 0 &&
                 ((uintptr_t)out % 16) == 0 && (!mask || ((uintptr_t)mask % 16) == 0),
             SG_EINVAL, "staged gather: rows must be 16-byte aligned");
  const int64_t need = sg_propagate_workspace_bytes(0, n_splits, n_slots, F, mode);
  SG_REQUIRE(workspace && workspace_bytes >= need, SG_EBUDGET, "staged gather workspace too small");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
  StageArgs a;
  a.pieces = pieces; a.group_batch = group_batch; a.batch_src_off = batch_src_off; a.batch_src = batch_src;
  a.batch_ent_off = batch_ent_off; a.entries = entries; a.batch_pofs = batch_pofs;
  a.n_groups = (int32_t)n_groups; a.pofs_stride = (group_pieces + 1 + 7) / 8 * 8;
  a.S = batch_rows; a.EMAX = batch_entries;
  a.queue = reinterpret_cast<int32_t*>(ws);
  a.counters = reinterpret_cast<int32_t*>(ws + 256);
  a.partial = reinterpret_cast<float*>(ws + 256 + align_up(4 * std::max<int64_t>(n_splits, 1), 256));
  a.pld = align_up(F, 8);
  a.accumulate = accumulate;
  a.use_w = mode == SG_PROP_GCN;
  int n_sm = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  }
  SG_REQUIRE(F <= 640, SG_EINVAL, "staged gather: rows of at most 640 fp32 (F = %lld)", (long long)F);
  SG_REQUIRE(batch_entries % 2 == 0, SG_EINVAL, "staged gather: batch_entries must be even");
  SG_REQUIRE(batch_rows <= NPROD * 64, SG_EINVAL, "staged gather: at most %d rows per batch", NPROD * 64);
  {
    const int Fv = (int)((F + 3) / 4);
    const int ncw = (Fv + 31) / 32;
    a.G = G; a.ldg = ldg; a.out = out; a.ldo = ldo; a.mask = mask; a.ldm = ldm;
    a.Fv = Fv; a.Fcols = (int32_t)F;
    cudaError_t e = cudaMemsetAsync(ws, 0, 256 + align_up(4 * std::max<int64_t>(n_splits, 1), 256), st);
    if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "memset: %s", cudaGetErrorString(e));
    SG_REQUIRE(group_pieces == kStageWarps, SG_EINVAL, "staged gather: plan groups of %d pieces, kernel %d",
               (int)group_pieces, kStageWarps);
    switch (ncw) {
      case 1: e = launch_staged<1>(a, st, n_sm, stages); break;
      case 2: e = launch_staged<2>(a, st, n_sm, stages); break;
      case 3: e = launch_staged<3>(a, st, n_sm, stages); break;
      case 4: e = launch_staged<4>(a, st, n_sm, stages); break;
      default: e = launch_staged<5>(a, st, n_sm, stages); break;
    }
    if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "staged gather launch: %s", cudaGetErrorString(e));
  }
  return SG_OK;
}

}  // extern "C"
