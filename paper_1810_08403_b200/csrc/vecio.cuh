// 128-bit vector loads/stores with fp32 compute for fp32 / bf16 storage.
//
// A "vector" is W elements = 16 bytes (W = 4 fp32 or 8 bf16) or a single element
// (W = 1).  Loads return the raw bits (Raw) so that in-flight data costs the same
// registers for both dtypes; unpack() widens to fp32 at the point of use.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/sagann.h"

#ifndef SG_ROW_LOAD
#define SG_ROW_LOAD 3
#endif

namespace sg {

// bf16 gathered rows with the same L1 policy as the fp32 ones (SG_ROW_LOAD 3: evict_last)
__device__ __forceinline__ uint4 ld_row_u4(const uint4* p) {
#if SG_ROW_LOAD == 3
  uint4 r;
  asm volatile("ld.global.nc.L1::evict_last.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
#else
  return __ldg(p);
#endif
}
__device__ __forceinline__ uint2 ld_row_u2(const uint2* p) {
#if SG_ROW_LOAD == 3
  uint2 r;
  asm volatile("ld.global.nc.L1::evict_last.v2.u32 {%0, %1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
#else
  return __ldg(p);
#endif
}

template <int DT, int W>
struct VecIO;

template <>
struct VecIO<SG_F32, 4> {
  using Elem = float;
  using Raw = float4;
  // gathered-row load (SG_ROW_LOAD for A/B builds): 0 = ld.global.nc, 1 = +L1::no_allocate,
  // 2 = +L1::evict_first, 3 = +L1::evict_last (default), 4 = ld.global.cg (L2 only).  Reddit epoch
  // (profiles/r02_occupancy_ab.txt): evict_last 19.2-19.3 ms vs 20.1 (nc), 25.1 (no_allocate),
  // 24.4 (evict_first), 21.2-21.4 (cg): the gathered rows are re-read by later edges, the
  // index / weight / output streams (ld.cs / st.cs) are not
  static __device__ __forceinline__ Raw ld_raw(const Elem* p) {
#if SG_ROW_LOAD == 0
    return __ldg(reinterpret_cast<const float4*>(p));
#elif SG_ROW_LOAD == 4
    return __ldcg(reinterpret_cast<const float4*>(p));
#else
    float4 r;
#if SG_ROW_LOAD == 1
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
#elif SG_ROW_LOAD == 2
    asm volatile("ld.global.nc.L1::evict_first.v4.f32 {%0, %1, %2, %3}, [%4];"
#else
    asm volatile("ld.global.nc.L1::evict_last.v4.f32 {%0, %1, %2, %3}, [%4];"
#endif
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
#endif
  }
  static __device__ __forceinline__ void unpack(const Raw& r, float* v) {
    v[0] = r.x; v[1] = r.y; v[2] = r.z; v[3] = r.w;
  }
  static __device__ __forceinline__ void ld_nc(const void* base, int64_t off, float* v) {
    unpack(ld_raw(static_cast<const float*>(base) + off), v);
  }
  static __device__ __forceinline__ void ld_cs(const void* base, int64_t off, float* v) {
    unpack(__ldcs(reinterpret_cast<const float4*>(static_cast<const float*>(base) + off)), v);
  }
  static __device__ __forceinline__ void st(void* base, int64_t off, const float* v, int nvalid) {
    float* p = static_cast<float*>(base) + off;
    if (nvalid >= 4) {
      __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
    } else {
      for (int k = 0; k < nvalid; ++k) p[k] = v[k];
    }
  }
};

// 8 fp32 (two float4): the fp32 output side of a pass whose inputs are 8-element bf16 vectors
template <>
struct VecIO<SG_F32, 8> {
  using Elem = float;
  static __device__ __forceinline__ void ld_cs(const void* base, int64_t off, float* v) {
    const float4* p = reinterpret_cast<const float4*>(static_cast<const float*>(base) + off);
    const float4 a = __ldcs(p), b = __ldcs(p + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  static __device__ __forceinline__ void st(void* base, int64_t off, const float* v, int nvalid) {
    float* p = static_cast<float*>(base) + off;
    if (nvalid >= 8) {
      __stcs(reinterpret_cast<float4*>(p), make_float4(v[0], v[1], v[2], v[3]));
      __stcs(reinterpret_cast<float4*>(p) + 1, make_float4(v[4], v[5], v[6], v[7]));
    } else {
      for (int k = 0; k < nvalid; ++k) p[k] = v[k];
    }
  }
};

template <>
struct VecIO<SG_F32, 1> {
  using Elem = float;
  using Raw = float;
  static __device__ __forceinline__ Raw ld_raw(const Elem* p) { return __ldg(p); }
  static __device__ __forceinline__ void unpack(const Raw& r, float* v) { v[0] = r; }
  static __device__ __forceinline__ void ld_nc(const void* base, int64_t off, float* v) {
    v[0] = __ldg(static_cast<const float*>(base) + off);
  }
  static __device__ __forceinline__ void ld_cs(const void* base, int64_t off, float* v) {
    v[0] = __ldcs(static_cast<const float*>(base) + off);
  }
  static __device__ __forceinline__ void st(void* base, int64_t off, const float* v, int nvalid) {
    if (nvalid >= 1) static_cast<float*>(base)[off] = v[0];
  }
};

template <>
struct VecIO<SG_BF16, 8> {
  using Elem = __nv_bfloat16;
  using Raw = uint4;
  static __device__ __forceinline__ Raw ld_raw(const Elem* p) {
    return ld_row_u4(reinterpret_cast<const uint4*>(p));
  }
  static __device__ __forceinline__ void unpack(const Raw& r, float* v) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float2 f = __bfloat1622float2(h[k]);
      v[2 * k] = f.x;
      v[2 * k + 1] = f.y;
    }
  }
  static __device__ __forceinline__ void ld_nc(const void* base, int64_t off, float* v) {
    unpack(ld_raw(static_cast<const __nv_bfloat16*>(base) + off), v);
  }
  static __device__ __forceinline__ void ld_cs(const void* base, int64_t off, float* v) {
    unpack(__ldcs(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(base) + off)), v);
  }
  static __device__ __forceinline__ void st(void* base, int64_t off, const float* v, int nvalid) {
    __nv_bfloat16* p = static_cast<__nv_bfloat16*>(base) + off;
    if (nvalid >= 8) {
      uint4 r;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
      for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
      __stcs(reinterpret_cast<uint4*>(p), r);
    } else {
      for (int k = 0; k < nvalid; ++k) p[k] = __float2bfloat16_rn(v[k]);
    }
  }
};

// half vector (4 bf16 = 8 bytes): bf16 rows of <= 128 columns fill a whole warp with it
template <>
struct VecIO<SG_BF16, 4> {
  using Elem = __nv_bfloat16;
  using Raw = uint2;
  static __device__ __forceinline__ Raw ld_raw(const Elem* p) {
    return ld_row_u2(reinterpret_cast<const uint2*>(p));
  }
  static __device__ __forceinline__ void unpack(const Raw& r, float* v) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&r);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      float2 f = __bfloat1622float2(h[k]);
      v[2 * k] = f.x;
      v[2 * k + 1] = f.y;
    }
  }
  static __device__ __forceinline__ void ld_nc(const void* base, int64_t off, float* v) {
    unpack(ld_raw(static_cast<const __nv_bfloat16*>(base) + off), v);
  }
  static __device__ __forceinline__ void ld_cs(const void* base, int64_t off, float* v) {
    unpack(__ldcs(reinterpret_cast<const uint2*>(static_cast<const __nv_bfloat16*>(base) + off)), v);
  }
  static __device__ __forceinline__ void st(void* base, int64_t off, const float* v, int nvalid) {
    __nv_bfloat16* p = static_cast<__nv_bfloat16*>(base) + off;
    if (nvalid >= 4) {
      uint2 r;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&r);
      h[0] = __floats2bfloat162_rn(v[0], v[1]);
      h[1] = __floats2bfloat162_rn(v[2], v[3]);
      __stcs(reinterpret_cast<uint2*>(p), r);
    } else {
      for (int k = 0; k < nvalid; ++k) p[k] = __float2bfloat16_rn(v[k]);
    }
  }
};

template <>
struct VecIO<SG_BF16, 1> {
  using Elem = __nv_bfloat16;
  using Raw = __nv_bfloat16;
  static __device__ __forceinline__ Raw ld_raw(const Elem* p) { return p[0]; }
  static __device__ __forceinline__ void unpack(const Raw& r, float* v) { v[0] = __bfloat162float(r); }
  static __device__ __forceinline__ void ld_nc(const void* base, int64_t off, float* v) {
    v[0] = __bfloat162float(static_cast<const __nv_bfloat16*>(base)[off]);
  }
  static __device__ __forceinline__ void ld_cs(const void* base, int64_t off, float* v) {
    v[0] = __bfloat162float(static_cast<const __nv_bfloat16*>(base)[off]);
  }
  static __device__ __forceinline__ void st(void* base, int64_t off, const float* v, int nvalid) {
    if (nvalid >= 1) static_cast<__nv_bfloat16*>(base)[off] = __float2bfloat16_rn(v[0]);
  }
};

// (a0, a1) += (t0, t1) with one packed FADD2 (add.rn.f32x2): per-lane IEEE
// round-to-nearest, i.e. bitwise the same as two scalar adds.  (ptxas contracts a
// packed mul.rn.f32x2 feeding this into FFMA2, so products stay scalar __fmul_rn.)
__device__ __forceinline__ void add2_rn(float& a0, float& a1, float t0, float t1) {
  asm("{\n\t.reg .b64 a, t;\n\t"
      "mov.b64 a, {%0, %1};\n\t"
      "mov.b64 t, {%2, %3};\n\t"
      "add.rn.f32x2 a, a, t;\n\t"
      "mov.b64 {%0, %1}, a;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "f"(t0), "f"(t1));
}

}  // namespace sg
