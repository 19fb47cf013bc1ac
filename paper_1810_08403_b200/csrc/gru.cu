// GG-NN ApplyVertex = GRU(vertex, accum) (Li et al. form
// without biases): the element-wise stages around the ApplyVertex GEMMs, each one fused
// kernel over the [V, F] state.  The GEMMs themselves (a [Wz|Wr|Wh], h [Uz|Ur], (r*h) Uh
// and their backward products) run on the tcgen05 GEMM; stacked weights put the three
// (two) gate blocks side by side with column-block stride `bs` (16-B aligned).
//
// Forward  (tensor.py op order, IEEE mul/add/div; sigmoid = 1 / (1 + exp(-x)) tensor.py:205):
//   gates:  z = s(G1[:,0] + G2[:,0]),  r = s(G1[:,bs] + G2[:,bs]),  rh = r * h
//   out:    c = tanh(G1[:,2bs] + G3),  h' = (1 - z) * h + z * c
// Backward (the tape's reverse sweep, tensor.py:231-236 and :258-263):
//   bwd1:   gz = g*c + (-(g*h)),  gc = g*z,  gh = g*(1-z),  gcp = gc*(1-c*c),  gzp = (gz*z)*(1-z)
//   bwd2:   (after grh = gcp Uh^T)  gr = grh*h,  gh += grh*r,  grp = (gr*r)*(1-r)
// D3 = [gzp | grp | gcp] (block stride bs) then feeds ga = D3 [Wz|Wr|Wh]^T and the weight
// gradients in single GEMMs.
#include <cuda_runtime.h>

#include <algorithm>

#include "common.h"

namespace {

// one 32 x 8 block per 8 rows (lanes over columns: coalesced, no index division), grid-stride
int grid_rows(int64_t V) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((V + 7) / 8, 148 * 16));
}

__device__ __forceinline__ float sigmoid_ref(float x) {
  return __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-x)));
}

__global__ void gru_gates_kernel(int64_t V, int64_t F, const float* G1, int64_t ld1,
                                 const float* G2, int64_t ld2, int64_t bs, const float* h,
                                 int64_t ldh, float* z, float* r, float* rh, int64_t ldo) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.y + threadIdx.y; v < V;
       v += (int64_t)gridDim.x * blockDim.y)
    for (int64_t c = threadIdx.x; c < F; c += 32) {
      const float zv = sigmoid_ref(__fadd_rn(G1[v * ld1 + c], G2[v * ld2 + c]));
      const float rv = sigmoid_ref(__fadd_rn(G1[v * ld1 + bs + c], G2[v * ld2 + bs + c]));
      z[v * ldo + c] = zv;
      r[v * ldo + c] = rv;
      rh[v * ldo + c] = __fmul_rn(rv, h[v * ldh + c]);
    }
}

__global__ void gru_out_kernel(int64_t V, int64_t F, const float* G1, int64_t ld1, int64_t bs,
                               const float* G3, int64_t ld3, const float* z, const float* h,
                               int64_t ldh, float* c_out, float* hn, int64_t ldo, int64_t ldn) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.y + threadIdx.y; v < V;
       v += (int64_t)gridDim.x * blockDim.y)
    for (int64_t k = threadIdx.x; k < F; k += 32) {
      const float cv = tanhf(__fadd_rn(G1[v * ld1 + 2 * bs + k], G3[v * ld3 + k]));
      const float zv = z[v * ldo + k], hv = h[v * ldh + k];
      c_out[v * ldo + k] = cv;
      hn[v * ldn + k] = __fadd_rn(__fmul_rn(__fsub_rn(1.0f, zv), hv), __fmul_rn(zv, cv));
    }
}

__global__ void gru_bwd1_kernel(int64_t V, int64_t F, const float* g, int64_t ldg, const float* z,
                                const float* c, int64_t ldo, const float* h, int64_t ldh, float* D3,
                                int64_t ld3, int64_t bs, float* gh, int64_t ldgh) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.y + threadIdx.y; v < V;
       v += (int64_t)gridDim.x * blockDim.y)
    for (int64_t k = threadIdx.x; k < F; k += 32) {
      const float gv = g[v * ldg + k], zv = z[v * ldo + k], cv = c[v * ldo + k], hv = h[v * ldh + k];
      const float gz = __fadd_rn(__fmul_rn(gv, cv), -__fmul_rn(gv, hv));
      const float gc = __fmul_rn(gv, zv);
      gh[v * ldgh + k] = __fmul_rn(gv, __fsub_rn(1.0f, zv));
      D3[v * ld3 + 2 * bs + k] = __fmul_rn(gc, __fsub_rn(1.0f, __fmul_rn(cv, cv)));
      D3[v * ld3 + k] = __fmul_rn(__fmul_rn(gz, zv), __fsub_rn(1.0f, zv));
    }
}

__global__ void gru_bwd2_kernel(int64_t V, int64_t F, const float* grh, int64_t ldr,
                                const float* r, int64_t ldo, const float* h, int64_t ldh,
                                float* gh, int64_t ldgh, float* D3, int64_t ld3, int64_t bs) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.y + threadIdx.y; v < V;
       v += (int64_t)gridDim.x * blockDim.y)
    for (int64_t k = threadIdx.x; k < F; k += 32) {
      const float g = grh[v * ldr + k], rv = r[v * ldo + k];
      const float gr = __fmul_rn(g, h[v * ldh + k]);
      gh[v * ldgh + k] = __fadd_rn(gh[v * ldgh + k], __fmul_rn(g, rv));
      D3[v * ld3 + bs + k] = __fmul_rn(__fmul_rn(gr, rv), __fsub_rn(1.0f, rv));
    }
}

}  // namespace

extern "C" {

int sg_gru_gates(int64_t V, int64_t F, const float* G1, int64_t ld1, const float* G2, int64_t ld2,
                 int64_t bs, const float* h, int64_t ldh, float* z, float* r, float* rh, int64_t ldo,
                 void* stream) {
  SG_REQUIRE(V >= 0 && F >= 0 && bs >= F, SG_ESHAPE, "gru_gates: bad extents");
  if (V * F == 0) return SG_OK;
  SG_REQUIRE(G1 && G2 && h && z && r && rh, SG_EINVAL, "gru_gates: null pointer");
  gru_gates_kernel<<<grid_rows(V), dim3(32, 8), 0, (cudaStream_t)stream>>>(V, F, G1, ld1, G2, ld2, bs, h,
                                                                      ldh, z, r, rh, ldo);
  sg::count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "gru_gates: %s", cudaGetErrorString(e));
  return SG_OK;
}

int sg_gru_out(int64_t V, int64_t F, const float* G1, int64_t ld1, int64_t bs, const float* G3,
               int64_t ld3, const float* z, const float* h, int64_t ldh, float* c, float* hn,
               int64_t ldo, int64_t ldn, void* stream) {
  SG_REQUIRE(V >= 0 && F >= 0 && bs >= F, SG_ESHAPE, "gru_out: bad extents");
  if (V * F == 0) return SG_OK;
  SG_REQUIRE(G1 && G3 && z && h && c && hn, SG_EINVAL, "gru_out: null pointer");
  gru_out_kernel<<<grid_rows(V), dim3(32, 8), 0, (cudaStream_t)stream>>>(V, F, G1, ld1, bs, G3, ld3, z, h,
                                                                    ldh, c, hn, ldo, ldn);
  sg::count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "gru_out: %s", cudaGetErrorString(e));
  return SG_OK;
}

int sg_gru_bwd1(int64_t V, int64_t F, const float* g, int64_t ldg, const float* z, const float* c,
                int64_t ldo, const float* h, int64_t ldh, float* D3, int64_t ld3, int64_t bs, float* gh,
                int64_t ldgh, void* stream) {
  SG_REQUIRE(V >= 0 && F >= 0 && bs >= F, SG_ESHAPE, "gru_bwd1: bad extents");
  if (V * F == 0) return SG_OK;
  SG_REQUIRE(g && z && c && h && D3 && gh, SG_EINVAL, "gru_bwd1: null pointer");
  gru_bwd1_kernel<<<grid_rows(V), dim3(32, 8), 0, (cudaStream_t)stream>>>(V, F, g, ldg, z, c, ldo, h, ldh,
                                                                     D3, ld3, bs, gh, ldgh);
  sg::count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "gru_bwd1: %s", cudaGetErrorString(e));
  return SG_OK;
}

int sg_gru_bwd2(int64_t V, int64_t F, const float* grh, int64_t ldr, const float* r, int64_t ldo,
                const float* h, int64_t ldh, float* gh, int64_t ldgh, float* D3, int64_t ld3, int64_t bs,
                void* stream) {
  SG_REQUIRE(V >= 0 && F >= 0 && bs >= F, SG_ESHAPE, "gru_bwd2: bad extents");
  if (V * F == 0) return SG_OK;
  SG_REQUIRE(grh && r && h && gh && D3, SG_EINVAL, "gru_bwd2: null pointer");
  gru_bwd2_kernel<<<grid_rows(V), dim3(32, 8), 0, (cudaStream_t)stream>>>(V, F, grh, ldr, r, ldo, h, ldh, gh,
                                                                     ldgh, D3, ld3, bs);
  sg::count_launch();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) SG_FAIL(SG_ECUDA, "gru_bwd2: %s", cudaGetErrorString(e));
  return SG_OK;
}

}  // extern "C"
