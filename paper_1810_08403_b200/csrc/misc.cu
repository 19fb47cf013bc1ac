// Loss head, optimizer step, strict-mode check, elementwise ApplyEdge ops, dtype staging.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "common.h"

namespace {

int grid_for(int64_t work, int per_block) {
  int64_t g = (work + per_block - 1) / per_block;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 148 * 32));
}

// softmax_cross_entropy (tensor.py:487-506): one warp per row.
__global__ void xent_rows_kernel(const float* Z, int64_t ldz, int relu_input, const int64_t* lab,
                                 int64_t n, int64_t C, int64_t n_total, float* dZ, int64_t lddz,
                                 float* logp_out, int32_t* err) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const float inv_n = 1.0f / (float)n_total;
  for (int64_t r = warp; r < n; r += nwarps) {
    const float* z = Z + r * ldz;
    int64_t l = lab[r];
    if (l < 0 || l >= C) {
      if (lane == 0) atomicOr(err, 1);
      l = 0;
    }
    float zmax = -INFINITY;
    for (int64_t c = lane; c < C; c += 32) {
      float v = z[c];
      if (relu_input) v = sg::relu_np(v);
      zmax = fmaxf(zmax, v);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) zmax = fmaxf(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
    float denom = 0.f;
    for (int64_t c = lane; c < C; c += 32) {
      float v = z[c];
      if (relu_input) v = sg::relu_np(v);
      denom += expf(v - zmax);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) denom += __shfl_xor_sync(0xffffffffu, denom, o);
    const float logd = logf(denom);
    for (int64_t c = lane; c < C; c += 32) {
      const float zc = z[c];
      const float v = relu_input ? sg::relu_np(zc) : zc;
      const float p = expf(v - zmax) / denom;
      float g = (p - (c == l ? 1.f : 0.f)) * inv_n;     // g * (p - onehot) / n, g = 1
      if (relu_input) g = g * (zc > 0.f ? 1.f : 0.f);   // relu bwd (tensor.py:236)
      dZ[r * lddz + c] = g;
      if (c == l) logp_out[r] = (v - zmax) - logd;
    }
  }
}

// Deterministic mean in two launches: kXentParts blocks each sum a fixed contiguous range
// (fixed per-thread strided order, fixed tree, fp64), then one block adds the partials in a
// fixed tree.  kXentParts is a constant (not the SM count) so results do not depend on the GPU.
constexpr int kXentParts = 148;

__global__ void xent_partial_kernel(const float* logp, int64_t n, double* part) {
  __shared__ double s[256];
  const int64_t chunk = (n + kXentParts - 1) / kXentParts;
  const int64_t b = (int64_t)blockIdx.x * chunk, e = min(n, b + chunk);
  double acc = 0.0;
  for (int64_t i = b + threadIdx.x; i < e; i += blockDim.x) acc += (double)logp[i];
  s[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = s[0];
}

__global__ void xent_mean_kernel(const double* part, int64_t n_total, float* loss) {
  __shared__ double s[256];
  s[threadIdx.x] = (int)threadIdx.x < kXentParts ? part[threadIdx.x] : 0.0;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = (float)(-s[0] / (double)n_total);
}

__global__ void sgd_kernel(float* W, const float* dW, int64_t n, float lr) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    W[i] = __fsub_rn(W[i], __fmul_rn(lr, dW[i]));  // W - lr * g
}

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
__global__ void finite_kernel(const T* X, int64_t rows, int64_t cols, int64_t ld, int32_t* flag) {
  const int64_t total = rows * cols;
  int bad = 0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const float v = to_f<T>(X[(t / cols) * ld + t % cols]);
    bad |= !isfinite(v);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

__global__ void ewise_kernel(int op, int64_t rows, int64_t cols, const float* a, int64_t lda,
                             const float* b, int64_t b_rows, int64_t b_cols, int64_t ldb, float* out,
                             int64_t ldo) {
  const int64_t total = rows * cols;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / cols, c = t % cols;
    const float x = a[r * lda + c];
    float y = 0.f, w = 0.f;
    if (op <= 4 || op >= 8) w = b[(b_rows == 1 ? 0 : r) * ldb + (b_cols == 1 ? 0 : c)];
    switch (op) {  // tensor.py:204-303
      case 0: y = __fadd_rn(x, w); break;
      case 1: y = __fsub_rn(x, w); break;
      case 2: y = __fmul_rn(x, w); break;
      case 3: y = __fdiv_rn(x, w); break;
      case 4: y = x >= w ? x : w; break;
      case 5: y = __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-x))); break;
      case 6: y = tanhf(x); break;
      case 7: y = sg::relu_np(x); break;
      case 8: y = __fmul_rn(x, w > 0.f ? 1.f : 0.f); break;  // relu bwd: g * (z > 0)
      case 9: y = __fmul_rn(__fmul_rn(x, w), __fsub_rn(1.0f, w)); break;  // sigmoid bwd g*y*(1-y)
      default: y = __fmul_rn(x, __fsub_rn(1.0f, __fmul_rn(w, w))); break;  // tanh bwd g*(1-y*y)
    }
    out[r * ldo + c] = y;
  }
}

// Backward of the binary ops (tensor.py:255-265), both partials in one pass over the full
// [rows, cols] shape: x is a (already expanded by the caller), w is b with its broadcast.  The
// reductions of _reduce_to (tensor.py:191-201) run afterwards in reduce_*_kernel.
__global__ void ewise_bwd_kernel(int op, int64_t rows, int64_t cols, const float* g, int64_t ldg,
                                 const float* a, int64_t lda, const float* b, int64_t b_rows,
                                 int64_t b_cols, int64_t ldb, float* ga, int64_t ldga, float* gb,
                                 int64_t ldgb) {
  const int64_t total = rows * cols;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / cols, c = t % cols;
    const float gv = g[r * ldg + c];
    const float x = a[r * lda + c];
    const float w = b[(b_rows == 1 ? 0 : r) * ldb + (b_cols == 1 ? 0 : c)];
    float u, v;
    switch (op) {
      case 0: u = gv; v = gv; break;                                   // add
      case 1: u = gv; v = -gv; break;                                  // sub
      case 2: u = __fmul_rn(gv, w); v = __fmul_rn(gv, x); break;       // mul
      case 3:                                                          // div: g/w, -g*x/(w*w)
        u = __fdiv_rn(gv, w);
        v = __fdiv_rn(__fmul_rn(-gv, x), __fmul_rn(w, w));
        break;
      default: {                                                       // max: ties -> a
        const bool m = x >= w;
        u = __fmul_rn(gv, m ? 1.f : 0.f);
        v = __fmul_rn(gv, m ? 0.f : 1.f);
      }
    }
    ga[r * ldga + c] = u;
    gb[r * ldgb + c] = v;
  }
}

// out[r] = sum_c X[r, c] (the "row-scalar side" of _reduce_to, tensor.py:201): one warp per
// row, lanes stride the columns, fixed shuffle tree -- deterministic.
__global__ void reduce_cols_kernel(const float* X, int64_t ld, int64_t rows, int64_t cols, float* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nwarps) {
    float acc = 0.f;
    for (int64_t c = lane; c < cols; c += 32) acc = __fadd_rn(acc, X[r * ld + c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
    if (lane == 0) out[r] = acc;
  }
}

// Leading-axis reduction (tensor.py:197-198, g.sum over the broadcast rows) in two fixed-order
// passes: kRedParts row ranges -> partial[kRedParts, cols], then the partials in order.
constexpr int kRedParts = 148;

__global__ void reduce_rows_partial_kernel(const float* X, int64_t ld, int64_t rows, int64_t cols,
                                           float* part) {
  const int64_t chunk = (rows + kRedParts - 1) / kRedParts;
  const int64_t r0 = (int64_t)blockIdx.y * chunk, r1 = min(rows, r0 + chunk);
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cols;
       c += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int64_t r = r0; r < r1; ++r) acc = __fadd_rn(acc, X[r * ld + c]);
    part[(int64_t)blockIdx.y * cols + c] = acc;
  }
}

__global__ void reduce_rows_final_kernel(const float* part, int64_t cols, float* out) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < cols;
       c += (int64_t)gridDim.x * blockDim.x) {
    float acc = 0.f;
    for (int p = 0; p < kRedParts; ++p) acc = __fadd_rn(acc, part[(int64_t)p * cols + c]);
    out[c] = acc;
  }
}

template <typename S, typename D>
__device__ __forceinline__ D cvt(S v);
template <>
__device__ __forceinline__ float cvt<float, float>(float v) { return v; }
template <>
__device__ __forceinline__ __nv_bfloat16 cvt<float, __nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
template <>
__device__ __forceinline__ float cvt<__nv_bfloat16, float>(__nv_bfloat16 v) { return __bfloat162float(v); }
template <>
__device__ __forceinline__ __nv_bfloat16 cvt<__nv_bfloat16, __nv_bfloat16>(__nv_bfloat16 v) { return v; }

template <typename S, typename D>
__global__ void convert_kernel(const S* X, int64_t ldx, D* Y, int64_t ldy, int64_t rows, int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = t / cols, c = t % cols;
    Y[r * ldy + c] = cvt<S, D>(X[r * ldx + c]);
  }
}

#define SG_LAUNCH_CHECK(what)                                                  \
  do {                                                                         \
    cudaError_t e_ = cudaGetLastError();                                       \
    if (e_ != cudaSuccess) SG_FAIL(SG_ECUDA, "%s: %s", what, cudaGetErrorString(e_)); \
  } while (0)

}  // namespace

extern "C" {

int64_t sg_xent_workspace_bytes(int64_t n) {
  return (std::max<int64_t>(n, 1) * 4 + 255) / 256 * 256 + kXentParts * 8;
}

int sg_softmax_xent(const float* Z, int64_t ldz, int relu_input, const int64_t* labels, int64_t n,
                    int64_t C, int64_t n_total, float* loss, float* dZ, int64_t lddz,
                    int32_t* err_flag, void* workspace, int64_t workspace_bytes, void* stream) {
  if (n_total <= 0) n_total = n;
  SG_REQUIRE(n >= 1 && C >= 1, SG_ESHAPE, "logits must be [n, classes] with n, classes >= 1");
  SG_REQUIRE(workspace_bytes >= sg_xent_workspace_bytes(n), SG_EBUDGET, "xent workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  float* logp = (float*)workspace;
  xent_rows_kernel<<<grid_for(n * 32, 256), 256, 0, st>>>(Z, ldz, relu_input, labels, n, C, n_total,
                                                         dZ, lddz, logp, err_flag);
  SG_LAUNCH_CHECK("xent rows");
  double* part = reinterpret_cast<double*>(static_cast<char*>(workspace) +
                                           (std::max<int64_t>(n, 1) * 4 + 255) / 256 * 256);
  xent_partial_kernel<<<kXentParts, 256, 0, st>>>(logp, n, part);
  SG_LAUNCH_CHECK("xent partial");
  xent_mean_kernel<<<1, 256, 0, st>>>(part, n_total, loss);
  SG_LAUNCH_CHECK("xent mean");
  sg::count_launch(3);
  return SG_OK;
}

int sg_sgd(float* W, const float* dW, int64_t n, float lr, void* stream) {
  if (n == 0) return SG_OK;
  sgd_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(W, dW, n, lr);
  SG_LAUNCH_CHECK("sgd");
  sg::count_launch(1);
  return SG_OK;
}

int sg_check_finite(int dtype, const void* X, int64_t rows, int64_t cols, int64_t ld, int32_t* flag,
                    void* stream) {
  if (rows == 0 || cols == 0) return SG_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int g = grid_for(rows * cols, 256);
  if (dtype == SG_F32)
    finite_kernel<float><<<g, 256, 0, st>>>((const float*)X, rows, cols, ld, flag);
  else
    finite_kernel<__nv_bfloat16><<<g, 256, 0, st>>>((const __nv_bfloat16*)X, rows, cols, ld, flag);
  SG_LAUNCH_CHECK("check_finite");
  sg::count_launch(1);
  return SG_OK;
}

int sg_ewise(int op, int64_t rows, int64_t cols, const float* a, int64_t lda, const float* b,
             int64_t b_rows, int64_t b_cols, int64_t ldb, float* out, int64_t ldo, void* stream) {
  SG_REQUIRE(op >= 0 && op <= 10, SG_EINVAL, "ewise: unknown op %d", op);
  SG_REQUIRE((op > 4 && op < 8) || b, SG_EINVAL, "ewise: binary op needs b");
  if (rows == 0 || cols == 0) return SG_OK;
  ewise_kernel<<<grid_for(rows * cols, 256), 256, 0, (cudaStream_t)stream>>>(
      op, rows, cols, a, lda, b, b_rows, b_cols, ldb, out, ldo);
  SG_LAUNCH_CHECK("ewise");
  sg::count_launch(1);
  return SG_OK;
}

int sg_ewise_bwd(int op, int64_t rows, int64_t cols, const float* g, int64_t ldg, const float* a,
                 int64_t lda, const float* b, int64_t b_rows, int64_t b_cols, int64_t ldb, float* ga,
                 int64_t ldga, float* gb, int64_t ldgb, void* stream) {
  SG_REQUIRE(op >= 0 && op <= 4, SG_EINVAL, "ewise_bwd: unknown binary op %d", op);
  SG_REQUIRE(g && a && b && ga && gb, SG_EINVAL, "ewise_bwd: null operand");
  if (rows == 0 || cols == 0) return SG_OK;
  ewise_bwd_kernel<<<grid_for(rows * cols, 256), 256, 0, (cudaStream_t)stream>>>(
      op, rows, cols, g, ldg, a, lda, b, b_rows, b_cols, ldb, ga, ldga, gb, ldgb);
  SG_LAUNCH_CHECK("ewise_bwd");
  sg::count_launch(1);
  return SG_OK;
}

int64_t sg_reduce_workspace_bytes(int64_t cols) { return (int64_t)kRedParts * std::max<int64_t>(cols, 1) * 4; }

int sg_reduce_sum(int axis, const float* X, int64_t ld, int64_t rows, int64_t cols, float* out,
                  void* workspace, int64_t workspace_bytes, void* stream) {
  SG_REQUIRE(axis == 0 || axis == 1, SG_EINVAL, "reduce_sum: axis must be 0 or 1");
  cudaStream_t st = (cudaStream_t)stream;
  if (axis == 1) {
    if (rows == 0) return SG_OK;
    if (cols == 0) return cudaMemsetAsync(out, 0, rows * 4, st) == cudaSuccess ? SG_OK : SG_ECUDA;
    reduce_cols_kernel<<<grid_for(rows * 32, 256), 256, 0, st>>>(X, ld, rows, cols, out);
    SG_LAUNCH_CHECK("reduce_sum cols");
    sg::count_launch(1);
    return SG_OK;
  }
  if (cols == 0) return SG_OK;
  SG_REQUIRE(workspace_bytes >= sg_reduce_workspace_bytes(cols), SG_EBUDGET, "reduce workspace too small");
  float* part = (float*)workspace;
  dim3 g1((unsigned)std::min<int64_t>((cols + 127) / 128, 64), kRedParts);
  reduce_rows_partial_kernel<<<g1, 128, 0, st>>>(X, ld, rows, cols, part);
  SG_LAUNCH_CHECK("reduce_sum rows partial");
  reduce_rows_final_kernel<<<grid_for(cols, 128), 128, 0, st>>>(part, cols, out);
  SG_LAUNCH_CHECK("reduce_sum rows final");
  sg::count_launch(2);
  return SG_OK;
}

int sg_convert(int sdt, int ddt, const void* X, int64_t ldx, void* Y, int64_t ldy, int64_t rows,
               int64_t cols, void* stream) {
  if (rows == 0 || cols == 0) return SG_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int g = grid_for(rows * cols, 256);
  if (sdt == SG_F32 && ddt == SG_BF16)
    convert_kernel<float, __nv_bfloat16><<<g, 256, 0, st>>>((const float*)X, ldx, (__nv_bfloat16*)Y, ldy, rows, cols);
  else if (sdt == SG_BF16 && ddt == SG_F32)
    convert_kernel<__nv_bfloat16, float><<<g, 256, 0, st>>>((const __nv_bfloat16*)X, ldx, (float*)Y, ldy, rows, cols);
  else if (sdt == SG_F32)
    convert_kernel<float, float><<<g, 256, 0, st>>>((const float*)X, ldx, (float*)Y, ldy, rows, cols);
  else
    convert_kernel<__nv_bfloat16, __nv_bfloat16><<<g, 256, 0, st>>>((const __nv_bfloat16*)X, ldx, (__nv_bfloat16*)Y, ldy, rows, cols);
  SG_LAUNCH_CHECK("convert");
  sg::count_launch(1);
  return SG_OK;
}

}  // extern "C"
