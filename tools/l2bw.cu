// L2 -> SM read-bandwidth probe (the ceiling of the L2-resident propagation passes).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2bw tools/l2bw.cu && tools/l2bw
// Each warp reads random 16-B-per-lane rows (like the gather) from a buffer that fits in
// L2 (hit rate ~100%) or is far larger than L2 (DRAM); prints GB/s for row sizes 512 B
// (F = 128 fp32) and 2432 B (F = 602 fp32, ld 608).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void gather_rows(const float4* __restrict__ buf, int64_t rows, int vec_per_row,
                            int iters, uint64_t seed, float* out) {
  const int lane = threadIdx.x & 31;
  uint32_t s = (uint32_t)(seed * 2654435761u) ^ (blockIdx.x * 0x9E3779B9u) ^ ((threadIdx.x >> 5) * 0x85EBCA6Bu) | 1u;
  float4 acc = make_float4(0, 0, 0, 0);
  for (int it = 0; it < iters; it += 4) {
    int64_t r[4];
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      s ^= s << 13; s ^= s >> 17; s ^= s << 5;  // xorshift32, warp-uniform
      r[d] = (int64_t)__umulhi(s, (uint32_t)rows);
    }
    float4 v[4][8];
#pragma unroll
    for (int d = 0; d < 4; ++d)
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k * 32 + lane < vec_per_row) v[d][k] = __ldg(buf + r[d] * vec_per_row + k * 32 + lane);
#pragma unroll
    for (int d = 0; d < 4; ++d)
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (k * 32 + lane < vec_per_row) {
          acc.x += v[d][k].x; acc.y += v[d][k].y; acc.z += v[d][k].z; acc.w += v[d][k].w;
        }
  }
  if (acc.x == 12345.f) out[0] = acc.y + acc.z + acc.w;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
  cudaMalloc(&out, 16);
  for (int64_t bytes : {int64_t(48) << 20, int64_t(4) << 30}) {
    float4* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0, bytes);
    for (int vpr : {32, 152}) {
      const int64_t rows = bytes / (vpr * 16);
      for (int warps_per_sm : {16, 32, 48}) {
        const int threads = 256, blocks = sms * warps_per_sm / 8, iters = 512;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        gather_rows<<<blocks, threads>>>(buf, rows, vpr, 64, 1, out);
        cudaEventRecord(a);
        gather_rows<<<blocks, threads>>>(buf, rows, vpr, iters, 2, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double moved = (double)blocks * (threads / 32) * iters * vpr * 16;
        printf("{\"buffer_MB\": %lld, \"row_bytes\": %d, \"warps_per_sm\": %d, \"GBps\": %.0f}\n",
               (long long)(bytes >> 20), vpr * 16, warps_per_sm, moved / ms / 1e6);
      }
    }
    cudaFree(buf);
  }
  return 0;
}
