// Microbenchmarks for the roofline model of the fused kernel (B200):
//  1. MUFU.EX2 throughput per SM (independent chains, all warps busy)
//  2. a streaming read bf16 -> 2 x ex2 per element -> write bf16 kernel with no
//     row-level synchronisation: the compute+memory ceiling the fused kernel
//     could reach if its per-row sync were free.
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

__global__ void mufu_kernel(float* out, int iters) {
  float a[8];
  for (int j = 0; j < 8; ++j) a[j] = -0.001f * (threadIdx.x + j);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = ex2(a[j]) - 1.0f;
  }
  float s = 0; for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 12345.f) out[0] = s;
}

__global__ void stream_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, int64_t n, float m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint4 v = in[i];
    uint32_t w[4] = {v.x, v.y, v.z, v.w};
    float s = 0.f;
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      float lo = __uint_as_float(w[k] << 16), hi = __uint_as_float(w[k] & 0xffff0000u);
      float e0 = ex2((lo - m) * 1.4426950f), e1 = ex2((hi - m) * 1.4426950f);   // pass-B exp
      s += e0 + e1;
      float p0 = ex2((lo - m) * 1.4426950f - 0.5f), p1 = ex2((hi - m) * 1.4426950f - 0.5f);  // pass-C exp
      __nv_bfloat162 b = __floats2bfloat162_rn(p0 * 0.001f + s * 1e-30f, p1 * 0.001f);
      o[k] = *reinterpret_cast<uint32_t*>(&b);
    }
    out[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

__global__ void copy_kernel(const uint4* __restrict__ in, uint4* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) out[i] = in[i];
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* d; cudaMalloc(&d, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 4096;
  mufu_kernel<<<sms * 4, 512>>>(d, iters);
  cudaEventRecord(a); mufu_kernel<<<sms * 4, 512>>>(d, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = (double)sms * 4 * 512 * iters * 8;
  printf("MUFU.EX2: %.3f Tops/s = %.2f per clk per SM at %d MHz (clock attr)\n", ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  int64_t bytes = 8LL << 30;  // 8 GiB each way
  int64_t n = bytes / 16;
  uint4 *in, *out; cudaMalloc(&in, bytes); cudaMalloc(&out, bytes); cudaMemset(in, 0, bytes);
  for (int rep = 0; rep < 2; ++rep) {
    copy_kernel<<<sms * 8, 512>>>(in, out, n);
    cudaEventRecord(a); copy_kernel<<<sms * 8, 512>>>(in, out, n); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("copy: %.1f GB/s (read+write)\n", 2.0 * bytes / ms / 1e6);
    stream_kernel<<<sms * 8, 512>>>(in, out, n, 1.0f);
    cudaEventRecord(a); stream_kernel<<<sms * 8, 512>>>(in, out, n, 1.0f); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("stream 2xex2/elem: %.1f GB/s (read+write), %.2f Gelem/s\n", 2.0 * bytes / ms / 1e6, n * 8.0 / ms / 1e6);
  }
  return 0;
}
