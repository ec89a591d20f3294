// Minimal, correct TMA-ring pattern (the one the loss kernels use): a
// producer thread refills a shared-memory slot with cp.async.bulk once the
// consumer warp has released it through an "empty" mbarrier; the consumer
// reads the slot after waiting on the "full" mbarrier (complete_tx). Run it
// under `compute-sanitizer --tool racecheck` to see whether racecheck models
// mbarrier-ordered async-proxy writes (it reports the same TMA-write /
// shared-load hazard class as on the loss kernels if it does not).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n"
               ::"r"(bar), "r"(par) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}

template <bool FENCE>
__global__ void ring(const uint4* in, float* out, int iters) {
  __shared__ __align__(128) uint4 slot[256];  // 4 KB
  __shared__ __align__(8) uint64_t full, empty;
  const uint32_t fb = smem_u32(&full), eb = smem_u32(&empty), sb = smem_u32(slot);
  if (threadIdx.x == 0) {
    mbar_init(fb, 1);
    mbar_init(eb, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 32) {  // producer
    for (int i = 0; i < iters; ++i) {
      mbar_wait(eb, (i & 1) ^ 1);
      mbar_expect(fb, sizeof(slot));
      bulk_g2s(sb, in + i * 256, sizeof(slot), fb);
    }
  } else if (threadIdx.x < 32) {  // consumer warp
    float acc = 0.f;
    for (int i = 0; i < iters; ++i) {
      mbar_wait(fb, i & 1);
      for (int j = threadIdx.x; j < 256; j += 32) acc += __uint_as_float(slot[j].x);
      // generic-proxy reads ordered before the async-proxy refill
      if (FENCE) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (threadIdx.x == 0) mbar_arrive(eb);
    }
    out[threadIdx.x] = acc;
  }
}

int main(int argc, char** argv) {
  const int iters = 4;
  uint4* in;
  float* out;
  cudaMalloc(&in, iters * 256 * sizeof(uint4));
  cudaMemset(in, 0, iters * 256 * sizeof(uint4));
  cudaMalloc(&out, 32 * sizeof(float));
  // argv[1] == "fence": consumers fence.proxy.async before releasing the slot
  const bool fence = argc > 1 && argv[1][0] == 'f';
  if (fence) ring<true><<<1, 64>>>(in, out, iters);
  else ring<false><<<1, 64>>>(in, out, iters);
  cudaError_t e = cudaDeviceSynchronize();
  printf("ring (%s): %s\n", fence ? "fence.proxy.async on release" : "mbarrier only", cudaGetErrorString(e));
  return e == cudaSuccess ? 0 : 1;
}
