// reduce.cuh — deterministic reduction of the per-token loss outputs (obj,
// flags) into out4 = {objective, tokens, stale, clipped}, shared by
// reduce_kernel and the last CTA of every fused loss launch (kernels.cu,
// pair.cu). Reference: grpo.hpp:113-115,183 (one ordered fp64 accumulation);
// here a fixed tile partition and fixed-order trees, so reruns and chunkings
// are bitwise identical and no floating-point atomics are used.
#pragma once

#include <cstdint>

#include "kernels.cuh"
#include "ptx.cuh"
#include "token_math.cuh"

namespace copris_b200 {
namespace {

// Deterministic reduction of the per-token outputs (obj, flags) of a batch.
// The token range is cut into TILES whose size depends on n only
// (reduce_tile); each tile's partial is formed by 256 threads in a fixed order
// (4-token quads, then a fixed tree), and the final result sums the tile
// partials in a fixed order (thread i takes partials i, i + 256, ..., then the
// same tree). The same device code runs in reduce_kernel (blocks take tiles
// b, b + nb, ...; the last block to finish sums) and in the last CTA of a
// fused loss launch (it takes every tile): both give bitwise the same out4,
// and any rerun is bitwise identical. No floating-point atomics.
constexpr int kReduceBlocks = 512;
constexpr int kReduceThreads = 256;
constexpr int kReduceMaxTiles = 8192;
constexpr int kFuseReduceTiles = 8;  // fused into the loss launch up to 8 tiles (8,192 tokens)
struct ReduceScratch {
  double obj[kReduceMaxTiles];
  unsigned long long stale[kReduceMaxTiles];  // stale | masked << 32
  unsigned long long clipped[kReduceMaxTiles];
  unsigned int ticket;        // reduce_kernel blocks done
  unsigned int fused_ticket;  // fused-launch CTAs done
};

__host__ __device__ inline int64_t reduce_tile(int64_t n) {
  const int64_t per = (n + kReduceMaxTiles - 1) / kReduceMaxTiles;
  const int64_t t = (per + 1023) / 1024 * 1024;
  return t < 1024 ? 1024 : t;
}

// Shared-memory arrays of the 256-thread trees.
struct ReduceSmem {
  double o[kReduceThreads];
  unsigned long long s[kReduceThreads], c[kReduceThreads], m[kReduceThreads];
};

// Tree over the 256 participating threads (named barrier 1: the caller's CTA
// may have more threads; those do not take part).
__device__ __forceinline__ void reduce_tree(ReduceSmem& sm, int tid, bool four) {
  ptx::named_bar_sync(1, kReduceThreads);
  for (int h = kReduceThreads / 2; h > 0; h >>= 1) {
    if (tid < h) {
      sm.o[tid] += sm.o[tid + h];
      sm.s[tid] += sm.s[tid + h];
      sm.c[tid] += sm.c[tid + h];
      if (four) sm.m[tid] += sm.m[tid + h];
    }
    ptx::named_bar_sync(1, kReduceThreads);
  }
}

// Partial of tile `k` (tokens [k tile, min(n, (k+1) tile))) by threads 0..255,
// written to sc by thread 0. VEC: obj 16-byte and flags 4-byte aligned.
template <bool VEC>
__device__ __forceinline__ void reduce_tile_partial(const double* __restrict__ obj,
                                                    const uint8_t* __restrict__ flags, int64_t n,
                                                    int64_t tile, int64_t k, ReduceScratch* sc,
                                                    ReduceSmem& sm, int tid) {
  const int64_t t0 = k * tile, t1 = min(n, t0 + tile);
  double o = 0.0;
  unsigned long long st = 0, cl = 0, mk = 0;
  auto tally = [&](uint32_t f) {
    st += f & FLAG_STALE;
    cl += (f >> 1) & 1u;
    mk += (f >> 2) & 1u;
  };
  if constexpr (VEC) {
    const int64_t q1 = t0 + ((t1 - t0) & ~int64_t{3});  // end of whole quads
    for (int64_t t = t0 + 4 * tid; t < q1; t += 4 * kReduceThreads) {
      const double2 a0 = *reinterpret_cast<const double2*>(obj + t);
      const double2 a1 = *reinterpret_cast<const double2*>(obj + t + 2);
      const uint32_t fa = *reinterpret_cast<const uint32_t*>(flags + t);
      o += (a0.x + a0.y) + (a1.x + a1.y);
      tally(fa & 0xFFu); tally((fa >> 8) & 0xFFu); tally((fa >> 16) & 0xFFu); tally(fa >> 24);
    }
    for (int64_t u = q1 + tid; u < t1; u += kReduceThreads) {
      o += obj[u];
      tally(flags[u]);
    }
  } else {
    for (int64_t t = t0 + tid; t < t1; t += kReduceThreads) {
      o += obj[t];
      tally(flags[t]);
    }
  }
  // stale/clipped counts < 2^32 per tile: pack the masked count with stale
  sm.o[tid] = o;
  sm.s[tid] = st | (mk << 32);
  sm.c[tid] = cl;
  reduce_tree(sm, tid, false);
  if (tid == 0) {
    sc->obj[k] = sm.o[0];
    sc->stale[k] = sm.s[0];
    sc->clipped[k] = sm.c[0];
  }
  ptx::named_bar_sync(1, kReduceThreads);  // sm is reused by the next tile
}

// The final sum over the tile partials (fixed order) -> out4; resets tickets.
__device__ __forceinline__ void reduce_final(int64_t n, int64_t ntiles, double* __restrict__ out4,
                                             ReduceScratch* sc, ReduceSmem& sm, int tid) {
  double O = 0.0;
  unsigned long long Sx = 0, Cx = 0, Mx = 0;
  for (int64_t i = tid; i < ntiles; i += kReduceThreads) {
    O += *reinterpret_cast<volatile double*>(&sc->obj[i]);
    const unsigned long long sm2 = *reinterpret_cast<volatile unsigned long long*>(&sc->stale[i]);
    Sx += sm2 & 0xFFFFFFFFull;
    Mx += sm2 >> 32;
    Cx += *reinterpret_cast<volatile unsigned long long*>(&sc->clipped[i]);
  }
  sm.o[tid] = O;
  sm.s[tid] = Sx;
  sm.c[tid] = Cx;
  sm.m[tid] = Mx;
  reduce_tree(sm, tid, true);
  if (tid == 0) {
    out4[0] = sm.o[0];
    out4[1] = static_cast<double>(n - static_cast<int64_t>(sm.m[0]));
    out4[2] = static_cast<double>(sm.s[0]);
    out4[3] = static_cast<double>(sm.c[0]);
    sc->ticket = 0;
    sc->fused_ticket = 0;
  }
}

// All tiles by one CTA (threads 0..255 of it), then the final sum: the last
// CTA of a fused loss launch (fused_reduce_if_last).
template <bool VEC>
__device__ __forceinline__ void reduce_all_in_cta(const double* obj, const uint8_t* flags, int64_t n,
                                                  double* out4, ReduceScratch* sc, ReduceSmem& sm,
                                                  int tid) {
  const int64_t tile = reduce_tile(n), ntiles = (n + tile - 1) / tile;
  for (int64_t k = 0; k < ntiles; ++k) reduce_tile_partial<VEC>(obj, flags, n, tile, k, sc, sm, tid);
  reduce_final(n, ntiles, out4, sc, sm, tid);
}

// Whether a launch over p.red_n tokens reduces in its last CTA (<= 8 tiles, and
// the CTA has dynamic shared memory for the trees) instead of reduce_kernel.
inline bool fuse_reduce_ok(const LossParams& p, int smem_bytes) {
  return p.out4 && p.red_scratch && smem_bytes >= static_cast<int>(sizeof(ReduceSmem)) &&
         p.red_n <= kFuseReduceTiles * reduce_tile(p.red_n);
}

// End of a fused loss launch (every CTA, after its rows' outputs are written by
// the scalar-phase thread, which fences them): the CTA counts itself done and the
// LAST one (a) resets the row-claim counter when `reset_ctr` (so the next launch —
// or a CUDA-graph replay of this one — starts at 0 without a memset node) and
// (b) with P.out4 set, reduces rows [0, P.red_n) into P.out4. `sm_raw` is shared
// memory the CTA no longer needs (>= sizeof(ReduceSmem)).
__device__ __forceinline__ void end_of_launch(const LossParams& P, void* sm_raw, bool reset_ctr) {
  __shared__ bool last;
  __threadfence();  // this thread's obj/flags stores, before the ticket
  __syncthreads();
  auto* sc = static_cast<ReduceScratch*>(P.red_scratch);
  if (threadIdx.x == 0) last = atomicAdd(&sc->fused_ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last || threadIdx.x >= kReduceThreads) return;
  __threadfence();
  if (threadIdx.x == 0) {
    if (reset_ctr) *P.row_ctr = 0ull;  // every CTA has made its last claim
    if (!P.out4) sc->fused_ticket = 0;  // else reduce_final resets it
  }
  if (!P.out4) return;
  ReduceSmem& sm = *static_cast<ReduceSmem*>(sm_raw);
  const bool vec = (reinterpret_cast<uintptr_t>(P.obj) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(P.flags) % 4 == 0);
  if (vec)
    reduce_all_in_cta<true>(P.obj, P.flags, P.red_n, P.out4, sc, sm, threadIdx.x);
  else
    reduce_all_in_cta<false>(P.obj, P.flags, P.red_n, P.out4, sc, sm, threadIdx.x);
}

__device__ __forceinline__ void fused_reduce_if_last(const LossParams& P, void* sm_raw) {
  end_of_launch(P, sm_raw, false);
}

}  // namespace
}  // namespace copris_b200
