// reduce.cuh — deterministic reduction of the per-token loss outputs (obj,
// flags) into out4 = {objective, tokens, stale, clipped}, shared by
// reduce_kernel and one CTA of every small fused loss launch (kernels.cu: the
// last CTA to exit; pair.cu: the CTA whose scalar warp completes the launch's
// scalar phases). Reference: grpo.hpp:113-115,183 (one ordered fp64 accumulation);
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
  unsigned int rows_done;     // pair family: clusters whose rows have all written obj/flags
  unsigned int claims_failed; // pair family: clusters whose row claim has come back empty
};

__host__ __device__ inline int64_t reduce_tile(int64_t n) {
  const int64_t per = (n + kReduceMaxTiles - 1) / kReduceMaxTiles;
  const int64_t t = (per + 1023) / 1024 * 1024;
  return t < 1024 ? 1024 : t;
}

// Shared memory of the 256-thread trees: one slot per warp, plus the tile
// partials of the in-CTA path (at most kFuseReduceTiles tiles).
struct ReduceSmem {
  double o[kReduceThreads / 32];
  unsigned long long s[kReduceThreads / 32], c[kReduceThreads / 32], m[kReduceThreads / 32];
  double po[kFuseReduceTiles];
  unsigned long long ps[kFuseReduceTiles], pc[kFuseReduceTiles];
};

// Fixed-order tree over the 256 participating threads (named barrier 1: the
// caller's CTA may have more threads; those do not take part): a shuffle
// butterfly inside each warp (a + b == b + a exactly, so every lane holds the
// same bits), the 8 warp results through shared memory, the same butterfly in
// warp 0. The result is valid in thread 0. Two barriers instead of a
// shared-memory tree's nine: the reduction is on the tail of every small step.
template <bool FOUR>
__device__ __forceinline__ void reduce_tree(ReduceSmem& sm, int tid, double& o, unsigned long long& s,
                                            unsigned long long& c, unsigned long long& m) {
  constexpr unsigned kAll = 0xffffffffu;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    o += __shfl_xor_sync(kAll, o, off);
    s += __shfl_xor_sync(kAll, s, off);
    c += __shfl_xor_sync(kAll, c, off);
    if (FOUR) m += __shfl_xor_sync(kAll, m, off);
  }
  const int w = tid >> 5, lane = tid & 31;
  if (lane == 0) {
    sm.o[w] = o;
    sm.s[w] = s;
    sm.c[w] = c;
    if (FOUR) sm.m[w] = m;
  }
  ptx::named_bar_sync(1, kReduceThreads);
  if (w == 0) {
    constexpr int NW = kReduceThreads / 32;
    o = lane < NW ? sm.o[lane] : 0.0;
    s = lane < NW ? sm.s[lane] : 0ull;
    c = lane < NW ? sm.c[lane] : 0ull;
    if (FOUR) m = lane < NW ? sm.m[lane] : 0ull;
#pragma unroll
    for (int off = NW / 2; off > 0; off >>= 1) {
      o += __shfl_xor_sync(kAll, o, off);
      s += __shfl_xor_sync(kAll, s, off);
      c += __shfl_xor_sync(kAll, c, off);
      if (FOUR) m += __shfl_xor_sync(kAll, m, off);
    }
  }
  ptx::named_bar_sync(1, kReduceThreads);  // sm is reused by the next tree
}

// Partial of tile `k` (tokens [k tile, min(n, (k+1) tile))) by threads 0..255;
// valid in thread 0. VEC: obj 16-byte and flags 4-byte aligned.
template <bool VEC>
__device__ __forceinline__ void reduce_tile_partial(const double* __restrict__ obj,
                                                    const uint8_t* __restrict__ flags, int64_t n,
                                                    int64_t tile, int64_t k, ReduceSmem& sm, int tid,
                                                    double& po, unsigned long long& ps,
                                                    unsigned long long& pc) {
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
  unsigned long long sv = st | (mk << 32), unused = 0;
  reduce_tree<false>(sm, tid, o, sv, cl, unused);
  po = o;
  ps = sv;
  pc = cl;
}

// The final sum over the tile partials (fixed order: thread i takes partials
// i, i + 256, ... starting from 0, then the tree) -> out4. `part(i, o, s, c)`
// yields partial i (global scratch in reduce_kernel, shared memory in the
// in-CTA path: the same values, so the same bits).
template <typename Part>
__device__ __forceinline__ void reduce_final(int64_t n, int64_t ntiles, double* __restrict__ out4,
                                             ReduceSmem& sm, int tid, Part part) {
  double O = 0.0;
  unsigned long long Sx = 0, Cx = 0, Mx = 0;
  for (int64_t i = tid; i < ntiles; i += kReduceThreads) {
    double po;
    unsigned long long ps, pc;
    part(i, po, ps, pc);
    O += po;
    Sx += ps & 0xFFFFFFFFull;
    Mx += ps >> 32;
    Cx += pc;
  }
  reduce_tree<true>(sm, tid, O, Sx, Cx, Mx);
  if (tid == 0) {
    out4[0] = O;
    out4[1] = static_cast<double>(n - static_cast<int64_t>(Mx));
    out4[2] = static_cast<double>(Sx);
    out4[3] = static_cast<double>(Cx);
  }
}

// Partials in the global scratch (reduce_kernel: written by other blocks).
__device__ __forceinline__ void scratch_part(const ReduceScratch* sc, int64_t i, double& o,
                                             unsigned long long& s, unsigned long long& c) {
  o = *reinterpret_cast<const volatile double*>(&sc->obj[i]);
  s = *reinterpret_cast<const volatile unsigned long long*>(&sc->stale[i]);
  c = *reinterpret_cast<const volatile unsigned long long*>(&sc->clipped[i]);
}

// All tiles by one CTA (threads 0..255 of it), partials kept in shared memory,
// then the final sum: the last CTA of a fused loss launch (<= kFuseReduceTiles).
template <bool VEC>
__device__ __forceinline__ void reduce_all_in_cta(const double* obj, const uint8_t* flags, int64_t n,
                                                  double* out4, ReduceSmem& sm, int tid) {
  const int64_t tile = reduce_tile(n), ntiles = (n + tile - 1) / tile;
  for (int64_t k = 0; k < ntiles; ++k) {
    double po;
    unsigned long long ps, pc;
    reduce_tile_partial<VEC>(obj, flags, n, tile, k, sm, tid, po, ps, pc);
    if (tid == 0) {
      sm.po[k] = po;
      sm.ps[k] = ps;
      sm.pc[k] = pc;
    }
  }
  ptx::named_bar_sync(1, kReduceThreads);
  reduce_final(n, ntiles, out4, sm, tid, [&](int64_t i, double& o, unsigned long long& s,
                                             unsigned long long& c) {
    o = sm.po[i];
    s = sm.ps[i];
    c = sm.pc[i];
  });
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
  // every thread's stores (the per-token outputs) are ordered before thread 0's
  // release fence by the barrier (fence cumulativity), as in a grid barrier
  __syncthreads();
  auto* sc = static_cast<ReduceScratch*>(P.red_scratch);
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&sc->fused_ticket, 1u) == gridDim.x - 1;
    if (last) {
      __threadfence();  // acquire: the other CTAs' outputs, before this CTA reads them
      if (reset_ctr) *P.row_ctr = 0ull;  // every CTA has made its last claim
      sc->fused_ticket = 0;
    }
  }
  __syncthreads();
  if (!last || !P.out4 || threadIdx.x >= kReduceThreads) return;
  ReduceSmem& sm = *static_cast<ReduceSmem*>(sm_raw);
  const bool vec = (reinterpret_cast<uintptr_t>(P.obj) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(P.flags) % 4 == 0);
  if (vec)
    reduce_all_in_cta<true>(P.obj, P.flags, P.red_n, P.out4, sm, threadIdx.x);
  else
    reduce_all_in_cta<false>(P.obj, P.flags, P.red_n, P.out4, sm, threadIdx.x);
}

__device__ __forceinline__ void fused_reduce_if_last(const LossParams& P, void* sm_raw) {
  end_of_launch(P, sm_raw, false);
}

}  // namespace
}  // namespace copris_b200
