// fused_common.cuh — device helpers shared by the fused loss kernels
// (kernels.cu: TMA / streaming / generic kernels; pair.cu: the CTA-pair
// kernel): element types, the online log-sum-exp state and its merges, row
// metadata prefetch, phase tracing and the TMA ring position. Included inside
// an anonymous namespace by each translation unit.
#pragma once

#include <cuda_bf16.h>

#include <cstdint>

#include "kernels.cuh"
#include "ptx.cuh"
#include "token_math.cuh"

namespace copris_b200 {
namespace {

// ---------------------------------------------------------------------------
// element types
// ---------------------------------------------------------------------------
template <typename T>
struct Vec;
template <>
struct Vec<__nv_bfloat16> {
  static constexpr int N = 8;  // elements per 16-byte vector
  __device__ static __forceinline__ void unpack(uint4 v, float* x) {
    x[0] = ptx::bf16_lo(v.x); x[1] = ptx::bf16_hi(v.x);
    x[2] = ptx::bf16_lo(v.y); x[3] = ptx::bf16_hi(v.y);
    x[4] = ptx::bf16_lo(v.z); x[5] = ptx::bf16_hi(v.z);
    x[6] = ptx::bf16_lo(v.w); x[7] = ptx::bf16_hi(v.w);
  }
  __device__ static __forceinline__ float load1(const void* p) {
    return __bfloat162float(*static_cast<const __nv_bfloat16*>(p));
  }
};
template <>
struct Vec<float> {
  static constexpr int N = 4;
  __device__ static __forceinline__ void unpack(uint4 v, float* x) {
    x[0] = __uint_as_float(v.x); x[1] = __uint_as_float(v.y);
    x[2] = __uint_as_float(v.z); x[3] = __uint_as_float(v.w);
  }
  __device__ static __forceinline__ float load1(const void* p) {
    return *static_cast<const float*>(p);
  }
};

__device__ __forceinline__ void store1(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }
__device__ __forceinline__ void store1(float* p, float v) { *p = v; }

// Store N floats as TOut at a 16-byte aligned address.
template <typename TOut, int N>
__device__ __forceinline__ void store_vec(TOut* p, const float* d, uint64_t pol) {
  if constexpr (sizeof(TOut) == 2) {
    static_assert(N == 8 || N == 4, "");
    if constexpr (N == 8) {
      uint4 v{ptx::pack_bf16x2(d[0], d[1]), ptx::pack_bf16x2(d[2], d[3]),
              ptx::pack_bf16x2(d[4], d[5]), ptx::pack_bf16x2(d[6], d[7])};
      ptx::st_global_v4_hint(p, v, pol);
    } else {
      uint2 v{ptx::pack_bf16x2(d[0], d[1]), ptx::pack_bf16x2(d[2], d[3])};
      *reinterpret_cast<uint2*>(p) = v;
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; j += 4) {
      uint4 v{__float_as_uint(d[j]), __float_as_uint(d[j + 1]), __float_as_uint(d[j + 2]),
              __float_as_uint(d[j + 3])};
      ptx::st_global_v4_hint(p + j, v, pol);
    }
  }
}

// ---------------------------------------------------------------------------
// online log-sum-exp state: (m, s = sum exp(z-m), u = sum exp(z-m)(z-m))
// ---------------------------------------------------------------------------
// Online log-sum-exp state of a set of columns, relative to the running max m:
//   s = sum exp(z - m) over the columns EXCEPT the target column,
//   u = sum exp(z - m)(z - m) and a = sum exp(z - m) over ALL columns
//       (entropy only; dead code otherwise).
// Keeping the target out of s lets the scalar phase add exp(z_y - m) back so
// both p_y and 1 - p_y = s/S stay accurate when the target saturates the row.
struct Lse {
  float m, s, u, a;
};

__device__ __forceinline__ Lse lse_empty() { return Lse{-INFINITY, 0.f, 0.f, 0.f}; }

template <int N, bool ENT>
__device__ __forceinline__ void online_update(const float* x, Lse& st, int jt) {
  float vm = x[0];
#pragma unroll
  for (int j = 1; j < N; ++j) vm = fmaxf(vm, x[j]);
  if (vm > st.m) {
    const float r = ptx::ex2((st.m - vm) * kLog2e);  // 0 when m = -inf
    if (ENT) {
      st.u = (st.m == -INFINITY) ? 0.f : r * fmaf(st.a, st.m - vm, st.u);
      st.a *= r;
    }
    st.s *= r;
    st.m = vm;
  }
  if (st.m == -INFINITY) return;  // every column so far is -inf (masked vocabulary): adds 0
  if (jt < 0) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const float d = x[j] - st.m;
      const float e = ptx::ex2(d * kLog2e);
      st.s += e;
      if (ENT) {
        st.u = fmaf(e, e > 0.f ? d : 0.f, st.u);  // exp(-inf) * -inf = 0, not NaN
        st.a += e;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const float d = x[j] - st.m;
      const float e = ptx::ex2(d * kLog2e);
      if (j != jt) st.s += e;
      if (ENT) {
        st.u = fmaf(e, e > 0.f ? d : 0.f, st.u);
        st.a += e;
      }
    }
  }
}

// Commutative merge (bitwise symmetric in its two operands, so a butterfly
// leaves every lane with the same value).
template <bool ENT>
__device__ __forceinline__ void lse_merge(Lse& x, const Lse& y) {
  if (y.m == -INFINITY) return;
  if (x.m == -INFINITY) {
    x = y;
    return;
  }
  const float M = fmaxf(x.m, y.m);
  const float r1 = ptx::ex2((x.m - M) * kLog2e), r2 = ptx::ex2((y.m - M) * kLog2e);
  if (ENT) {
    x.u = r1 * fmaf(x.a, x.m - M, x.u) + r2 * fmaf(y.a, y.m - M, y.u);
    x.a = x.a * r1 + y.a * r2;
  }
  x.s = x.s * r1 + y.s * r2;
  x.m = M;
}

// Butterfly over the first WIDTH lanes (a power of two); when only lanes
// [0, n) hold partials and the rest are empty, WIDTH = pow2ceil(n) gives lane 0
// the same bits as the full 32-lane butterfly (merging an empty state is a no-op).
constexpr int lse_width(int n) { return n <= 1 ? 1 : (n <= 2 ? 2 : (n <= 4 ? 4 : (n <= 8 ? 8 : (n <= 16 ? 16 : 32)))); }

template <bool ENT, int WIDTH = 32>
__device__ __forceinline__ void warp_lse(Lse& st) {
#pragma unroll
  for (int off = WIDTH / 2; off > 0; off >>= 1) {
    Lse o;
    o.m = __shfl_xor_sync(0xffffffffu, st.m, off);
    o.s = __shfl_xor_sync(0xffffffffu, st.s, off);
    o.u = ENT ? __shfl_xor_sync(0xffffffffu, st.u, off) : 0.f;
    o.a = ENT ? __shfl_xor_sync(0xffffffffu, st.a, off) : 0.f;
    lse_merge<ENT>(st, o);
  }
}

// Phase timer for COPRIS_TRACE (one thread per CTA accumulates cycle deltas).
struct PhaseTimer {
  long long acc[kTraceSlots] = {};
  long long last = 0, c0 = 0;
  unsigned long long g0 = 0;
  bool on = false;
  __device__ __forceinline__ static unsigned long long gtimer() {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    return g;
  }
  __device__ __forceinline__ void start(bool enable) {
    on = enable;
    if (on) {
      last = c0 = clock64();
      g0 = gtimer();
    }
  }
  __device__ __forceinline__ void mark(int k) {
    if (on) {
      const long long now = clock64();
      acc[k] += now - last;
      last = now;
    }
  }
  // slots 8/9: the traced thread's lifetime in ns and SM cycles
  __device__ __forceinline__ void flush(long long* trace) {
    if (on) {
      acc[8] = static_cast<long long>(gtimer() - g0);
      acc[9] = clock64() - c0;
      for (int k = 0; k < kTraceSlots; ++k) trace[blockIdx.x * kTraceSlots + k] += acc[k];
    }
  }
};

// Per-token metadata of one row, loaded by one thread early in the row.
struct RowMeta {
  int32_t y;
  uint32_t st;
  float blp, rl;
  double adv;
  bool keep;  // loss_mask[t] != 0 (true without a mask)
};

__device__ __forceinline__ RowMeta load_meta(const LossParams& P, int64_t t) {
  RowMeta m{};
  m.y = P.target[t];
  m.keep = true;
  if (P.gather_only) return m;
  m.st = P.stage[t];
  m.blp = P.buffered_lp[t];
  m.rl = P.ref_lp ? P.ref_lp[t] : 0.f;
  m.adv = P.adv[P.tok_traj[t]];
  m.keep = P.loss_mask ? P.loss_mask[t] != 0 : true;
  return m;
}

// Row metadata prefetched two rows ahead so that no load depends on a load
// issued in the same row: tok_traj of row r+2s is fetched while row r runs,
// and adv[traj] of row r+s then uses it. (A dependent tok_traj -> adv pair
// on the critical path costs a full memory round trip per row.)
struct MetaPipe {
  RowMeta next{};
  int32_t traj_ahead = 0;
  __device__ __forceinline__ void init(const LossParams& P, int64_t r, int64_t stride) {
    if (r < P.n_rows) next = load_meta(P, P.row_base + r);
    if (!P.gather_only && r + stride < P.n_rows) traj_ahead = P.tok_traj[P.row_base + r + stride];
  }
  // Returns row r's metadata and starts the loads for row r + stride.
  __device__ __forceinline__ RowMeta advance(const LossParams& P, int64_t r, int64_t stride) {
    const RowMeta cur = next;
    const int64_t r1 = r + stride;
    if (r1 < P.n_rows && P.gather_only) {
      next.y = P.target[P.row_base + r1];
    } else if (r1 < P.n_rows) {
      const int64_t t1 = P.row_base + r1;
      next.y = P.target[t1];
      next.st = P.stage[t1];
      next.blp = P.buffered_lp[t1];
      next.rl = P.ref_lp ? P.ref_lp[t1] : 0.f;
      next.adv = P.adv[traj_ahead];
      next.keep = P.loss_mask ? P.loss_mask[t1] != 0 : true;
      if (r1 + stride < P.n_rows) traj_ahead = P.tok_traj[t1 + stride];
    }
    return cur;
  }
  // The same over an explicit row sequence (rows claimed at run time): r0 and r1
  // are the first two rows, -1 past the end.
  __device__ __forceinline__ void init_ids(const LossParams& P, int64_t r0, int64_t r1) {
    if (r0 >= 0) next = load_meta(P, P.row_base + r0);
    if (!P.gather_only && r1 >= 0) traj_ahead = P.tok_traj[P.row_base + r1];
  }
  // Returns the current row's metadata; r1 = the next row, r2 = the one after.
  __device__ __forceinline__ RowMeta advance_ids(const LossParams& P, int64_t r1, int64_t r2) {
    const RowMeta cur = next;
    if (r1 >= 0 && P.gather_only) {
      next.y = P.target[P.row_base + r1];
    } else if (r1 >= 0) {
      const int64_t t1 = P.row_base + r1;
      next.y = P.target[t1];
      next.st = P.stage[t1];
      next.blp = P.buffered_lp[t1];
      next.rl = P.ref_lp ? P.ref_lp[t1] : 0.f;
      next.adv = P.adv[traj_ahead];
      next.keep = P.loss_mask ? P.loss_mask[t1] != 0 : true;
      if (r2 >= 0) traj_ahead = P.tok_traj[P.row_base + r2];
    }
    return cur;
  }
};

// dlogits for N consecutive columns starting at column c.
template <int N, bool ENT>
__device__ __forceinline__ void row_grad(const float* x, float* d, int32_t c,
                                         const RowBroadcast& b) {
#pragma unroll
  for (int j = 0; j < N; ++j) {
    const float xm = x[j] - b.m;
    const float p = ptx::ex2(fmaf(xm, kLog2e, -b.log2s));
    float v = -b.coef * p;
    if (c + j == b.y) v = b.dy;  // one-hot term: coef*(1 - p_y) (policy.hpp:193-194)
    if (ENT && p > 0.f) v = fmaf(b.eg * p, xm + b.k0, v);  // p = 0 at -inf: no entropy term
    d[j] = v;
  }
}


// Pass-B accumulation over the vectors [v, v+32) of one lane's pair: fast
// path (no entropy) with packed fp32x2 math. Each lane keeps its running max m
// and two packed partial sums; the target column (if present) is forced to
// -inf after the max so it stays out of s (see Lse).
template <typename TIn>
struct PassB;

template <>
struct PassB<__nv_bfloat16> {
  __device__ static __forceinline__ float vmax(uint4 a, uint4 b) {
    uint32_t w = ptx::bmax2(ptx::bmax2(ptx::bmax2(a.x, a.y), ptx::bmax2(a.z, a.w)),
                            ptx::bmax2(ptx::bmax2(b.x, b.y), ptx::bmax2(b.z, b.w)));
    return fmaxf(ptx::bf16_lo(w), ptx::bf16_hi(w));
  }
  __device__ static __forceinline__ void unpack2(uint4 a, uint64_t* x) {
    x[0] = ptx::bf16x2_to_f2(a.x);
    x[1] = ptx::bf16x2_to_f2(a.y);
    x[2] = ptx::bf16x2_to_f2(a.z);
    x[3] = ptx::bf16x2_to_f2(a.w);
  }
  static constexpr uint32_t kNegInfWord = 0xFF80FF80u;
};

template <>
struct PassB<float> {
  __device__ static __forceinline__ float vmax(uint4 a, uint4 b) {
    return fmaxf(fmaxf(fmaxf(__uint_as_float(a.x), __uint_as_float(a.y)),
                       fmaxf(__uint_as_float(a.z), __uint_as_float(a.w))),
                 fmaxf(fmaxf(__uint_as_float(b.x), __uint_as_float(b.y)),
                       fmaxf(__uint_as_float(b.z), __uint_as_float(b.w))));
  }
  __device__ static __forceinline__ void unpack2(uint4 a, uint64_t* x) {
    x[0] = ptx::f2(__uint_as_float(a.x), __uint_as_float(a.y));
    x[1] = ptx::f2(__uint_as_float(a.z), __uint_as_float(a.w));
  }
  static constexpr uint32_t kNegInfWord = 0xFF800000u;
};

// Position in the slot ring (slot index + phase parity), advanced without
// integer division.
struct Ring {
  uint32_t slot = 0, ph = 0, n;
  __device__ explicit Ring(uint32_t nslots) : n(nslots) {}
  __device__ __forceinline__ void next() {
    if (++slot == n) {
      slot = 0;
      ph ^= 1u;
    }
  }
};

// ---------------------------------------------------------------------------
// fused_stream_la_kernel: the streaming kernel with a one-row lookahead that
// takes the per-row scalar phase off the consumers' critical path.
//
// Segment order through the ring (producer and consumers agree on it):
//   P1(r0) | P1(r1)[0,L) P2(r0) P1(r1)[L,n) | P1(r2)[0,L) P2(r1) P1(r2)[L,n) | ...
// After pass 1 of row r the consumers hand their partials to a dedicated
// scalar warp (mbarrier p1done) and continue with the first L segments of the
// next row; the scalar warp merges the partials, runs the token math and
// publishes the row broadcast (mbarrier sdone) while they do. Rows stay in L2
// between their two passes for about one row plus L segments.
// ---------------------------------------------------------------------------
struct P1Acc {
  float m = -INFINITY, nml = -INFINITY;  // -inf until a finite column: -inf columns add 0
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  float zy = 0.f;
  bool have_zy = false;
  Lse st = lse_empty();  // entropy path
};

// Pass-1 work of one consumer thread on one ring segment.
template <typename TIn, int NC, int K, int kSlotVec, bool ENT>
__device__ __forceinline__ void p1_segment(P1Acc& a, uint32_t sb, int32_t v0, int32_t cnt,
                                           int32_t y, int tid) {
  using VI = Vec<TIn>;
  using PB = PassB<TIn>;
  constexpr int VN = VI::N;
  if constexpr (ENT) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int32_t j = tid + k * NC;
      if (j < cnt) {
        float x[VN];
        VI::unpack(ptx::lds_v4(sb + j * 16), x);
        const int jt = y - (v0 + j) * VN;
        if (static_cast<uint32_t>(jt) < VN) {
#pragma unroll
          for (int q = 0; q < VN; ++q)
            if (q == jt) a.zy = x[q];
          a.have_zy = true;
        }
        online_update<VN, true>(x, a.st, static_cast<uint32_t>(jt) < VN ? jt : -1);
      }
    }
  } else {
    const bool tseg = static_cast<uint32_t>(y - v0 * VN) < static_cast<uint32_t>(cnt * VN);
    const bool full_seg = cnt == kSlotVec;
#pragma unroll
    for (int k = 0; k < K; k += 2) {
      const int32_t ja_i = tid + k * NC, jb_i = ja_i + NC;
      uint4 va, vb;
      if (full_seg) {
        va = ptx::lds_v4(sb + ja_i * 16);
        vb = ptx::lds_v4(sb + jb_i * 16);
      } else {
        const uint4 ninf{PB::kNegInfWord, PB::kNegInfWord, PB::kNegInfWord, PB::kNegInfWord};
        va = ja_i < cnt ? ptx::lds_v4(sb + ja_i * 16) : ninf;
        vb = jb_i < cnt ? ptx::lds_v4(sb + jb_i * 16) : ninf;
      }
      const float vm = PB::vmax(va, vb);
      if (vm > a.m) {
        const float rs = ptx::ex2((a.m - vm) * kLog2e);
        a.s0 *= rs;
        a.s1 *= rs;
        a.s2 *= rs;
        a.s3 *= rs;
        a.m = vm;
        a.nml = -(a.m * kLog2e);
      }
      float xa[VN], xb[VN];
      VI::unpack(va, xa);
      VI::unpack(vb, xb);
      if (tseg) {
        const int ja = y - (v0 + ja_i) * VN, jb = y - (v0 + jb_i) * VN;
#pragma unroll
        for (int q = 0; q < VN; ++q) {
          if (q == ja) {
            a.zy = xa[q];
            a.have_zy = true;
            xa[q] = -INFINITY;
          }
          if (q == jb) {
            a.zy = xb[q];
            a.have_zy = true;
            xb[q] = -INFINITY;
          }
        }
      }
      const float nml = a.nml;
      a.s0 += ptx::ex2(fmaf(xa[0], kLog2e, nml));
      a.s1 += ptx::ex2(fmaf(xa[1], kLog2e, nml));
      a.s2 += ptx::ex2(fmaf(xb[0], kLog2e, nml));
      a.s3 += ptx::ex2(fmaf(xb[1], kLog2e, nml));
      a.s0 += ptx::ex2(fmaf(xa[2], kLog2e, nml));
      a.s1 += ptx::ex2(fmaf(xa[3], kLog2e, nml));
      a.s2 += ptx::ex2(fmaf(xb[2], kLog2e, nml));
      a.s3 += ptx::ex2(fmaf(xb[3], kLog2e, nml));
      if constexpr (VN == 8) {
        a.s0 += ptx::ex2(fmaf(xa[4], kLog2e, nml));
        a.s1 += ptx::ex2(fmaf(xa[5], kLog2e, nml));
        a.s2 += ptx::ex2(fmaf(xb[4], kLog2e, nml));
        a.s3 += ptx::ex2(fmaf(xb[5], kLog2e, nml));
        a.s0 += ptx::ex2(fmaf(xa[6], kLog2e, nml));
        a.s1 += ptx::ex2(fmaf(xa[7], kLog2e, nml));
        a.s2 += ptx::ex2(fmaf(xb[6], kLog2e, nml));
        a.s3 += ptx::ex2(fmaf(xb[7], kLog2e, nml));
      }
    }
  }
}

// Pass-2 work (dlogits) of one consumer thread on one ring segment.
template <typename TIn, typename TOut, int NC, int K, int kSlotVec, bool ENT>
__device__ __forceinline__ void p2_segment(const RowBroadcast& b, bool zero_row, uint32_t sb,
                                           int32_t v0, int32_t cnt, TOut* dseg, int tid,
                                           uint64_t pol) {
  using VI = Vec<TIn>;
  constexpr int VN = VI::N;
  const bool tseg = static_cast<uint32_t>(b.y - v0 * VN) < static_cast<uint32_t>(cnt * VN);
  if constexpr (!ENT && sizeof(TOut) == 2 && VN == 8) {
    if (!zero_row && cnt == kSlotVec) {
      // |coef| folded into the exponent and the sign applied to the packed
      // bf16 pair: d_k = -coef p_k = sign * 2^(z_k log2(e) - c2)
      const float nc2 = -b.c2;
      const float sdy = b.smask ? -b.dy : b.dy;
      uint4 raw[K];
#pragma unroll
      for (int q = 0; q < K; ++q) raw[q] = ptx::lds_v4(sb + (tid + q * NC) * 16);
      // packed f32x2 FFMA (same per-lane rounding as fmaf): half the FMA-pipe
      // instructions of the scalar form; measured +1.3% under the power cap
      const uint64_t l2e = ptx::f2(kLog2e, kLog2e), nc22 = ptx::f2(nc2, nc2);
#pragma unroll
      for (int q = 0; q < K; ++q) {
        uint64_t p[4];
        PassB<TIn>::unpack2(raw[q], p);
#pragma unroll
        for (int j = 0; j < 4; ++j) p[j] = ptx::ex2x2(ptx::ffma2(p[j], l2e, nc22));
        if (tseg) {
          const int jt = b.y - (v0 + tid + q * NC) * VN;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            if (jt == 2 * j) p[j] = ptx::f2(sdy, ptx::f2hi(p[j]));
            if (jt == 2 * j + 1) p[j] = ptx::f2(ptx::f2lo(p[j]), sdy);
          }
        }
        const uint4 v{ptx::f2_to_bf16x2(p[0]) ^ b.smask, ptx::f2_to_bf16x2(p[1]) ^ b.smask,
                      ptx::f2_to_bf16x2(p[2]) ^ b.smask, ptx::f2_to_bf16x2(p[3]) ^ b.smask};
        ptx::st_global_v4_hint(dseg + static_cast<int64_t>(tid + q * NC) * VN, v, pol);
      }
      return;
    }
  }
  if (!ENT && !zero_row && cnt == kSlotVec) {
    uint4 raw[K];
#pragma unroll
    for (int q = 0; q < K; ++q) raw[q] = ptx::lds_v4(sb + (tid + q * NC) * 16);
#pragma unroll
    for (int q = 0; q < K; ++q) {
      float x[VN], d[VN];
      VI::unpack(raw[q], x);
#pragma unroll
      for (int e = 0; e < VN; ++e) d[e] = ptx::ex2(fmaf(x[e], kLog2e, -b.c1)) * -b.coef;
      if (tseg) {
        const int jt = b.y - (v0 + tid + q * NC) * VN;
#pragma unroll
        for (int e = 0; e < VN; ++e)
          if (e == jt) d[e] = b.dy;
      }
      store_vec<TOut, VN>(dseg + static_cast<int64_t>(tid + q * NC) * VN, d, pol);
    }
  } else {
#pragma unroll
    for (int q = 0; q < K; ++q) {
      const int32_t j = tid + q * NC;
      if (j < cnt) {
        float d[VN];
        if (zero_row) {
#pragma unroll
          for (int e = 0; e < VN; ++e) d[e] = 0.f;
        } else {
          float x[VN];
          VI::unpack(ptx::lds_v4(sb + j * 16), x);
          if constexpr (ENT) {
            row_grad<VN, ENT>(x, d, (v0 + j) * VN, b);
          } else {
#pragma unroll
            for (int e = 0; e < VN; ++e) d[e] = ptx::ex2(fmaf(x[e], kLog2e, -b.c1)) * -b.coef;
            if (tseg) {
              const int jt = b.y - (v0 + j) * VN;
#pragma unroll
              for (int e = 0; e < VN; ++e)
                if (e == jt) d[e] = b.dy;
            }
          }
        }
        store_vec<TOut, VN>(dseg + static_cast<int64_t>(j) * VN, d, pol);
      }
    }
  }
}

}  // namespace
}  // namespace copris_b200
