// pair.cu — fused_pair_kernel: the IS-corrected loss pass for bf16 logits rows
// too large for one SM's shared memory (V = 151,936: 297 KB per row), with ONE
// exponential per element.
//
// A 2-CTA cluster owns a row; CTA h of the pair owns half of its columns.
// Per CTA: 1 producer warp streams the half-row HBM -> shared memory through a
// ring of 32 KB slots (cp.async.bulk + mbarrier complete_tx, read once,
// evict_first); 16 consumer warps (PShape<16>) run pass 1 on each slot as it lands and
// release it at once; 1 scalar warp merges the row's partials and runs the
// token math. Nothing is re-read from L2: the slot ring is pure streaming.
//
// Pass 1, per thread and slot (32 columns): m = max of the thread's columns
// (packed bf16 max, target column excluded), then for each column
// e = 2^((z - m) log2(e) + 15) on MUFU — summed in fp32 for the log-sum-exp
// (the sum never sees the rounding below) and stored as bf16 in TENSOR MEMORY
// (tcgen05.st, 16 columns of 32-bit per thread and slot), with
// nml = 15 - m log2(e) kept in shared memory. Pass 2, after the scalar phase:
// d = e * sign(-coef) 2^(-nml - c2) with the scale rounded to bf16 once per
// thread and slot (one MUFU per thread and slot, none per element):
// tcgen05.ld, then ONE packed bf16x2 multiply per two columns, stored as is.
// Three bf16 roundings (e, scale, product) bound the error by 3 * 2^-9 <
// 2^-7 relative, the bf16-dlogits tolerance. (pair_bf16_stage = 0: f16
// exponentials — the 2^15 offset keeps them in f16's normal range down to
// 2^-29 of the slot maximum — and an f32 multiply, <= 2^-12 before the final
// bf16 rounding; 3.4% slower on one box, more instructions per column.)
//
// f32 dlogits (the parity mode, within 1e-5): f16 staging would cost 2^-12, so
// pass 1 stages the RAW bf16 logits in TMEM instead (same 16 bits per column,
// still no L2 re-read) and pass 2 recomputes p_k = 2^(z_k log2(e) - c1) on MUFU
// — two exponentials per element in this mode, the arithmetic of the other
// fused kernels' f32 pass 2 (fused_common.cuh p2_segment).
//
// The pair exchanges its per-warp partials (m, s, z_y) through DSMEM: every
// consumer warp writes its entry into its own CTA's table (st.shared + local
// mbarrier arrive) and into the peer's with st.async, whose bytes complete
// on the peer's mbarrier (complete_tx: no cluster-scope fence on the
// consumers' path). Both scalar warps merge the same 32 entries in the same
// order — bitwise the same row statistics in both halves, no second
// exchange. Rank 0 writes the per-token outputs.
//
// The same kernel with CL = 1 ("solo", rows up to 7 x 8,192 columns, e.g.
// V = 32,000): one CTA owns the whole row, its warp partials are merged
// locally and nothing crosses DSMEM; it replaces the two exponentials per
// element of the row-resident TMA kernel with one. The solo CTA has 8
// consumer warps and 16 KB slots (PShape<8>: 104 KB of shared memory, 256
// TMEM columns), so two CTAs share an SM and overlap each other's phases.
//
// Small steps (<= 8,192 tokens) reduce obj/flags into out4 in the CTA whose
// scalar warp finishes the launch's scalar phases last (a per-launch count off
// the consumers' path), with its consumer warps once their own dlogits are out
// (reduce.cuh), bitwise what reduce_kernel produces. Nothing global runs on the
// CTAs' exit path: the row counter is rearmed by the last failing claim.
//
// Reference semantics: policy.hpp:110-121,160-173 (log-softmax, gather),
// grpo.hpp:117-185 + policy.hpp:180-196 (objective and dlogits) via
// token_math.cuh, exactly as the other fused kernels.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdint>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

#include "fused_common.cuh"
#include "kernels.cuh"
#include "pair.cuh"
#include "ptx.cuh"
#include "reduce.cuh"
#include "tc.cuh"
#include "token_math.cuh"

namespace copris_b200 {
namespace {

constexpr int kPK = 4;                      // 16-byte vectors per consumer thread per slot
constexpr int kPTSlots = 8;                 // TMEM slots per thread (16 columns each)
constexpr uint32_t kNegInf2 = 0xFF80FF80u;  // bf16x2 (-inf, -inf)

// Shape of a CTA with PW consumer warps: PW = 16 for the CTA pair (one CTA per
// SM, 32 KB slots, the SM's whole 512-column TMEM), PW = 8 for the solo kernel
// (16 KB slots, 256 TMEM columns, 104 KB of shared memory: TWO CTAs per SM,
// whose independent row pipelines overlap one CTA's exponentials with the
// other's stores).
template <int PW>
struct PShape {
  static constexpr int kPW = PW;                      // consumer warps per CTA
  static constexpr int kPThreads = PW * 32;           // consumer threads
  static constexpr int kPSlotVec = kPThreads * kPK;   // 16-byte vectors per slot
  static constexpr int kPSlotBytes = kPSlotVec * 16;  // 32 KB (PW 16) / 16 KB (PW 8)
  static constexpr int kPTmemCols = PW * 32;          // 4 lane quarters x PW/4 warps x 128 columns
};
#define COPRIS_PSHAPE(PW)                                       \
  constexpr int kPW = PShape<PW>::kPW;                          \
  constexpr int kPThreads = PShape<PW>::kPThreads;              \
  constexpr int kPSlotVec = PShape<PW>::kPSlotVec;              \
  constexpr int kPSlotBytes = PShape<PW>::kPSlotBytes;          \
  constexpr int kPTmemCols = PShape<PW>::kPTmemCols;            \
  (void)kPW; (void)kPThreads; (void)kPSlotVec; (void)kPSlotBytes; (void)kPTmemCols

__device__ __forceinline__ uint32_t f2_to_f16x2(uint64_t a) {
  uint32_t r;
  asm("{\n.reg .f32 lo, hi;\nmov.b64 {lo, hi}, %1;\ncvt.rn.f16x2.f32 %0, hi, lo;\n}" : "=r"(r) : "l"(a));
  return r;
}

__device__ __forceinline__ uint64_t f16x2_to_f2(uint32_t w) {
  uint64_t r;
  asm("{\n.reg .f16 lo, hi;\n.reg .f32 a, b;\nmov.b32 {lo, hi}, %1;\n"
      "cvt.f32.f16 a, lo;\ncvt.f32.f16 b, hi;\nmov.b64 %0, {a, b};\n}"
      : "=l"(r)
      : "r"(w));
  return r;
}

__device__ __forceinline__ void tmem_st_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

__device__ __forceinline__ void tmem_ld_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
}

// 16 bytes into the peer CTA's shared memory; the bytes complete on the
// peer's mbarrier `rbar` (both shared::cluster addresses from mapa).
__device__ __forceinline__ void st_async_v4(uint32_t raddr, float a, float b, float c, float d,
                                            uint32_t rbar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
          raddr),
      "f"(a), "f"(b), "f"(c), "f"(d), "r"(rbar)
      : "memory");
}

__device__ __forceinline__ void st_global_b16(void* p, uint16_t v) {
  asm volatile("st.global.b16 [%0], %1;" ::"l"(p), "h"(v) : "memory");
}

__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Per-warp partial of one half-row, exchanged through DSMEM: (m, s) relative
// to m over the non-target columns, the target logit and whether this warp
// holds it.
struct __align__(16) PairPart {
  float m, s, zy, have;
};
// The entropy term's extra per-warp partial: u = sum e (z - m) (same frame as s).
struct __align__(16) PairPartU {
  float u, pad0, pad1, pad2;
};

constexpr float kLn2 = 0.69314718055994531f;
// Row sequence of a cluster: entry j = the j-th row it processes (-1 past the
// end), published by rank 0's producer kRowAhead entries ahead of its own use.
// Every role lags the publisher by a few rows (the ring, the lookahead and the
// two-row scalar pipeline), far fewer than kRowQ, so an entry is never rewritten
// while a CTA of the cluster can still wait on its previous phase.
constexpr int kRowQ = 16;
constexpr uint32_t kRowAhead = 3;
// bf16x2 {-9.9e29, -9.9e29}: -inf columns clamped to it stay finite through
// (z - m) log2(e) (the lowest finite bf16 would overflow to -inf there)
constexpr uint32_t kClampLo2 = 0xF149F149u;

// Lane state of pass 1: running max and the lane's sum of 2^15-scaled
// exponentials relative to it.
struct LaneAcc {
  float m = -INFINITY, s = 0.f;
  float u = 0.f;  // entropy term only: sum e (z - m), natural-log units
  float zy = 0.f;
  bool have = false;
};

// If column jt of a 16-byte vector lies in word k: record it as z_y and set it
// to -inf (keeps the target out of the max and the sum).
__device__ __forceinline__ void kill_col(uint32_t& w, int jt, int k, float& zy) {
  if ((jt >> 1) != k) return;
  if (jt & 1) {
    zy = ptx::bf16_hi(w);
    w = (w & 0x0000FFFFu) | 0xFF800000u;
  } else {
    zy = ptx::bf16_lo(w);
    w = (w & 0xFFFF0000u) | 0xFF80u;
  }
}

// Pass 1 of one consumer thread on one ring slot: `cnt` valid vectors starting
// at vector v0 of this CTA's half; ycol = target column relative to the half.
// STORE: stage the f16 exponentials in TMEM at taddr (16 columns). Returns
// nml = 15 - m log2(e) of this thread's columns (+inf when it saw no finite
// column) for pass 2.
template <bool STORE, bool RAW, bool BST, int PW, bool ENT = false>
__device__ __forceinline__ float p1_slot(LaneAcc& a, uint32_t sb, int32_t v0, int32_t cnt,
                                         int32_t ycol, int tid, uint32_t taddr) {
  COPRIS_PSHAPE(PW);
  uint4 raw[kPK];
  if (cnt == kPSlotVec) {
#pragma unroll
    for (int q = 0; q < kPK; ++q) raw[q] = ptx::lds_v4(sb + (tid + q * kPThreads) * 16);
  } else {
#pragma unroll
    for (int q = 0; q < kPK; ++q) {
      const int32_t j = tid + q * kPThreads;
      raw[q] = j < cnt ? ptx::lds_v4(sb + j * 16) : uint4{kNegInf2, kNegInf2, kNegInf2, kNegInf2};
    }
  }
  if (STORE && RAW) {
    // the logits themselves, target column included (pass 2 overwrites it with
    // the one-hot term; the entropy term there needs p_y)
    uint32_t h[16];
#pragma unroll
    for (int q = 0; q < kPK; ++q) {
      h[q * 4 + 0] = raw[q].x;
      h[q * 4 + 1] = raw[q].y;
      h[q * 4 + 2] = raw[q].z;
      h[q * 4 + 3] = raw[q].w;
    }
    tmem_st_x16(taddr, h);
  }
  // the target column: record z_y, then keep it out of the max and the sum
  if (static_cast<uint32_t>(ycol - v0 * 8) < static_cast<uint32_t>(cnt * 8)) {
#pragma unroll
    for (int q = 0; q < kPK; ++q) {
      const int jt = ycol - (v0 + tid + q * kPThreads) * 8;
      if (static_cast<uint32_t>(jt) < 8u) {
        a.have = true;
        kill_col(raw[q].x, jt, 0, a.zy);
        kill_col(raw[q].y, jt, 1, a.zy);
        kill_col(raw[q].z, jt, 2, a.zy);
        kill_col(raw[q].w, jt, 3, a.zy);
      }
    }
  }
  uint32_t mx = ptx::bmax2(ptx::bmax2(raw[0].x, raw[0].y), ptx::bmax2(raw[0].z, raw[0].w));
#pragma unroll
  for (int q = 1; q < kPK; ++q)
    mx = ptx::bmax2(mx, ptx::bmax2(ptx::bmax2(raw[q].x, raw[q].y), ptx::bmax2(raw[q].z, raw[q].w)));
  const float ml = fmaxf(ptx::bf16_lo(mx), ptx::bf16_hi(mx));
  const bool fin = ml != -INFINITY;
  // all columns -inf: exponentials of -inf (0) with a finite offset
  const float nml = fmaf(-(fin ? ml : 0.f), kLog2e, 15.f);
  const uint64_t l2e = ptx::f2(kLog2e, kLog2e), nml2 = ptx::f2(nml, nml);
  uint64_t acc0 = 0, acc1 = 0;  // two packed fp32 partial sums (0.0f bits)
  uint64_t accu = 0;            // entropy: sum e d, d = (z - ml) log2(e) + 15
  uint32_t h[16];
#pragma unroll
  for (int q = 0; q < kPK; ++q) {
    const uint32_t w[4] = {raw[q].x, raw[q].y, raw[q].z, raw[q].w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      // entropy: -inf columns clamped to a huge finite negative (after the max):
      // e is still 0 there and e d = 0 instead of NaN
      const uint64_t d = ptx::ffma2(ptx::bf16x2_to_f2(ENT ? ptx::bmax2(w[k], kClampLo2) : w[k]), l2e, nml2);
      const uint64_t e = ptx::ex2x2(d);
      if (k & 1) acc1 = ptx::fadd2(acc1, e);
      else acc0 = ptx::fadd2(acc0, e);
      if (ENT) accu = ptx::ffma2(e, d, accu);
      if (STORE && !RAW) h[q * 4 + k] = BST ? ptx::f2_to_bf16x2(e) : f2_to_f16x2(e);
    }
  }
  if (STORE && !RAW) tmem_st_x16(taddr, h);
  const uint64_t acc = ptx::fadd2(acc0, acc1);
  const float sl = ptx::f2lo(acc) + ptx::f2hi(acc);
  // online merge into the lane state (branch-free; both parts relative to mn)
  const float mn = fmaxf(a.m, ml);
  if (mn != -INFINITY) {
    const float ra = a.m == -INFINITY ? 0.f : ptx::ex2((a.m - mn) * kLog2e);
    const float rl = fin ? ptx::ex2((ml - mn) * kLog2e) : 0.f;
    if (ENT) {
      // slot: u_l = sum e (z - ml) = ln2 (sum e d - 15 sl); both parts to frame mn
      const float ul = fin ? kLn2 * ((ptx::f2lo(accu) + ptx::f2hi(accu)) - 15.f * sl) : 0.f;
      const float ua = a.m == -INFINITY ? 0.f : ra * fmaf(a.s, a.m - mn, a.u);
      a.u = ua + (fin ? rl * fmaf(sl, ml - mn, ul) : 0.f);
    }
    a.s = fmaf(a.s, ra, sl * rl);
    a.m = mn;
  }
  return fin ? nml : INFINITY;
}

// Pass 2 of one consumer thread on one slot: dlogits from the staged
// exponentials (or zeros), bf16 out. W256 (full slots, 32-byte aligned rows):
// lane pairs swap one vector each so that every thread writes two ADJACENT
// vectors with one 32-byte store (STG.256); the target column is patched into
// its vector before the swap. Otherwise 16-byte stores and the target column
// written by its owner afterwards (a later store of the same thread).
template <bool W256, bool BST, int PW>
__device__ __forceinline__ void p2_slot(const RowBroadcast& b, bool zero_row, float nml,
                                        uint32_t taddr, int32_t v0, int32_t cnt, int32_t ycol,
                                        __nv_bfloat16* dseg, int tid) {
  COPRIS_PSHAPE(PW);
  __nv_bfloat16* base = dseg + static_cast<int64_t>(tid) * 8;
  const int32_t rel = ycol - v0 * 8;
  const bool own_y = static_cast<uint32_t>(rel) < static_cast<uint32_t>(cnt * 8) &&
                     ((rel >> 3) & (kPThreads - 1)) == tid;
  if (zero_row) {
    const uint4 z{0u, 0u, 0u, 0u};
    if (W256) {
      const int64_t pb = (tid & 1) ? -8 : 0;  // the pair's even vector
#pragma unroll
      for (int q = (tid & 1); q < kPK; q += 2) ptx::st_global_cs_v8u(base + pb + q * kPThreads * 8, z, z);
    } else {
#pragma unroll
      for (int q = 0; q < kPK; ++q)
        if (tid + q * kPThreads < cnt) ptx::st_global_cs_v4(base + q * kPThreads * 8, z);
    }
    return;
  }
  // |coef| p_k = e_k 2^(m log2(e) - 15 - c2) = e_k 2^(-nml - c2); 0 for a lane
  // without finite columns (its staged e are 0 too)
  float sc = nml == INFINITY ? 0.f : ptx::ex2(-(nml + b.c2));
  if (b.coef > 0.f) sc = -sc;  // d = -coef p
  const uint64_t sc2 = ptx::f2(sc, sc);
  uint32_t h[16];
  tmem_ld_x16(taddr, h);
  tc::tmem_wait_ld();
  uint4 v[kPK];
  if (BST) {
    // bf16 staging: one packed bf16 multiply per two columns (sc rounded to bf16)
    const uint32_t sb = ptx::f2_to_bf16x2(sc2);
#pragma unroll
    for (int q = 0; q < kPK; ++q)
      v[q] = uint4{ptx::bmul2(h[q * 4 + 0], sb), ptx::bmul2(h[q * 4 + 1], sb), ptx::bmul2(h[q * 4 + 2], sb),
                   ptx::bmul2(h[q * 4 + 3], sb)};
  } else {
#pragma unroll
    for (int q = 0; q < kPK; ++q) {
      uint32_t o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) o[k] = ptx::f2_to_bf16x2(ptx::fmul2(f16x2_to_f2(h[q * 4 + k]), sc2));
      v[q] = uint4{o[0], o[1], o[2], o[3]};
    }
  }
  if (W256) {
    // one-hot term coef (1 - p_y) (policy.hpp:193-194) into its vector first
    if (own_y) {
      const int qy = rel >> 12, jy = rel & 7;  // vector (tid + qy * 512), column jy of it
      const uint32_t dyb = __bfloat16_as_ushort(__float2bfloat16_rn(b.dy));
      // register-only patch (no address of v is taken: v stays in registers)
      auto patch = [&](uint32_t w, int k) {
        if ((jy >> 1) != k) return w;
        return (jy & 1) ? (w & 0x0000FFFFu) | (dyb << 16) : (w & 0xFFFF0000u) | dyb;
      };
#pragma unroll
      for (int q = 0; q < kPK; ++q)
        if (q == qy) v[q] = uint4{patch(v[q].x, 0), patch(v[q].y, 1), patch(v[q].z, 2), patch(v[q].w, 3)};
    }
    // pair (q, q+1): the even lane stores {own, partner} of q, the odd lane
    // {partner, own} of q+1
    const bool odd = tid & 1;
#pragma unroll
    for (int q = 0; q < kPK; q += 2) {
      const uint4 send = odd ? v[q] : v[q + 1];
      uint4 got;
      got.x = __shfl_xor_sync(0xffffffffu, send.x, 1);
      got.y = __shfl_xor_sync(0xffffffffu, send.y, 1);
      got.z = __shfl_xor_sync(0xffffffffu, send.z, 1);
      got.w = __shfl_xor_sync(0xffffffffu, send.w, 1);
      if (odd)
        ptx::st_global_cs_v8u(base - 8 + (q + 1) * kPThreads * 8, got, v[q + 1]);
      else
        ptx::st_global_cs_v8u(base + q * kPThreads * 8, v[q], got);
    }
    return;
  }
  if (cnt == kPSlotVec) {
#pragma unroll
    for (int q = 0; q < kPK; ++q) ptx::st_global_cs_v4(base + q * kPThreads * 8, v[q]);
  } else {
#pragma unroll
    for (int q = 0; q < kPK; ++q)
      if (tid + q * kPThreads < cnt) ptx::st_global_cs_v4(base + q * kPThreads * 8, v[q]);
  }
  // one-hot term coef (1 - p_y) (policy.hpp:193-194), by the thread that owns it
  if (own_y) st_global_b16(dseg + rel, __bfloat16_as_ushort(__float2bfloat16_rn(b.dy)));
}

// Pass 2, f32 dlogits: the staged raw logits -> d_k = -coef 2^(z_k log2(e) - c1)
// (fused_common.cuh p2_segment's f32 arithmetic), one 32-byte store per 8
// columns (a warp writes 1 KB contiguous per instruction).
template <int PW>
__device__ __forceinline__ void p2_slot_f32(const RowBroadcast& b, bool zero_row, uint32_t taddr,
                                            int32_t v0, int32_t cnt, int32_t ycol, float* dseg,
                                            int tid) {
  COPRIS_PSHAPE(PW);
  float* base = dseg + static_cast<int64_t>(tid) * 8;
  if (zero_row) {
    const float z[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int q = 0; q < kPK; ++q)
      if (tid + q * kPThreads < cnt) ptx::st_global_cs_v8f(base + q * kPThreads * 8, z);
    return;
  }
  uint32_t h[16];
  tmem_ld_x16(taddr, h);
  tc::tmem_wait_ld();
  const float nc = -b.coef, nc1 = -b.c1;
#pragma unroll
  for (int q = 0; q < kPK; ++q) {
    if (cnt == kPSlotVec || tid + q * kPThreads < cnt) {
      float d[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t w = h[q * 4 + k];
        d[2 * k] = ptx::ex2(fmaf(ptx::bf16_lo(w), kLog2e, nc1)) * nc;
        d[2 * k + 1] = ptx::ex2(fmaf(ptx::bf16_hi(w), kLog2e, nc1)) * nc;
      }
      ptx::st_global_cs_v8f(base + q * kPThreads * 8, d);
    }
  }
  const int32_t rel = ycol - v0 * 8;
  if (static_cast<uint32_t>(rel) < static_cast<uint32_t>(cnt * 8) && ((rel >> 3) & (kPThreads - 1)) == tid)
    dseg[rel] = b.dy;
}

// Pass 2 with the entropy term (entropy_coeff != 0): the staged raw logits
// through row_grad (fused_common.cuh), the same per-column arithmetic as the
// other fused kernels, f32 or bf16 out; c0 = absolute column of vector v0.
template <int PW, typename TOut>
__device__ __forceinline__ void p2_slot_ent(const RowBroadcast& b, bool zero_row, uint32_t taddr,
                                            int32_t v0, int32_t cnt, int32_t ycol, TOut* dseg, int tid) {
  COPRIS_PSHAPE(PW);
  constexpr bool kF32 = sizeof(TOut) == 4;
  TOut* base = dseg + static_cast<int64_t>(tid) * 8;
  uint32_t h[16];
  if (!zero_row) {
    tmem_ld_x16(taddr, h);
    tc::tmem_wait_ld();
  }
  // d_k = p_k (eg (x_k + k0) - coef), x = z - m, p = 2^(x log2(e) - log2 S):
  // row_grad's arithmetic, two columns per packed op; -inf columns clamped
  // (kClampLo2) give p = 0 and d = 0 (row_grad's p > 0 guard)
  // folded: 2^(z log2(e) + A) with A = -m log2(e) - log2 S, and eg z + C with
  // C = eg (k0 - m) - coef — no separate x = z - m per column
  const uint64_t l2e = ptx::f2(kLog2e, kLog2e), eg2 = ptx::f2(b.eg, b.eg);
  const float A = fmaf(-b.m, kLog2e, -b.log2s);
  const uint64_t A2 = ptx::f2(A, A);
  const float c0 = fmaf(b.eg, b.k0 - b.m, -b.coef);
  const uint64_t c02 = ptx::f2(c0, c0);
  const int32_t rel = ycol - v0 * 8;
  const bool own_y = static_cast<uint32_t>(rel) < static_cast<uint32_t>(cnt * 8) &&
                     ((rel >> 3) & (kPThreads - 1)) == tid;
#pragma unroll
  for (int q = 0; q < kPK; ++q) {
    if (cnt == kPSlotVec || tid + q * kPThreads < cnt) {
      uint64_t d2[4] = {0, 0, 0, 0};
      if (!zero_row) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint64_t z = ptx::bf16x2_to_f2(ptx::bmax2(h[q * 4 + k], kClampLo2));
          const uint64_t pk = ptx::ex2x2(ptx::ffma2(z, l2e, A2));
          d2[k] = ptx::fmul2(pk, ptx::ffma2(eg2, z, c02));
        }
        // the target column: coef (1 - p_y) + the entropy term (row_grad)
        if (own_y && (rel >> 3) == tid + q * kPThreads) {
          // register-only selects (a dynamic index would put h and d2 in local memory)
          const int jy = rel & 7, ky = jy >> 1;
          uint32_t wy = h[q * 4];
#pragma unroll
          for (int k = 1; k < 4; ++k) wy = ky == k ? h[q * 4 + k] : wy;
          const float zy = (jy & 1) ? ptx::bf16_hi(wy) : ptx::bf16_lo(wy);
          const float xm = zy - b.m;
          const float py = ptx::ex2(fmaf(xm, kLog2e, -b.log2s));
          const float vy = py > 0.f ? fmaf(b.eg * py, xm + b.k0, b.dy) : b.dy;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t pk = (jy & 1) ? ptx::f2(ptx::f2lo(d2[k]), vy) : ptx::f2(vy, ptx::f2hi(d2[k]));
            d2[k] = ky == k ? pk : d2[k];
          }
        }
      }
      if constexpr (kF32) {
        const float d[8] = {ptx::f2lo(d2[0]), ptx::f2hi(d2[0]), ptx::f2lo(d2[1]), ptx::f2hi(d2[1]),
                            ptx::f2lo(d2[2]), ptx::f2hi(d2[2]), ptx::f2lo(d2[3]), ptx::f2hi(d2[3])};
        ptx::st_global_cs_v8f(reinterpret_cast<float*>(base) + q * kPThreads * 8, d);
      } else {
        const uint4 o{ptx::f2_to_bf16x2(d2[0]), ptx::f2_to_bf16x2(d2[1]), ptx::f2_to_bf16x2(d2[2]),
                      ptx::f2_to_bf16x2(d2[3])};
        ptx::st_global_cs_v4(reinterpret_cast<__nv_bfloat16*>(base) + q * kPThreads * 8, o);
      }
    }
  }
}

// grid = CL x clusters, cluster (CL, 1, 1); block = (PW + 2) warps. Dynamic
// shared memory: nslots ring slots, then nml[kPTSlots][kPThreads] floats.
// nvec0 = vectors of CTA ranks 0 .. CL-2 (the last rank takes the rest);
// look = slots of row r+1 run through pass 1 before pass 2 of row r.
// CL = 4 ("quad", rows too wide for a pair's TMEM staging, V > 229,376): every
// consumer warp sends its partial to the three other CTAs; each scalar warp
// merges the 64 entries in rank order (two per lane, then a butterfly).
template <bool F32, int CL, bool BST, int PW, bool ENT>
__global__ void __launch_bounds__((PW + 2) * 32, 16 / PW)
    fused_pair_kernel(const LossParams P, const int nslots, const int look, const int32_t nvec0,
                      const int st256, const int dyn) {
  COPRIS_PSHAPE(PW);
  static_assert(CL == 1 || CL == 2 || CL == 4, "a row is split over one, two or four CTAs");
  constexpr int kNE = CL * PW;  // warp partials per row (entries of the exchange table)
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[16], empty[16], p1done[2], sdone[2];
  __shared__ PairPart red[2][kNE];
  __shared__ PairPartU redu[2][ENT ? kNE : 1];  // entropy: the u of each entry
  constexpr bool kRaw = F32 || ENT;             // stage the raw logits for pass 2
  __shared__ RowBroadcast bc[2];
  __shared__ uint32_t tmem_slot;
  __shared__ bool red_mine;  // small step: this CTA reduces obj/flags into out4
  __shared__ __align__(8) uint64_t rqfull[kRowQ];
  __shared__ __align__(8) int64_t rq[kRowQ];

  const unsigned long long t_entry = P.trace ? PhaseTimer::gtimer() : 0ull;  // trace slot 6
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CL > 1 ? ptx::cluster_ctarank() : 0u;
  const int64_t cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  const int32_t nvec_all = P.vocab / 8;
  const int32_t vbase = static_cast<int32_t>(rank) * nvec0;       // first vector of this part
  const int32_t nvec = min(nvec0, nvec_all - vbase);               // vectors of this part
  const int32_t col0 = vbase * 8;
  const int32_t nseg = (nvec + kPSlotVec - 1) / kPSlotVec;
  const int32_t L = min(look, nseg);
  const bool grad = P.dlogits != nullptr && !P.gather_only;
  // bf16 rows whose every half starts 32-byte aligned: 32-byte stores in pass 2
  const bool w256 = st256 && !F32 && grad && (P.ld_d % 16) == 0 && (reinterpret_cast<uintptr_t>(P.dlogits) % 32) == 0 &&
                    (col0 % 16) == 0;
  const uint32_t sbase = ptx::smem_u32(smem);
  float* nml_sh = reinterpret_cast<float*>(smem + nslots * kPSlotBytes);
  const uint32_t fbase = ptx::smem_u32(full), ebase = ptx::smem_u32(empty);
  const uint32_t p1b = ptx::smem_u32(p1done), sdb = ptx::smem_u32(sdone);
  const uint32_t rqb = ptx::smem_u32(rqfull), rqa = ptx::smem_u32(rq);
  // entry j of the row sequence (waits until rank 0 has published it)
  auto rq_get = [&](uint32_t j) -> int64_t {
    const uint32_t k = j % kRowQ, par = (j / kRowQ) & 1u;
    if constexpr (CL > 1) ptx::mbar_wait_acq_cluster(rqb + k * 8, par);
    else ptx::mbar_wait_u32(rqb + k * 8, par);
    return *reinterpret_cast<volatile int64_t*>(&rq[k]);
  };

  if (threadIdx.x == 0) {
    for (int i = 0; i < nslots; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], kPW);
    }
    for (int i = 0; i < 2; ++i) {
      // the local warps + the scalar warp's arrive that expects the peers' st.async entries
      ptx::mbar_init(&p1done[i], kPW + 1);
      ptx::mbar_init(&sdone[i], 1);
    }
    for (int i = 0; i < kRowQ; ++i) ptx::mbar_init(&rqfull[i], 1);  // rank 0's producer arrives
    ptx::fence_mbarrier_init();
  }
  if (warp == 0) {
    if (grad) tc::tmem_alloc<kPTmemCols>(ptx::smem_u32(&tmem_slot));
    else tc::tmem_relinquish();  // else the next CTA on this SM waits for this one to exit
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if constexpr (CL > 1) ptx::cluster_sync_all();  // the peers' barriers exist before any remote write
  const uint32_t tmem_base = grad ? tmem_slot : 0u;

  if (warp == kPW) {
    // ---------------- producer: this half of every row, slot by slot ------------
    if (lane == 0) {
      const uint64_t pol = ptx::policy_evict_first();  // read once
      Ring ring(nslots);
      // rank 0: the cluster's first row is cid, every later one is claimed from
      // the context's counter (rows ncl, ncl + 1, ...): clusters that run faster
      // take more rows and all finish within about a row of each other (a static
      // stride ended the slowest CTAs 7% (pair) to 17% (solo) of the launch after
      // the mean, scripts/cta_tail.py). The last failing claim rearms the counter.
      bool done = false;
      auto publish = [&](uint32_t j) {
        int64_t r = -1;
        if (!done) {
          r = j == 0 ? cid
                     : (dyn ? ncl + static_cast<int64_t>(atomicAdd(P.row_ctr, 1ull))
                            : cid + static_cast<int64_t>(j) * ncl);
          if (r >= P.n_rows) {
            done = true;
            r = -1;
            // every cluster makes exactly one failing claim (its first row is
            // cid < n_rows); the last of them rearms the counter for the next
            // launch or graph replay — no ticket on the CTAs' exit path
            if (dyn && j > 0) {
              auto* sc = static_cast<ReduceScratch*>(P.red_scratch);
              __threadfence();  // this claim before the count
              if (atomicAdd(&sc->claims_failed, 1u) == static_cast<unsigned>(ncl - 1)) {
                __threadfence();
                *P.row_ctr = 0ull;
                sc->claims_failed = 0u;
              }
            }
          }
        }
        const uint32_t k = j % kRowQ;
        if constexpr (CL > 1) {
#pragma unroll
          for (uint32_t c = 0; c < static_cast<uint32_t>(CL); ++c) {
            ptx::st_cluster_b64(ptx::mapa(rqa + k * 8, c), r);
            ptx::mbar_arrive_remote(ptx::mapa(rqb + k * 8, c));  // releases the store
          }
        } else {
          rq[k] = r;
          ptx::mbar_arrive_u32(rqb + k * 8);
        }
      };
      // row 0 (the cluster index, no claim) goes out first; the claims for rows
      // 1 .. kRowAhead (global atomics, ~1 us each at launch) are made once row
      // 0's loads are in flight, so they are not on the first row's path
      if (rank == 0) publish(0);
      for (uint32_t j = 0;; ++j) {
        const int64_t r = rq_get(j);
        if (r < 0) break;
        const __nv_bfloat16* row = static_cast<const __nv_bfloat16*>(P.logits) + r * P.ld + col0;
        for (int32_t sg = 0; sg < nseg; ++sg, ring.next()) {
          const uint32_t slot = ring.slot;
          ptx::mbar_wait_sleep(ebase + slot * 8, ring.ph ^ 1u);
          const int32_t v0 = sg * kPSlotVec;
          const uint32_t bytes = static_cast<uint32_t>(min(kPSlotVec, nvec - v0)) * 16u;
          ptx::mbar_arrive_expect_tx_u32(fbase + slot * 8, bytes);
          ptx::bulk_g2s_u32(sbase + slot * kPSlotBytes, row + static_cast<int64_t>(v0) * 8, bytes,
                            fbase + slot * 8, pol);
        }
        if (rank == 0) {
          if (j == 0)
            for (uint32_t k = 1; k < kRowAhead; ++k) publish(k);
          publish(j + kRowAhead);
        }
      }
    }
  } else if (warp == kPW + 1) {
    // ---------------- scalar warp: merge the pair's 32 partials, token math ------
    MetaPipe mp;
    int64_t r = rq_get(0);
    int64_t r1 = r >= 0 ? rq_get(1) : -1;
    if (lane == 0) mp.init_ids(P, r, r1);
    uint32_t i = 0;
    for (; r >= 0; ++i) {
      const int64_t r2 = r1 >= 0 ? rq_get(i + 2) : -1;
      RowMeta meta{};
      if (lane == 0) meta = mp.advance_ids(P, r1, r2);
      const uint32_t bsel = i & 1u, par = (i >> 1) & 1u;
      if (lane == 0) {
        if constexpr (CL > 1)
          ptx::mbar_arrive_expect_tx_u32(p1b + bsel * 8,
                                         (CL - 1) * kPW * (sizeof(PairPart) + (ENT ? sizeof(PairPartU) : 0)));
        else ptx::mbar_arrive_u32(p1b + bsel * 8);
      }
      ptx::mbar_wait_sleep(p1b + bsel * 8, par);
      // entry = rank * PW + warp: the same order in every CTA of the cluster
      // (solo: lanes PW..31 empty; 4 x 16 entries: lane l merges l, then l + 32)
      // (entropy: u and a = s of the non-target columns; the target joins below)
      const PairPart e = lane < kNE ? red[bsel][lane] : PairPart{-INFINITY, 0.f, 0.f, 0.f};
      Lse tot{e.m, e.s, ENT && lane < kNE ? redu[bsel][lane % kNE].u : 0.f, ENT ? e.s : 0.f};
      bool have = e.have != 0.f;
      float ezy = e.zy;
      if constexpr (kNE > 32) {
        static_assert(kNE <= 64, "two entries per lane at most");
        const PairPart e2 = red[bsel][lane + 32];
        lse_merge<ENT>(tot, Lse{e2.m, e2.s, ENT ? redu[bsel][(lane + 32) % kNE].u : 0.f, ENT ? e2.s : 0.f});
        if (e2.have != 0.f) {
          have = true;
          ezy = e2.zy;
        }
      }
      warp_lse<ENT>(tot);
      const uint32_t hv = __ballot_sync(0xffffffffu, have);
      float zy = __shfl_sync(0xffffffffu, ezy, hv ? __ffs(hv) - 1 : 0);
      if (lane == 0) {
        const bool ok = static_cast<uint32_t>(meta.y) < static_cast<uint32_t>(P.vocab);
        if (!ok) zy = 0.f;
        // the target column stayed out of every thread's max: fold it into M
        // so that M >= z_y as finish_logprob assumes
        if (ok && hv && zy > tot.m) {
          const float rz = ptx::ex2((tot.m - zy) * kLog2e);
          if (ENT) {
            tot.u = tot.m == -INFINITY ? 0.f : rz * fmaf(tot.a, tot.m - zy, tot.u);
            tot.a = tot.m == -INFINITY ? 0.f : tot.a * rz;
          }
          tot.s = tot.m == -INFINITY ? 0.f : tot.s * rz;
          tot.m = zy;
        }
        if (ENT && ok && hv) {  // u and a run over every column (fused_common.cuh Lse)
          const float ey = ptx::ex2((zy - tot.m) * kLog2e);
          if (ey > 0.f) {
            tot.a += ey;
            tot.u = fmaf(ey, zy - tot.m, tot.u);
          }
        }
        bc[bsel] = row_scalar_phase<ENT>(P, P.row_base + r, meta.y, meta.st, meta.blp, meta.rl,
                                           meta.adv, tot, zy, rank == 0, meta.keep);
        ptx::mbar_arrive_u32(sdb + bsel * 8);
      }
      __syncwarp();
      r = r1;
      r1 = r2;
    }
    // small step: this CTA's rows have all written obj/flags (rank 0 writes
    // them); the CTA whose count completes the launch reduces, with its consumer
    // warps once their last dlogits are out — the count is off their path and
    // the other CTAs may still be writing dlogits
    if (P.out4 && lane == 0) {
      bool last = false;
      if (rank == 0) {
        __threadfence();  // release this CTA's obj/flags
        auto* sc = static_cast<ReduceScratch*>(P.red_scratch);
        last = atomicAdd(&sc->rows_done, 1u) == static_cast<unsigned>(ncl - 1);
        if (last) {
          __threadfence();  // acquire: every CTA's obj/flags
          sc->rows_done = 0u;
        }
      }
      red_mine = last;
    }
    if (P.out4) ptx::named_bar_sync(2, (kPW + 1) * 32);  // the consumers read red_mine
  } else {
    // ---------------- consumers ------------------------------------------------------
    const int tid = threadIdx.x;
    const uint32_t taddr0 = tmem_base + (static_cast<uint32_t>((warp & 3) * 32) << 16) +
                            static_cast<uint32_t>((warp >> 2) * (kPTSlots * 16));
    Ring ring(nslots);
    uint32_t ts = 0;  // TMEM slot of the next pass-1 slot (mod kPTSlots)
    uint32_t red_peer[CL > 1 ? CL - 1 : 1], redu_peer[CL > 1 ? CL - 1 : 1], p1_peer[CL > 1 ? CL - 1 : 1];
#pragma unroll
    for (int c = 1; c < CL; ++c) {  // the other CTAs of the cluster, in rank order after this one
      const uint32_t pr = (rank + static_cast<uint32_t>(c)) % CL;
      red_peer[c - 1] = ptx::mapa(ptx::smem_u32(&red[0][0]), pr);
      if (ENT) redu_peer[c - 1] = ptx::mapa(ptx::smem_u32(&redu[0][0]), pr);
      p1_peer[c - 1] = ptx::mapa(p1b, pr);
    }
    PhaseTimer tm;    // trace slots: 0 pass 1, 2 broadcast wait, 4 pass 2, 6 kernel entry (globaltimer ns), 7 SM id
    tm.start(P.trace && tid == 0 && blockIdx.x < kTraceCtas);
    if (tm.on) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      tm.acc[6] = static_cast<long long>(t_entry);
      tm.acc[7] = smid;
    }

    auto run_p1 = [&](LaneAcc& a, int32_t ycol, int32_t sg0, int32_t sg1) {
      for (int32_t sg = sg0; sg < sg1; ++sg, ring.next()) {
        const uint32_t slot = ring.slot;
        const int32_t v0 = sg * kPSlotVec;
        const int32_t cnt = min(kPSlotVec, nvec - v0);
        ptx::mbar_wait_sleep(fbase + slot * 8, ring.ph);
        const uint32_t tsl = (ts + static_cast<uint32_t>(sg)) % kPTSlots;
        const float nml = grad ? p1_slot<true, kRaw, BST, PW, ENT>(a, sbase + slot * kPSlotBytes, v0, cnt, ycol,
                                                                  tid, taddr0 + tsl * 16)
                               : p1_slot<false, kRaw, BST, PW, ENT>(a, sbase + slot * kPSlotBytes, v0, cnt, ycol,
                                                                   tid, 0u);
        nml_sh[tsl * kPThreads + tid] = nml;
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_u32(ebase + slot * 8);
      }
    };
    // publish row i's warp partial: own table + arrive, peer table by st.async
    auto finish_p1 = [&](LaneAcc& a, uint32_t i) {
      // warp merge: common max, rescale, sum (lanes without columns hold -inf, 0)
      float M = a.m;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
      float sv = a.m == -INFINITY ? 0.f : a.s * ptx::ex2((a.m - M) * kLog2e);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sv += __shfl_xor_sync(0xffffffffu, sv, o);
      const Lse st{M, sv * (1.f / 32768.f), 0.f, 0.f};
      float uv = 0.f;
      if (ENT) {  // u to the warp frame M: r (u + s (m - M)), 2^15-scaled like s
        uv = a.m == -INFINITY ? 0.f : ptx::ex2((a.m - M) * kLog2e) * fmaf(a.s, a.m - M, a.u);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) uv += __shfl_xor_sync(0xffffffffu, uv, o);
        uv *= 1.f / 32768.f;
      }
      const uint32_t hv = __ballot_sync(0xffffffffu, a.have);
      const float zy = __shfl_sync(0xffffffffu, a.zy, hv ? __ffs(hv) - 1 : 0);
      if (lane == 0) {
        const uint32_t bsel = i & 1u;
        const uint32_t off = (bsel * kNE + rank * kPW + warp) * sizeof(PairPart);
        const float hvf = hv ? 1.f : 0.f;
        red[bsel][rank * kPW + warp] = PairPart{st.m, st.s, zy, hvf};
        if (ENT) redu[bsel][(rank * kPW + warp) % (ENT ? kNE : 1)] = PairPartU{uv, 0.f, 0.f, 0.f};
        ptx::mbar_arrive_u32(p1b + bsel * 8);
#pragma unroll
        for (int c = 0; c < CL - 1; ++c) {
          st_async_v4(red_peer[c] + off, st.m, st.s, zy, hvf, p1_peer[c] + bsel * 8);
          if (ENT)
            st_async_v4(redu_peer[c] + (off / sizeof(PairPart)) * sizeof(PairPartU), uv, 0.f, 0.f, 0.f,
                        p1_peer[c] + bsel * 8);
        }
      }
    };

    int64_t r = rq_get(0);
    uint32_t i = 0;
    if (r >= 0) {
      LaneAcc a0;
      run_p1(a0, P.target[P.row_base + r] - col0, 0, nseg);
      finish_p1(a0, 0);
    }
    for (; r >= 0; ++i) {
      const int64_t rn = rq_get(i + 1);
      const bool nx = rn >= 0;
      const uint32_t ts_row = ts;  // TMEM slots of row i: ts_row .. ts_row + nseg - 1
      LaneAcc an;
      const int32_t ycn = nx ? P.target[P.row_base + rn] - col0 : -1;
      ts = (ts + static_cast<uint32_t>(nseg)) % kPTSlots;
      tm.mark(0);
      if (nx) run_p1(an, ycn, 0, L);
      tm.mark(0);
      const uint32_t bsel = i & 1u, par = (i >> 1) & 1u;
      ptx::mbar_wait_backoff(sdb + bsel * 8, par);  // row i's broadcast
      tm.mark(2);
      if (grad) {
        const RowBroadcast b = bc[bsel];
        const bool zero_row = b.coef == 0.f && (!ENT || b.eg == 0.f);
        const int32_t ycol = b.y - col0;
        tmem_wait_st();  // this thread's pass-1 stores of row i have landed
        for (int32_t sg = 0; sg < nseg; ++sg) {
          const uint32_t tsl = (ts_row + static_cast<uint32_t>(sg)) % kPTSlots;
          const int32_t v0 = sg * kPSlotVec;
          if constexpr (ENT) {
            using TO = typename std::conditional<F32, float, __nv_bfloat16>::type;
            TO* drow = static_cast<TO*>(P.dlogits) + r * P.ld_d + col0;
            p2_slot_ent<PW, TO>(b, zero_row, taddr0 + tsl * 16, v0, min(kPSlotVec, nvec - v0), ycol,
                                drow + static_cast<int64_t>(v0) * 8, tid);
          } else if constexpr (F32) {
            float* drow = static_cast<float*>(P.dlogits) + r * P.ld_d + col0;
            p2_slot_f32<PW>(b, zero_row, taddr0 + tsl * 16, v0, min(kPSlotVec, nvec - v0), ycol,
                        drow + static_cast<int64_t>(v0) * 8, tid);
          } else {
            __nv_bfloat16* drow = static_cast<__nv_bfloat16*>(P.dlogits) + r * P.ld_d + col0;
            const int32_t cnt = min(kPSlotVec, nvec - v0);
            if (w256 && cnt == kPSlotVec)
              p2_slot<true, BST, PW>(b, zero_row, nml_sh[tsl * kPThreads + tid], taddr0 + tsl * 16, v0, cnt,
                            ycol, drow + static_cast<int64_t>(v0) * 8, tid);
            else
              p2_slot<false, BST, PW>(b, zero_row, nml_sh[tsl * kPThreads + tid], taddr0 + tsl * 16, v0, cnt,
                             ycol, drow + static_cast<int64_t>(v0) * 8, tid);
          }
        }
      }
      tm.mark(4);
      if (nx) {
        run_p1(an, ycn, L, nseg);
        finish_p1(an, i + 1);
      }
      tm.mark(0);
      tm.acc[5] += 1;
      r = rn;
    }
    tm.flush(P.trace);
    if (P.out4) {
      // the scalar warp has counted this CTA; the ring is idle (every slot it
      // was filled for has been through pass 1)
      ptx::named_bar_sync(2, (kPW + 1) * 32);
      if (red_mine && tid < kReduceThreads) {
        ReduceSmem& rsm = *reinterpret_cast<ReduceSmem*>(smem);
        if ((reinterpret_cast<uintptr_t>(P.obj) % 16 == 0) && (reinterpret_cast<uintptr_t>(P.flags) % 4 == 0))
          reduce_all_in_cta<true>(P.obj, P.flags, P.red_n, P.out4, rsm, tid);
        else
          reduce_all_in_cta<false>(P.obj, P.flags, P.red_n, P.out4, rsm, tid);
      }
    }
  }
  // no CTA may exit (or free TMEM) while its peer can still address its shared
  // memory or a thread of its own still reads TMEM
  tc::fence_before_sync();
  __syncthreads();
  if constexpr (CL > 1) ptx::cluster_sync_all();
  if (warp == 0 && grad) {
    tc::fence_after_sync();
    tc::tmem_dealloc<kPTmemCols>(tmem_base);
  }
  // (the row counter was rearmed by the last failing claim, the small-step
  // reduction done by the scalar warp of the last scalar phase: nothing global
  // on the exit path)
}

}  // namespace

bool pair_supported(const LossParams& p, DType in, DType out, bool ent, int cl) {
  (void)ent;  // entropy: the ENT instantiations (raw staging, u exchanged with the partials)
  if (in != DType::BF16) return false;
  if (p.dlogits != nullptr && !p.gather_only && out != DType::BF16 && out != DType::F32) return false;
  if (p.vocab % 16 != 0 || (p.ld * 2) % 16 != 0 || reinterpret_cast<uintptr_t>(p.logits) % 16 != 0)
    return false;
  // f32 rows leave through 32-byte stores
  const int64_t osz = out == DType::F32 ? 4 : 2, oal = out == DType::F32 ? 32 : 16;
  if (p.dlogits && ((p.ld_d * osz) % oal != 0 || reinterpret_cast<uintptr_t>(p.dlogits) % oal != 0))
    return false;
  // cl = 2: a CTA pair, or (rows too wide for the pair's TMEM staging, e.g.
  // V = 256,000) a 4-CTA cluster. K1 (gather-only) and forward-only launches
  // take the SAME kernel shape as the loss at their vocabulary, so their
  // log-probs are bitwise the loss kernel's recomputation (test_policy.cpp:157-172;
  // a solo K1 at V = 151,936 was also slower: 0.73 vs 0.80)
  return cl == 2 ? pair_fits(p.vocab, 2, 16) || pair_fits(p.vocab, 4, 16) : pair_fits(p.vocab, 1, 8);
}

// Whether a row's part per CTA (half for cl = 2) fits the TMEM staging of a
// CTA with `pw` consumer warps: at most kPTSlots - 1 slots, one left for the
// lookahead.
bool pair_fits(int32_t vocab, int cl, int pw) {
  const int32_t slot_vec = pw == 16 ? PShape<16>::kPSlotVec : PShape<8>::kPSlotVec;
  const int32_t nvec0 = (vocab / 8 + cl - 1) / cl;
  const int32_t nseg = (nvec0 + slot_vec - 1) / slot_vec;
  return nseg <= kPTSlots - 1;
}

namespace {
// CTAs of `kern` that fit one SM: shared memory (dynamic + static + the 1 KB the
// runtime reserves per CTA), registers, threads and TMEM columns. The occupancy
// API answered 1 for the 104 KB solo CTA where two fit and run (measured: 296
// co-resident CTAs, one group x L = 256 at 0.78 instead of 0.66 of peak).
int ctas_per_sm(const void* kern, int threads, int dyn_smem, int tmem_cols) {
  int dev = 0, smem_sm = 0, regs_sm = 0, thr_sm = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 1;
  // cached per (kernel, device, shared memory): the answer is static
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, int>, int> cache;
  const auto key = std::make_tuple(kern, dev, dyn_smem);
  {
    std::lock_guard<std::mutex> lock(mu);
    const auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) return 1;
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&thr_sm, cudaDevAttrMaxThreadsPerMultiProcessor, dev);
  const int per_cta = dyn_smem + static_cast<int>(fa.sharedSizeBytes) + 1024;
  int n = smem_sm / per_cta;
  const int regs = ((fa.numRegs + 7) / 8) * 8 * threads;
  if (regs > 0) n = std::min(n, regs_sm / regs);
  n = std::min(n, thr_sm / threads);
  n = std::min(n, 512 / tmem_cols);
  n = n < 1 ? 1 : n;
  std::lock_guard<std::mutex> lock(mu);
  cache[key] = n;
  return n;
}

template <int PW, int CL>
cudaError_t launch_pair_pw(const LossParams& p, DType out, int num_sms, const Tuning& tu,
                           cudaStream_t stream, LaunchInfo* info) {
  COPRIS_PSHAPE(PW);
  constexpr int cl = CL;
  const bool f32 = out == DType::F32 && p.dlogits != nullptr && !p.gather_only;
  const bool ent = p.entropy_coeff != 0.0;
  const bool bst = !f32 && !ent && tu.pair_bf16_stage;
  using Kern = void (*)(const LossParams, const int, const int, const int32_t, const int, const int);
  // entropy: raw logits staged (pass 2 needs z for the p log p term), f32 or bf16 out
  const Kern kern = ent ? (f32 ? fused_pair_kernel<true, CL, false, PW, true> : fused_pair_kernel<false, CL, false, PW, true>)
                  : f32 ? fused_pair_kernel<true, CL, false, PW, false>
                        : (bst ? fused_pair_kernel<false, CL, true, PW, false> : fused_pair_kernel<false, CL, false, PW, false>);
  // PW 16: 6 x 32 KB ring + 16 KB of per-thread nml fill the 227 KB a CTA may
  // use; PW 8: 6 x 16 KB + 8 KB = 104 KB, two CTAs per SM
  const int nslots = tu.slots > 0 ? (tu.slots > 6 ? 6 : tu.slots) : 6;
  const int smem = nslots * kPSlotBytes + kPTSlots * kPThreads * static_cast<int>(sizeof(float));
  cudaError_t e = allow_dyn_smem(reinterpret_cast<const void*>(kern), smem);
  if (e != cudaSuccess) return e;
  const int32_t nvec0 = (p.vocab / 8 + cl - 1) / cl;  // vectors per CTA (the last takes the rest)
  const int32_t nseg = (nvec0 + kPSlotVec - 1) / kPSlotVec;
  int look = tu.pair_lookahead;
  if (look > kPTSlots - nseg) look = kPTSlots - nseg;
  if (look < 0) look = 0;
  // no dlogits (K1's gather-only mode, forward-only losses): nothing is staged
  // in TMEM, so pass 1 of the whole next row may run before this row's scalar
  // phase is awaited
  if (p.dlogits == nullptr || p.gather_only) look = nseg;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cl;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = cl > 1 ? 1 : 0;
  cfg.blockDim = dim3((kPW + 2) * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  int64_t slots = 0;  // resident rows-in-flight units (CTA pairs or CTAs)
  if (cl > 1) {
    const int sms = num_sms / cl * cl;
    cfg.gridDim = dim3(static_cast<unsigned>(sms));
    int ncl = 0;
    e = cudaOccupancyMaxActiveClusters(&ncl, reinterpret_cast<const void*>(kern), &cfg);
    if (e != cudaSuccess) return e;
    slots = ncl;
    if (PW == 8) {
      // two 8-warp CTAs per SM: the API under-counts them as for the solo kernel
      const int per_sm = ctas_per_sm(reinterpret_cast<const void*>(kern), (kPW + 2) * 32, smem, kPTmemCols);
      slots = std::max<int64_t>(ncl, static_cast<int64_t>(per_sm) * sms / cl);
    }
    // (4-CTA clusters: the API's count is the truth — GPC placement leaves some
    // SMs without a whole cluster, and launching more than fit runs a second wave)
  } else {
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reinterpret_cast<const void*>(kern),
                                                      (kPW + 2) * 32, smem);
    if (e != cudaSuccess) return e;
    per_sm = std::max(per_sm, ctas_per_sm(reinterpret_cast<const void*>(kern), (kPW + 2) * 32, smem,
                                          kPTmemCols));
    slots = static_cast<int64_t>(per_sm) * num_sms;
  }
  if (slots < 1) return cudaErrorInvalidConfiguration;
  const int64_t nc = p.n_rows < slots ? p.n_rows : slots;
  cfg.gridDim = dim3(static_cast<unsigned>(cl * nc));
  // fused reduction for small steps: the last CTA reduces in its free ring
  LossParams q = p;
  const bool fuse = fuse_reduce_ok(p, smem);
  if (!fuse) q.out4 = nullptr;
  if (info) {
    info->cluster = cl;
    info->grid = static_cast<int>(cl * nc);
    info->kernel = cl == 4 ? "fused_quad_kernel" : cl == 2 ? "fused_pair_kernel" : "fused_solo_kernel";
    info->reduced = fuse ? 1 : 0;
  }
  // claimed rows need the counter and the ticket that lets the last CTA rearm it
  const int dyn = tu.pair_dynamic && p.row_ctr && p.red_scratch ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, q, nslots, look, nvec0, tu.pair_st256, dyn);
}
}  // namespace

cudaError_t launch_pair(const LossParams& p, DType out, int cl, int num_sms, const Tuning& tu,
                        cudaStream_t stream, LaunchInfo* info) {
  if (cl == 1) return launch_pair_pw<8, 1>(p, out, num_sms, tu, stream, info);
  // half rows that fit the 8-warp shape (V <= 114,688) run two CTAs per SM;
  // rows too wide for a 16-warp pair (V > 229,376) split over 4 CTAs
  if (pair_fits(p.vocab, 2, 8) && tu.pair_pw8) return launch_pair_pw<8, 2>(p, out, num_sms, tu, stream, info);
  if (pair_fits(p.vocab, 2, 16)) return launch_pair_pw<16, 2>(p, out, num_sms, tu, stream, info);
  return launch_pair_pw<16, 4>(p, out, num_sms, tu, stream, info);
}

}  // namespace copris_b200
