// lmhead.cu — the LM-head forward fused with the log-softmax statistics
// (the producer side of a8, trainer.hpp:146).
//
//   logits[T x V] = hidden[T x H] * weight[V x H]^T      (bf16 in, fp32 accumulate)
//
// is computed on the 5th-generation tensor cores (tcgen05.mma, accumulators in
// TMEM, operands staged by 2-D TMA with 128-byte swizzle) and the epilogue —
// while the tile is still on chip — rounds it to bf16, stores it, and emits the
// per-(token, 256-column tile) log-sum-exp partial {max, sum exp(z - max)} of
// the ROUNDED values with the target column left out of the sum. A tiny merge
// kernel then yields (cur_lp, lse) exactly as K1 (logprob_gather) would from
// the stored logits, without K1's full read of the [T x V] logits: the loss
// path that follows becomes a single streaming pass (bwd_kernel).
//
// Kernel anatomy (one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer: A = hidden[128 x 64], B = weight[256 x 64] per
//               k-step into a kStages-deep shared-memory ring (48 KB / stage).
//   warp 1      TMEM owner (allocates 512 columns = two 128 x 256 fp32
//               accumulators) and MMA issuer (one thread; 4 x K=16 MMAs per
//               k-step, tcgen05.commit frees the ring slot).
//   warps 2..5  epilogue: tcgen05.ld 32 rows x 32 columns at a time; each
//               thread owns one token row of the tile. Double-buffered TMEM lets
//               the epilogue of tile i overlap the MMAs of tile i + 1.
// Tile order is vocab-tile-major, so CTAs running concurrently share weight
// tiles through L2 while the hidden block (T_chunk x H) stays L2-resident.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "lmhead.cuh"
#include "ptx.cuh"
#include "tc.cuh"

namespace copris_b200 {

namespace {

constexpr int kBM = 128;       // tokens per tile (TMEM lanes)
constexpr int kBN = kLmTileN;  // vocab columns per tile (fp32 TMEM columns)
constexpr int kBK = 64;        // K per stage: one 128-byte swizzle row of bf16
constexpr int kStages = 4;
constexpr int kABytes = kBM * kBK * 2;  // 16 KB
constexpr int kBBytes = kBN * kBK * 2;  // 32 KB
constexpr int kStageBytes = kABytes + kBBytes;
constexpr int kTmemCols = 2 * kBN;      // double-buffered accumulator
constexpr int kThreads = 192;
constexpr int kEpiThreads = 128;
constexpr size_t kSmemBytes = 1024 /*align slack*/ + kStages * kStageBytes + 256 /*barriers*/;

struct LmParams {
  int64_t n_rows;
  int32_t H, V;
  int32_t n_mblk, n_vt;
  int64_t n_tiles;
  __nv_bfloat16* logits;
  int64_t ld;
  float2* partials;  // [n_rows][n_vt]
  const int32_t* target;
  int32_t group;     // token-pair blocks per raster group (pair kernel)
  // plain GEMM mode (EPI == 1, the LM-head backward dhidden = dlogits W):
  // C[split][M x N] fp32 partials over k-block ranges of k_per_split blocks
  float* c_out;
  int64_t ldc;
  int64_t split_stride;  // elements between the partial matrices of two splits
  int32_t n_split, k_per_split;
  int32_t a_evict_first;
};

__device__ __forceinline__ float bf16_round(float x) {
  return __bfloat162float(__float2bfloat16_rn(x));
}

// One thread = one token row of a 128 x kBN accumulator tile in TMEM: round
// to bf16, store, and reduce {max, sum exp(z - max)} over the tile's valid
// columns with the target column left out. Returns the partial.
__device__ __forceinline__ float2 epilogue_row(uint32_t taddr, int64_t row, bool row_ok,
                                               int32_t n0, int32_t ncols, int32_t yrel,
                                               const LmParams& P, uint64_t st_pol) {
  float m = -INFINITY, s = 0.f;
  __nv_bfloat16* out = P.logits + row * P.ld + n0;
#pragma unroll 1
  for (int c = 0; c < kBN; c += 32) {
    uint32_t r[32];
    tc::tmem_ld_32x32b_x32(taddr + c, r);
    tc::tmem_wait_ld();
    if (c >= ncols) break;  // uniform across the warp (tile-level)
    float z[32];
    float cm = -INFINITY;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      z[j] = bf16_round(__uint_as_float(r[j]));
      if (c + j < ncols) cm = fmaxf(cm, z[j]);
    }
    if (cm > m) {
      s *= ptx::ex2((m - cm) * kLog2e);
      m = cm;
    }
    const float mb = m * kLog2e;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float e = ptx::ex2(fmaf(z[j], kLog2e, -mb));
      if (c + j < ncols && c + j != yrel) s += e;
    }
    if (row_ok) {
      if (c + 32 <= ncols) {
        uint4* o = reinterpret_cast<uint4*>(out + c);
#pragma unroll
        for (int q = 0; q < 4; ++q)
          ptx::st_global_v4_hint(o + q,
                                 make_uint4(ptx::pack_bf16x2(z[8 * q + 0], z[8 * q + 1]),
                                            ptx::pack_bf16x2(z[8 * q + 2], z[8 * q + 3]),
                                            ptx::pack_bf16x2(z[8 * q + 4], z[8 * q + 5]),
                                            ptx::pack_bf16x2(z[8 * q + 6], z[8 * q + 7])),
                                 st_pol);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (c + j < ncols) out[c + j] = __float2bfloat16_rn(z[j]);
      }
    }
  }
  return make_float2(m, s);
}

// epilogue_row with the logits leaving through TMA stores: the warp stages its
// 32 rows x 64 columns of rounded bf16 in a swizzled 4 KB box (16-byte chunk j
// of row r at j ^ (r & 7)) and one lane stores it (full 128-byte lines instead
// of 16-byte pieces of 32 different rows per instruction). The {max, sum}
// arithmetic is exactly epilogue_row's. `box0` = this warp's two staging boxes.
__device__ __forceinline__ float2 epilogue_row_tma(uint32_t taddr, int32_t row0, int32_t n0,
                                                   int32_t ncols, int32_t yrel,
                                                   const CUtensorMap* tm_l, uint32_t box0,
                                                   int& buf, uint64_t st_pol, bool stats) {
  const int lane = threadIdx.x & 31;
  float m = -INFINITY, s = 0.f;
#pragma unroll 1
  for (int c = 0; c < kBN; c += 64) {
    if (c >= ncols) break;  // uniform across the warp (tile-level)
    const uint32_t box = box0 + static_cast<uint32_t>(buf) * 4096u;
    if (lane == 0) tc::bulk_wait_group_read<1>();  // the store issued 2 boxes ago read `box`
    __syncwarp();
#pragma unroll 1
    for (int h = 0; h < 2; ++h) {
      const int cc = c + 32 * h;
      uint32_t r[32];
      tc::tmem_ld_32x32b_x32(taddr + cc, r);
      tc::tmem_wait_ld();
      float z[32];
      float cm = -INFINITY;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        z[j] = bf16_round(__uint_as_float(r[j]));
        if (cc + j < ncols) cm = fmaxf(cm, z[j]);
      }
      if (stats && cc < ncols) {  // logits-only mode: no statistics, no exponentials
        if (cm > m) {
          s *= ptx::ex2((m - cm) * kLog2e);
          m = cm;
        }
        const float mb = m * kLog2e;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float e = ptx::ex2(fmaf(z[j], kLog2e, -mb));
          if (cc + j < ncols && cc + j != yrel) s += e;
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        ptx::sts_v4(box + lane * 128 + (((4 * h + q) ^ (lane & 7)) << 4),
                    make_uint4(ptx::pack_bf16x2(z[8 * q + 0], z[8 * q + 1]),
                               ptx::pack_bf16x2(z[8 * q + 2], z[8 * q + 3]),
                               ptx::pack_bf16x2(z[8 * q + 4], z[8 * q + 5]),
                               ptx::pack_bf16x2(z[8 * q + 6], z[8 * q + 7])));
    }
    ptx::fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tc::tma_store_2d(tm_l, box, n0 + c, row0, st_pol);
      tc::bulk_commit_group();
    }
    buf ^= 1;
  }
  return make_float2(m, s);
}

__global__ void __launch_bounds__(kThreads, 1)
    lmhead_fwd_kernel(const __grid_constant__ CUtensorMap tm_x,
                      const __grid_constant__ CUtensorMap tm_w, const LmParams P) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sA = base;                         // kStages x 16 KB
  const uint32_t sB = base + kStages * kABytes;     // kStages x 32 KB
  const uint32_t bars = base + kStages * kStageBytes;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (kStages + s); };
  auto tfull_bar = [&](int b) { return bars + 8u * (2 * kStages + b); };
  auto tempty_bar = [&](int b) { return bars + 8u * (2 * kStages + 2 + b); };
  const uint32_t tmem_slot = bars + 8u * (2 * kStages + 4);
  uint8_t* generic_base = smem_raw + (base - ptx::smem_u32(smem_raw));
  volatile uint32_t* tmem_slot_ptr =
      reinterpret_cast<volatile uint32_t*>(generic_base + (tmem_slot - base));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full_bar(s)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(empty_bar(s)));
    }
    for (int b = 0; b < 2; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tfull_bar(b)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tempty_bar(b)),
                   "r"(kEpiThreads));
    }
    ptx::fence_mbarrier_init();
    tc::prefetch_tensormap(&tm_x);
    tc::prefetch_tensormap(&tm_w);
  }
  if (warp == 1) tc::tmem_alloc<kTmemCols>(tmem_slot);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem_base = *tmem_slot_ptr;

  const int nk = (P.H + kBK - 1) / kBK;
  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      const uint64_t pol_w = ptx::policy_evict_normal();  // weight tiles: shared by concurrent CTAs
      const uint64_t pol_x = ptx::policy_evict_last();   // hidden block: re-read for every vocab tile
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
        const int32_t m0 = static_cast<int32_t>(t % P.n_mblk) * kBM;
        const int32_t n0 = static_cast<int32_t>(t / P.n_mblk) * kBN;
        for (int kb = 0; kb < nk; ++kb) {
          ptx::mbar_wait_u32(empty_bar(stage), phase ^ 1u);
          ptx::mbar_arrive_expect_tx_u32(full_bar(stage), kStageBytes);
          tc::tma_load_2d(sA + stage * kABytes, &tm_x, full_bar(stage), kb * kBK, m0, pol_x);
          tc::tma_load_2d(sB + stage * kBBytes, &tm_w, full_bar(stage), kb * kBK, n0, pol_w);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer =====
      constexpr uint32_t idesc = tc::idesc_bf16_f32<kBM, kBN>();
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int64_t t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
        ptx::mbar_wait_u32(tempty_bar(acc), acc_phase ^ 1u);
        tc::fence_after_sync();
        const uint32_t d = tmem_base + static_cast<uint32_t>(acc * kBN);
        for (int kb = 0; kb < nk; ++kb) {
          ptx::mbar_wait_u32(full_bar(stage), phase);
          tc::fence_after_sync();
          const uint32_t a = sA + stage * kABytes, b = sB + stage * kBBytes;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k)  // K = 16 per MMA: +32 bytes along the swizzled row
            tc::mma_bf16_ss(d, tc::smem_desc_sw128(a + 32 * k), tc::smem_desc_sw128(b + 32 * k),
                            idesc, (kb | k) != 0);
          tc::commit(empty_bar(stage));
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        tc::commit(tfull_bar(acc));
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1u;
        }
      }
    }
  } else {
    // ===== epilogue: TMEM -> bf16 logits + LSE partials =====
    const int sub = warp & 3;  // TMEM lane quarter this warp may access
    const int r_in = sub * 32 + lane;
    // logits are streamed out: keep L2 for the operand tiles
    const uint64_t st_pol = ptx::policy_evict_first();
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t t = blockIdx.x; t < P.n_tiles; t += gridDim.x) {
      const int64_t row = static_cast<int64_t>(t % P.n_mblk) * kBM + r_in;
      const int32_t vt = static_cast<int32_t>(t / P.n_mblk);
      const int32_t n0 = vt * kBN;
      const bool row_ok = row < P.n_rows;
      const int32_t yrel = row_ok ? P.target[row] - n0 : -1;
      const int32_t ncols = min(kBN, P.V - n0);
      ptx::mbar_wait_u32(tfull_bar(acc), acc_phase);
      tc::fence_after_sync();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(sub * 32) << 16) +
                             static_cast<uint32_t>(acc * kBN);
      const float2 part = epilogue_row(taddr, row, row_ok, n0, ncols, yrel, P, st_pol);
      tc::fence_before_sync();
      ptx::mbar_arrive_u32(tempty_bar(acc));
      if (row_ok) P.partials[row * P.n_vt + vt] = part;
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc<kTmemCols>(tmem_base);
  }
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of two CTAs on one TPC computes a
// 256-token x 256-column tile. Each CTA stages its 128 token rows of hidden
// and its 128-row half of the weight tile; the leader's single thread issues
// M=256 MMAs that read both CTAs' shared memory and write each CTA's half of
// the accumulator into its own TMEM. Per SM this halves the weight-operand
// traffic of the 1-SM kernel (32 KB instead of 48 KB staged per k-step for the
// same MMA work).
//   full[s]   leader only; both CTAs' TMA bytes complete on it
//   empty[s]  both CTAs; multicast tcgen05.commit from the leader
//   tfull[b]  both CTAs; multicast commit after the tile's last k-step
//   tempty[b] leader only; one arrive per epilogue warp of either CTA (8)
// ---------------------------------------------------------------------------
constexpr int kPStages = 7;
constexpr int kPABytes = 128 * kBK * 2;  // 16 KB: this CTA's 128 token rows
constexpr int kPBBytes = 128 * kBK * 2;  // 16 KB: this CTA's half of the weight tile
constexpr int kPStageBytes = kPABytes + kPBBytes;
constexpr size_t kPSmemBytes = 1024 + kPStages * kPStageBytes + 256;
// dW (EPI 2): one stage fewer, and per epilogue warp two 32 x 32 fp32 staging
// boxes (SWIZZLE_128B, 4 KB each) for the TMA reduce-add into dW
constexpr int kPStagesDw = 6;
constexpr uint32_t kDwBoxBytes = 32 * 32 * 4;
constexpr size_t kPSmemBytesDw = 1024 + kPStagesDw * kPStageBytes + 1024 + 8 * kDwBoxBytes;
static_assert(kPSmemBytesDw <= 232448, "dW smem");
constexpr int kPStagesWide = 4;  // 48 KB stages (A 16 KB + two B halves)
// + 1024 barrier block + 8 x 4 KB fp32 staging boxes for the TMA-store epilogue
constexpr size_t kPSmemBytesWide = 1024 + kPStagesWide * (kPABytes + 2 * kPBBytes) + 1024 + 8 * 4096;
static_assert(kPSmemBytesWide <= 232448, "wide smem");
constexpr uint32_t kMnBoxBytes = kBK * 128;  // MN-major box: kBK K-rows x 64 elements

// EPI 0: logits + LSE partials (the forward). EPI 3: the same with the logits
// leaving through swizzled staging boxes and TMA stores (epilogue_row_tma). EPI 1: C = A B^T as fp32 split-K
// partials (A [M x K], B [N x K], both K-major; M = tokens, N = P.V columns,
// K = P.H), e.g. dhidden = dlogits [T x V] * (W^T [H x V])^T.
// EPI 2: C += A^T B with both operands MN-major (A [K x M], B [K x N] row-major,
// the reduction over their rows; M = P.n_rows, N = P.V, K = P.H), i.e. the
// weight gradient dW [V x H] += dlogits [T x V]^T * hidden [T x H]. Each stage
// holds two 64-wide MN boxes per operand (LBO = one box); the fp32 epilogue
// adds the tile into C (each tile is owned by exactly one unit: no split).
template <int EPI, bool MC = false, bool WIDE = false>
__global__ void __launch_bounds__(kThreads, 1)
    lmhead_fwd_pair_kernel(const __grid_constant__ CUtensorMap tm_x,
                           const __grid_constant__ CUtensorMap tm_w,
                           const __grid_constant__ CUtensorMap tm_c, const LmParams P) {
  // WIDE (EPI 1 only): a 256 x 512 tile per pair, two N = 256 MMAs per k-step
  // into all 512 TMEM columns (no accumulator double buffer: with a 151,936-long
  // reduction the epilogue is ~0.3% of a unit); each A tile feeds twice the MMA
  // work, so the operand traffic per flop drops by a quarter
  static_assert(!WIDE || (EPI == 1 && !MC), "WIDE is the plain-GEMM mode only");
  constexpr int kNT = WIDE ? 2 * kBN : kBN;           // N columns per unit
  constexpr int kBStage = (kNT / kBN) * kPBBytes;     // this CTA's B bytes per stage
  constexpr int kStageB = kPABytes + kBStage;
  // EPI 2 / 3: one stage fewer, for the epilogue's staging boxes
  constexpr int kPStages = EPI >= 2 ? kPStagesDw : WIDE ? kPStagesWide : ::copris_b200::kPStages;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t sA = base;
  const uint32_t sB = base + kPStages * kPABytes;
  const uint32_t bars = base + kPStages * kStageB;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (kPStages + s); };
  auto tfull_bar = [&](int b) { return bars + 8u * (2 * kPStages + b); };
  auto tempty_bar = [&](int b) { return bars + 8u * (2 * kPStages + 2 + b); };
  const uint32_t tmem_slot = bars + 8u * (2 * kPStages + 4);
  const uint32_t stg = bars + 1024;  // EPI 2 staging (1024-aligned)
  volatile uint32_t* tmem_slot_ptr = reinterpret_cast<volatile uint32_t*>(
      smem_raw + (tmem_slot - ptx::smem_u32(smem_raw)));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  // MC: a 4-CTA cluster of two pairs on vertically adjacent tiles (same vocab /
  // N tile, consecutive token pairs); each B half is loaded once by pair 0 and
  // multicast to both pairs. prank = rank in the pair, lrank = pair leader.
  const uint32_t prank = rank & 1u, pair = MC ? rank >> 1 : 0u, lrank = rank & ~1u;
  const bool leader = prank == 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kPStages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(full_bar(s)));
      // MC: both pair leaders release a slot (B was multicast into both pairs)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(empty_bar(s)), "n"(MC ? 2 : 1));
    }
    for (int b = 0; b < 2; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tfull_bar(b)));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(tempty_bar(b)));
    }
    ptx::fence_mbarrier_init();
    tc::prefetch_tensormap(&tm_x);
    tc::prefetch_tensormap(&tm_w);
    if (EPI >= 2 || WIDE) tc::prefetch_tensormap(&tm_c);
  }
  if (warp == 1) tc::tmem_alloc_pair<kTmemCols>(tmem_slot);
  tc::fence_before_sync();
  ptx::cluster_sync_all();
  tc::fence_after_sync();
  const uint32_t tmem_base = *tmem_slot_ptr;

  const int nk = (P.H + kBK - 1) / kBK;
  const int64_t n_mpair = (P.n_rows + 255) / 256;
  const int32_t n_split = EPI == 1 ? P.n_split : 1;
  const int64_t n_mu = MC ? (n_mpair + 1) / 2 : n_mpair;  // token pairs (MC: pairs of pairs)
  const int64_t n_units = n_mu * P.n_vt * n_split;
  // k-block range of a unit's split
  auto k_range = [&](int64_t u, int& kb0, int& kb1) {
    if (EPI == 1) {
      const int64_t sp = u / (n_mu * P.n_vt);
      kb0 = static_cast<int>(sp * P.k_per_split);
      kb1 = min(nk, kb0 + P.k_per_split);
    } else {
      kb0 = 0;
      kb1 = nk;
    }
  };
  // Grouped raster: units sweep every vocab tile for a group of `grp` token
  // pairs before moving on, so the group's hidden rows stay L2-resident while
  // each weight tile is shared by the group's concurrently running clusters.
  const int64_t grp = P.group < n_mu ? static_cast<int64_t>(P.group) : n_mu;
  auto unit_coords = [&](int64_t u, int64_t& mp, int32_t& vt) {
    if (EPI == 1) u %= n_mu * P.n_vt;  // split-major: the same raster in every split
    const int64_t per = grp * P.n_vt;
    const int64_t g = u / per, w = u % per;
    const int64_t gsz = grp < n_mu - g * grp ? grp : n_mu - g * grp;  // last group may be short
    vt = static_cast<int32_t>(w / gsz);
    mp = g * grp + w % gsz;
    if (MC) mp = 2 * mp + pair;  // may be one past the last pair: rows masked, TMA zero-fills
  };
  const int64_t cid = blockIdx.x >> (MC ? 2 : 1), ncl = gridDim.x >> (MC ? 2 : 1);
  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer (both CTAs) =====
      // dW (EPI 2): COPRIS_DW_POLICY bit 0 keeps A (dlogits slices) and bit 1
      // keeps B (hidden) at evict_last against the dW read-modify-write stream
      const uint64_t pol_w = EPI == 2 && (P.a_evict_first & 2) ? ptx::policy_evict_last()
                                                               : ptx::policy_evict_normal();
      // forward: the hidden block is small and reused by every vocab tile;
      // GEMM mode: A (dlogits) is a large stream, no reason to pin it
      const uint64_t pol_x = EPI == 1   ? (P.a_evict_first ? ptx::policy_evict_first()
                                                           : ptx::policy_evict_normal())
                             : EPI == 2 ? ((P.a_evict_first & 1) ? ptx::policy_evict_last()
                                                                 : ptx::policy_evict_normal())
                                        : ptx::policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t u = cid; u < n_units; u += ncl) {
        int64_t mp;
        int32_t vt;
        unit_coords(u, mp, vt);
        const int32_t m0 = static_cast<int32_t>(mp) * 256 + 128 * prank;
        const int32_t n0 = vt * kNT + 128 * prank;
        int kb0, kb1;
        k_range(u, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait_u32(empty_bar(stage), phase ^ 1u);
          const uint32_t fb = ptx::mapa(full_bar(stage), lrank);
          if (leader) ptx::mbar_arrive_expect_tx_u32(full_bar(stage), 2 * kStageB);
          if constexpr (EPI == 2) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              tc::tma_load_2d_pair(sA + stage * kPABytes + j * kMnBoxBytes, &tm_x, fb, m0 + 64 * j,
                                   kb * kBK, pol_x);
              tc::tma_load_2d_pair(sB + stage * kBStage + j * kMnBoxBytes, &tm_w, fb, n0 + 64 * j,
                                   kb * kBK, pol_w);
            }
          } else if constexpr (MC) {
            tc::tma_load_2d_pair(sA + stage * kPABytes, &tm_x, fb, kb * kBK, m0, pol_x);
            if (pair == 0)
              tc::tma_load_2d_pair_mc(sB + stage * kBStage, &tm_w, fb, kb * kBK, n0,
                                      static_cast<uint16_t>(0x5u << prank), pol_w);
          } else {
            tc::tma_load_2d_pair(sA + stage * kPABytes, &tm_x, fb, kb * kBK, m0, pol_x);
            tc::tma_load_2d_pair(sB + stage * kBStage, &tm_w, fb, kb * kBK, n0, pol_w);
            if constexpr (WIDE)
              tc::tma_load_2d_pair(sB + stage * kBStage + kPBBytes, &tm_w, fb, kb * kBK, n0 + kBN,
                                   pol_w);
          }
          if (++stage == kPStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {
      // ===== MMA issuer (leader CTA) =====
      constexpr uint32_t idesc = tc::idesc_bf16_f32<256, kBN, EPI == 2, EPI == 2>();
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int64_t u = cid; u < n_units; u += ncl) {
        ptx::mbar_wait_u32(tempty_bar(acc), acc_phase ^ 1u);
        tc::fence_after_sync();
        const uint32_t d = tmem_base + static_cast<uint32_t>(WIDE ? 0 : acc * kBN);
        int kb0, kb1;
        k_range(u, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait_u32(full_bar(stage), phase);
          tc::fence_after_sync();
          const uint32_t a = sA + stage * kPABytes, b = sB + stage * kBStage;
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            // K-major: 16 elements = 32 bytes along the swizzled row;
            // MN-major: 16 K-rows = two 1024-byte atoms
            const uint64_t da = EPI == 2 ? tc::smem_desc_sw128_mn(a + 2048 * k, kMnBoxBytes)
                                         : tc::smem_desc_sw128(a + 32 * k);
            const uint64_t db = EPI == 2 ? tc::smem_desc_sw128_mn(b + 2048 * k, kMnBoxBytes)
                                         : tc::smem_desc_sw128(b + 32 * k);
            tc::mma_bf16_ss_pair(d, da, db, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
            if constexpr (WIDE)
              tc::mma_bf16_ss_pair(d + kBN, da, tc::smem_desc_sw128(b + kPBBytes + 32 * k), idesc,
                                   (kb != kb0 || k != 0) ? 1u : 0u);
          }
          tc::commit_pair(empty_bar(stage), MC ? 0xF : 0x3);
          if (++stage == kPStages) {
            stage = 0;
            phase ^= 1u;
          }
        }
        tc::commit_pair(tfull_bar(acc), static_cast<uint16_t>(0x3u << (2 * pair)));
        if (WIDE) {
          acc_phase ^= 1u;
        } else if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1u;
        }
      }
    }
  } else {
    // ===== epilogue (both CTAs): this CTA's 128 token rows x 256 columns =====
    const int sub = warp & 3;
    const int r_in = sub * 32 + lane;
    // logits are streamed out: keep L2 for the operand tiles
    const uint64_t st_pol = ptx::policy_evict_first();
    int dw_buf = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t u = cid; u < n_units; u += ncl) {
      int64_t mp;
      int32_t vt;
      unit_coords(u, mp, vt);
      const int64_t row = mp * 256 + 128 * prank + r_in;
      const int32_t n0 = vt * kNT;
      const bool row_ok = row < P.n_rows;
      const int32_t ncols = min(kNT, P.V - n0);
      ptx::mbar_wait_u32(tfull_bar(acc), acc_phase);
      tc::fence_after_sync();
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(sub * 32) << 16) +
                             static_cast<uint32_t>(WIDE ? 0 : acc * kBN);
      if constexpr (EPI == 2) {
        // C tile += the accumulator through TMA reduce-add: each warp stages
        // its 32 rows x 32 columns in a swizzled box (16-byte chunk j of row
        // r at j ^ (r & 7): conflict-free) and one lane issues the bulk add;
        // two boxes per warp alternate so staging overlaps the adds in flight
        const int32_t row0 = static_cast<int32_t>(mp * 256 + 128 * prank + sub * 32);
#pragma unroll 1
        for (int c = 0; c < kBN; c += 32) {
          uint32_t r[32];
          tc::tmem_ld_32x32b_x32(taddr + c, r);
          tc::tmem_wait_ld();
          if (c >= ncols) break;  // uniform across the warp
          const uint32_t box = stg + static_cast<uint32_t>(sub * 2 + dw_buf) * kDwBoxBytes;
          if (lane == 0) tc::bulk_wait_group_read<1>();  // the add issued 2 boxes ago read `box`
          __syncwarp();
#pragma unroll
          for (int q = 0; q < 8; ++q)
            ptx::sts_v4(box + lane * 128 + ((q ^ (lane & 7)) << 4),
                        make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]));
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tc::tma_reduce_add_2d(&tm_c, box, n0 + c, row0);
            tc::bulk_commit_group();
          }
          dw_buf ^= 1;
        }
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_remote(ptx::mapa(tempty_bar(acc), lrank));
      } else if constexpr (EPI == 1 && WIDE) {
        // fp32 partial tile through swizzled 32 x 32 staging boxes and 3-D TMA
        // stores (columns, rows, split: the box is clipped per split)
        const int32_t sp = static_cast<int32_t>(u / (n_mu * P.n_vt));
        const int32_t row0 = static_cast<int32_t>(mp * 256 + 128 * prank + sub * 32);
        const uint32_t box0 = stg + static_cast<uint32_t>(sub) * 8192u;
#pragma unroll 1
        for (int c = 0; c < kNT; c += 32) {
          uint32_t r[32];
          tc::tmem_ld_32x32b_x32(taddr + c, r);
          tc::tmem_wait_ld();
          if (c >= ncols) break;  // uniform across the warp
          const uint32_t box = box0 + static_cast<uint32_t>(dw_buf) * kDwBoxBytes;
          if (lane == 0) tc::bulk_wait_group_read<1>();
          __syncwarp();
#pragma unroll
          for (int q = 0; q < 8; ++q)
            ptx::sts_v4(box + lane * 128 + ((q ^ (lane & 7)) << 4),
                        make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]));
          ptx::fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tc::tma_store_3d(&tm_c, box, n0 + c, row0, sp, st_pol);
            tc::bulk_commit_group();
          }
          dw_buf ^= 1;
        }
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_remote(ptx::mapa(tempty_bar(acc), lrank));
      } else if constexpr (EPI == 1) {
        // fp32 tile row straight from TMEM to this split's partial matrix
        const int64_t sp = u / (n_mu * P.n_vt);
        float* out = P.c_out + sp * P.split_stride + row * P.ldc + n0;
#pragma unroll 1
        for (int c = 0; c < kNT; c += 32) {
          uint32_t r[32];
          tc::tmem_ld_32x32b_x32(taddr + c, r);
          tc::tmem_wait_ld();
          if (c >= ncols) break;  // uniform across the warp
          if (row_ok) {
            if (c + 32 <= ncols) {
#pragma unroll
              for (int q = 0; q < 8; ++q)
                ptx::st_global_v4_hint(out + c + 4 * q,
                                       make_uint4(r[4 * q], r[4 * q + 1], r[4 * q + 2], r[4 * q + 3]),
                                       st_pol);
            } else {
              for (int j = 0; j < 32 && c + j < ncols; ++j) out[c + j] = __uint_as_float(r[j]);
            }
          }
        }
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_remote(ptx::mapa(tempty_bar(acc), lrank));
      } else if constexpr (EPI == 3) {
        const bool stats = P.partials != nullptr;  // nullptr: logits only (uniform)
        const int32_t yrel = row_ok && stats ? P.target[row] - n0 : -1;
        const int32_t row0 = static_cast<int32_t>(mp * 256 + 128 * prank + sub * 32);
        const float2 part = epilogue_row_tma(taddr, row0, n0, ncols, yrel, &tm_c,
                                             stg + static_cast<uint32_t>(sub) * 8192u, dw_buf,
                                             st_pol, stats);
        tc::fence_before_sync();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_remote(ptx::mapa(tempty_bar(acc), lrank));
        if (row_ok && stats) P.partials[row * P.n_vt + vt] = part;
      } else {
      const int32_t yrel = row_ok ? P.target[row] - n0 : -1;
      const float2 part = epilogue_row(taddr, row, row_ok, n0, ncols, yrel, P, st_pol);
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive_remote(ptx::mapa(tempty_bar(acc), lrank));
      if (row_ok) P.partials[row * P.n_vt + vt] = part;
      }
      if (WIDE) {
        acc_phase ^= 1u;
      } else if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1u;
      }
    }
  }
  if ((EPI >= 2 || WIDE) && warp >= 2 && lane == 0) tc::bulk_wait_group<0>();
  tc::fence_before_sync();
  __syncthreads();
  ptx::cluster_sync_all();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc_pair<kTmemCols>(tmem_base);
  }
}

// Split-K finish of the plain GEMM: out[m][n] = bf16(sum_s part[s][m][n]) in a
// fixed split order (deterministic). 4 columns per thread.
__global__ void __launch_bounds__(256)
    splitk_sum_bf16_kernel(const float* __restrict__ part, int64_t split_stride, int32_t n_split,
                           int64_t M, int32_t N, int64_t ldc, __nv_bfloat16* __restrict__ out,
                           int64_t ldo) {
  const int32_t nq = N / 4;
  const int64_t total = M * nq;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t m = i / nq;
    const int32_t n = static_cast<int32_t>(i % nq) * 4;
    float4 a = *reinterpret_cast<const float4*>(part + m * ldc + n);
    for (int s = 1; s < n_split; ++s) {
      const float4 b = *reinterpret_cast<const float4*>(part + s * split_stride + m * ldc + n);
      a.x += b.x;
      a.y += b.y;
      a.z += b.z;
      a.w += b.w;
    }
    *reinterpret_cast<uint2*>(out + m * ldo + n) =
        make_uint2(ptx::pack_bf16x2(a.x, a.y), ptx::pack_bf16x2(a.z, a.w));
  }
}

// (cur_lp, lse) per token from the tile partials: one warp per token; the
// target logit is read back from the stored (rounded) logits.
__global__ void __launch_bounds__(256)
    lse_merge_kernel(const float2* __restrict__ partials, int32_t n_vt,
                     const __nv_bfloat16* __restrict__ logits, int64_t ld,
                     const int32_t* __restrict__ target, int64_t n_rows, int32_t V,
                     float* __restrict__ out_lp, float* __restrict__ out_lse, uint32_t* err) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < n_rows;
       r += warps) {
    const float2* pr = partials + r * n_vt;
    float m = -INFINITY, s = 0.f;
    for (int i = lane; i < n_vt; i += 32) {
      const float2 p = pr[i];
      if (p.x > m) {
        s = s * ptx::ex2((m - p.x) * kLog2e) + p.y;
        m = p.x;
      } else {
        s += p.y * ptx::ex2((p.x - m) * kLog2e);
      }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, m, off);
      const float os = __shfl_xor_sync(0xffffffffu, s, off);
      const float M = fmaxf(m, om);
      if (M != -INFINITY) {
        s = s * ptx::ex2((m - M) * kLog2e) + os * ptx::ex2((om - M) * kLog2e);
        m = M;
      }
    }
    if (lane == 0) {
      const int32_t y = target[r];
      const bool ok = static_cast<uint32_t>(y) < static_cast<uint32_t>(V);
      const float zy = ok ? __bfloat162float(logits[r * ld + y]) : 0.f;
      const LogProb lp = finish_logprob(m, s, zy, ok);
      if (!ok) atomicOr(err, ERR_TOKEN_OOV);
      out_lp[r] = lp.cur;
      if (out_lse) out_lse[r] = static_cast<float>(lp.lse);
    }
  }
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// K-major bf16 matrix [rows x k] with row stride ld elements, box [box_rows x 64].
bool make_map(CUtensorMap* map, const void* ptr, int64_t rows, int32_t k, int64_t ld,
              uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(k), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp32 matrix [rows x cols] with row stride ld elements, 32 x 32 boxes
// (128-byte rows, SWIZZLE_128B): the TMA reduce-add target of the dW epilogue.
bool make_map_f32_box32(CUtensorMap* map, const void* ptr, int64_t rows, int32_t cols, int64_t ld) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
  const cuuint32_t box[2] = {32, 32};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp32 partial matrices [splits][rows][cols] (contiguous), 32 x 32 x 1 boxes,
// SWIZZLE_128B: the TMA-store target of the 256 x 512 plain-GEMM epilogue.
bool make_map_f32_3d_box32(CUtensorMap* map, const void* ptr, int64_t splits, int64_t rows,
                           int32_t cols) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows),
                              static_cast<cuuint64_t>(splits)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(cols) * 4,
                                 static_cast<cuuint64_t>(cols) * 4 * static_cast<cuuint64_t>(rows)};
  const cuuint32_t box[3] = {32, 32, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(ptr), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int32_t lmhead_num_vtiles(int32_t vocab) { return (vocab + kBN - 1) / kBN; }

cudaError_t launch_lmhead_fwd(const void* hidden, int64_t ld_h, const void* weight, int64_t ld_w,
                              int64_t n_rows, int32_t H, int32_t V, const int32_t* target,
                              void* logits, int64_t ld, float* partials, int num_sms,
                              const Tuning& tu, cudaStream_t stream, LaunchInfo* info) {
  CUtensorMap tx, tw;
  if (!make_map(&tx, hidden, n_rows, H, ld_h, kBM) || !make_map(&tw, weight, V, H, ld_w, kBN))
    return cudaErrorInvalidValue;

  LmParams p;
  p.n_rows = n_rows;
  p.H = H;
  p.V = V;
  p.n_mblk = static_cast<int32_t>((n_rows + kBM - 1) / kBM);
  p.n_vt = lmhead_num_vtiles(V);
  p.n_tiles = static_cast<int64_t>(p.n_mblk) * p.n_vt;
  p.logits = static_cast<__nv_bfloat16*>(logits);
  p.ld = ld;
  p.partials = reinterpret_cast<float2*>(partials);
  p.target = target;
  p.group = std::max(1, tu.lmhead_group);
  // logits only (no partials): the CTA-pair kernel's TMA-store epilogue skips the
  // statistics; the other epilogues always produce them
  if (!partials && (tu.lmhead_impl == 1 || tu.lmhead_tma_store == 0 || V % 8 != 0))
    return cudaErrorInvalidValue;
  if (tu.lmhead_impl == 1) {
    cudaError_t ea = allow_dyn_smem(reinterpret_cast<const void*>(lmhead_fwd_kernel), static_cast<int>(kSmemBytes));
    if (ea != cudaSuccess) return ea;
    const int grid = static_cast<int>(std::min<int64_t>(p.n_tiles, num_sms));
    lmhead_fwd_kernel<<<grid, kThreads, kSmemBytes, stream>>>(tx, tw, p);
    if (info) *info = LaunchInfo{num_sms, 1, grid, "lmhead_fwd_kernel"};
    return cudaGetLastError();
  }
  // the pair kernel stages half of the weight tile per CTA: 128-row boxes
  if (!make_map(&tw, weight, V, H, ld_w, 128)) return cudaErrorInvalidValue;
  // per call: the attribute is per device, and one process may drive several
  // logits through staging boxes + TMA stores (EPI 3) unless lmhead_tma_store = 0;
  // only when a row is a whole number of 16-byte pieces (V % 8 == 0): TMA clips
  // a store box at 16-byte granularity, so it would write the row padding
  const bool tma_store = tu.lmhead_tma_store != 0 && V % 8 == 0;
  CUtensorMap tl = tw;
  if (tma_store && !make_map(&tl, logits, n_rows, V, ld, 32)) return cudaErrorInvalidValue;
  auto kern = tma_store ? lmhead_fwd_pair_kernel<3> : lmhead_fwd_pair_kernel<0>;
  const size_t smem = tma_store ? kPSmemBytesDw : kPSmemBytes;
  cudaError_t ea = allow_dyn_smem(reinterpret_cast<const void*>(kern), static_cast<int>(smem));
  if (ea != cudaSuccess) return ea;
  const int64_t units = (n_rows + 255) / 256 * p.n_vt;
  const int grid = static_cast<int>(std::min<int64_t>(2 * units, num_sms & ~1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr_cl[1];
  attr_cl[0].id = cudaLaunchAttributeClusterDimension;
  attr_cl[0].val.clusterDim.x = 2;
  attr_cl[0].val.clusterDim.y = 1;
  attr_cl[0].val.clusterDim.z = 1;
  cfg.attrs = attr_cl;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tx, tw, tl, p);
  if (info)
    *info = LaunchInfo{num_sms, 2, grid,
                       tma_store ? "lmhead_fwd_pair_kernel<tma_store>" : "lmhead_fwd_pair_kernel"};
  return e != cudaSuccess ? e : cudaGetLastError();
}

static bool gemm_wide(const Tuning& tu) {
  // default on; gemm_wide = 0 selects the 256 x 256 tile
  return tu.gemm_wide != 0 && tu.gemm_mc == 0;
}

int32_t gemm_nt_splits(int64_t M, int32_t N, int num_sms, const Tuning& tu) {
  if (tu.gemm_splits > 0) return tu.gemm_splits;
  const int64_t clusters = num_sms / 2;
  if (gemm_wide(tu)) {
    // 256 x 512 tiles are few: pick the split count whose units fill the last
    // wave of clusters best (ties: fewer splits, less partial traffic)
    const int64_t base = (M + 255) / 256 * ((N + 2 * kBN - 1) / (2 * kBN));
    int32_t best = 1;
    double best_eff = -1.0;
    for (int32_t s = 1; s <= 8; ++s) {
      const int64_t u = base * s;
      const int64_t rounds = (u + clusters - 1) / clusters;
      const double eff = static_cast<double>(u) / static_cast<double>(rounds * clusters);
      if (eff > best_eff + 1e-9) {
        best_eff = eff;
        best = s;
      }
    }
    return best;
  }
  const int64_t units = (M + 255) / 256 * ((N + kBN - 1) / kBN);
  int64_t s = (4 * clusters + units - 1) / units;  // >= ~4 waves of cluster tiles
  if (s < 1) s = 1;
  if (s > 8) s = 8;
  return static_cast<int32_t>(s);
}

cudaError_t launch_gemm_nt_bf16(const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M,
                                int32_t N, int32_t K, void* out, int64_t ldo, float* work,
                                int32_t n_split, int num_sms, const Tuning& tu,
                                cudaStream_t stream, LaunchInfo* info) {
  if (M == 0 || N == 0) return cudaSuccess;
  CUtensorMap ta, tb;
  if (!make_map(&ta, A, M, K, lda, 128) || !make_map(&tb, B, N, K, ldb, 128))
    return cudaErrorInvalidValue;
  const int nk = (K + kBK - 1) / kBK;
  if (n_split < 1) n_split = 1;
  if (n_split > nk) n_split = nk;
  LmParams p{};
  p.n_rows = M;
  p.H = K;
  p.V = N;
  p.n_vt = (N + kBN - 1) / kBN;
  p.group = std::max(1, tu.lmhead_group);
  p.a_evict_first = tu.gemm_a_evict_first;
  p.c_out = work;
  p.ldc = N;
  p.split_stride = M * static_cast<int64_t>(N);
  p.n_split = n_split;
  p.k_per_split = (nk + n_split - 1) / n_split;
  p.n_split = (nk + p.k_per_split - 1) / p.k_per_split;  // no empty split
  // default: 256 x 512 tiles per pair (two MMAs per k-step); gemm_wide = 0:
  // 256 x 256 tiles; gemm_mc = 1: 256 x 256 tiles on 4-CTA clusters with the
  // W^T halves multicast to two token pairs
  const bool mc = tu.gemm_mc != 0;
  const bool wide = gemm_wide(tu);
  auto kern = mc     ? lmhead_fwd_pair_kernel<1, true>
              : wide ? lmhead_fwd_pair_kernel<1, false, true>
                     : lmhead_fwd_pair_kernel<1, false>;
  const size_t smem = wide ? kPSmemBytesWide : kPSmemBytes;
  if (wide) p.n_vt = (N + 2 * kBN - 1) / (2 * kBN);
  cudaError_t e = allow_dyn_smem(reinterpret_cast<const void*>(kern), static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  const int cl = mc ? 4 : 2;
  const int64_t n_mu = mc ? ((M + 255) / 256 + 1) / 2 : (M + 255) / 256;
  const int64_t units = n_mu * p.n_vt * p.n_split;
  const int grid = static_cast<int>(std::min<int64_t>(cl * units, num_sms & ~(cl - 1)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr_cl[1];
  attr_cl[0].id = cudaLaunchAttributeClusterDimension;
  attr_cl[0].val.clusterDim.x = cl;
  attr_cl[0].val.clusterDim.y = 1;
  attr_cl[0].val.clusterDim.z = 1;
  cfg.attrs = attr_cl;
  cfg.numAttrs = 1;
  if (mc) {
    // 4-CTA clusters do not tile every GPC: size the persistent grid to the
    // clusters that are co-resident
    int max_cl = 0;
    if (cudaOccupancyMaxActiveClusters(&max_cl, kern, &cfg) == cudaSuccess && max_cl > 0)
      cfg.gridDim = dim3(static_cast<unsigned>(std::min<int64_t>(cl * units, cl * max_cl)));
  }
  CUtensorMap tp = tb;
  if (wide && !make_map_f32_3d_box32(&tp, work, p.n_split, M, N)) return cudaErrorInvalidValue;
  e = cudaLaunchKernelEx(&cfg, kern, ta, tb, tp, p);
  if (e != cudaSuccess) return e;
  const int64_t quads = M * (N / 4);
  const int64_t blocks = std::min<int64_t>((quads + 255) / 256, static_cast<int64_t>(num_sms) * 8);
  splitk_sum_bf16_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
      work, p.split_stride, p.n_split, M, N, N, static_cast<__nv_bfloat16*>(out), ldo);
  if (info)
    *info = LaunchInfo{num_sms, cl, static_cast<int>(cfg.gridDim.x),
                       mc     ? "lmhead_fwd_pair_kernel<gemm,mc>"
                       : wide ? "lmhead_fwd_pair_kernel<gemm,wide>"
                              : "lmhead_fwd_pair_kernel<gemm>"};
  return cudaGetLastError();
}

cudaError_t launch_gemm_tn_acc_f32(const void* A, int64_t lda, const void* B, int64_t ldb,
                                   int64_t K, int32_t M, int32_t N, float* c, int64_t ldc,
                                   int num_sms, const Tuning& tu, cudaStream_t stream,
                                   LaunchInfo* info) {
  if (K == 0 || M == 0 || N == 0) return cudaSuccess;
  CUtensorMap tc_map;
  if (!make_map_f32_box32(&tc_map, c, M, N, ldc)) return cudaErrorInvalidValue;
  LmParams p{};
  p.n_rows = M;
  p.V = N;
  p.n_vt = (N + kBN - 1) / kBN;
  // raster: every H tile of one vocab pair before the next (group 1), so the
  // 16 concurrent users of a dlogits slice share one DRAM read; the hidden
  // block is kept at evict_last (policy bit 1) and re-read from L2
  p.group = std::max(1, tu.dw_group);
  p.a_evict_first = tu.dw_policy;
  p.c_out = c;
  p.ldc = ldc;
  p.n_split = 1;
  // the token reduction runs in launches of <= kchunk rows, in order, so the
  // hidden block of one launch (kchunk x H bf16) stays L2-resident
  const int64_t kchunk = std::max<int64_t>(kBK, tu.dw_kchunk / kBK * kBK);
  cudaError_t e = allow_dyn_smem(reinterpret_cast<const void*>(lmhead_fwd_pair_kernel<2>), static_cast<int>(kPSmemBytesDw));
  if (e != cudaSuccess) return e;
  const int64_t units = (static_cast<int64_t>(M) + 255) / 256 * p.n_vt;
  const int grid = static_cast<int>(std::min<int64_t>(2 * units, num_sms & ~1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kPSmemBytesDw;
  cfg.stream = stream;
  cudaLaunchAttribute attr_cl[1];
  attr_cl[0].id = cudaLaunchAttributeClusterDimension;
  attr_cl[0].val.clusterDim.x = 2;
  attr_cl[0].val.clusterDim.y = 1;
  attr_cl[0].val.clusterDim.z = 1;
  cfg.attrs = attr_cl;
  cfg.numAttrs = 1;
  for (int64_t k0 = 0; k0 < K; k0 += kchunk) {
    const int64_t kn = std::min(kchunk, K - k0);
    // MN-major boxes: 64 columns (the contiguous dimension) x kBK rows
    CUtensorMap ta, tb;
    if (!make_map(&ta, static_cast<const __nv_bfloat16*>(A) + k0 * lda, kn, M, lda, kBK) ||
        !make_map(&tb, static_cast<const __nv_bfloat16*>(B) + k0 * ldb, kn, N, ldb, kBK))
      return cudaErrorInvalidValue;
    p.H = static_cast<int32_t>(kn);
    e = cudaLaunchKernelEx(&cfg, lmhead_fwd_pair_kernel<2>, ta, tb, tc_map, p);
    if (e != cudaSuccess) return e;
  }
  if (info) *info = LaunchInfo{num_sms, 2, grid, "lmhead_fwd_pair_kernel<dW>"};
  return cudaGetLastError();
}

cudaError_t launch_lse_merge(const float* partials, int32_t n_vt, const void* logits, int64_t ld,
                             const int32_t* target, int64_t n_rows, int32_t V, float* out_lp,
                             float* out_lse, uint32_t* err, int num_sms, cudaStream_t stream) {
  const int64_t blocks = std::min<int64_t>((n_rows + 7) / 8, static_cast<int64_t>(num_sms) * 8);
  lse_merge_kernel<<<static_cast<int>(blocks), 256, 0, stream>>>(
      reinterpret_cast<const float2*>(partials), n_vt,
      static_cast<const __nv_bfloat16*>(logits), ld, target, n_rows, V, out_lp, out_lse, err);
  return cudaGetLastError();
}

}  // namespace copris_b200
