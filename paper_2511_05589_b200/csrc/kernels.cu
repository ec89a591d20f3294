// kernels.cu — sm_100a kernels of the CoPRIS IS-corrected loss path.
//
//   fused_tma_kernel      one HBM read of every logits row: the row is pulled
//                         into shared memory with TMA bulk copies (split over a
//                         CL-CTA cluster at large vocab; partial max/sum/target
//                         exchanged through DSMEM), reduced once (online
//                         log-sum-exp), and dlogits are written from the
//                         shared-memory copy. Persistent: each cluster walks
//                         rows r, r + n_clusters, ... and prefetches row r+1
//                         piece by piece while finishing row r.
//   fused_stream_la_kernel  rows too large for shared memory: a TMA ring, pass 1
//                         from HBM, pass 2 from L2, dedicated scalar warp with
//                         a one-row lookahead (the default at V = 151,936).
//   fused_generic_kernel  same arithmetic for rows that are not 16-byte
//                         aligned (tiny/odd vocab); two passes through L2.
//   K1 (sequence_logprobs) is the fused kernels in gather-only mode.
//   bwd_kernel            unfused K3: second streaming pass from lse.
//   + behaviour select (K2), segment expansion, rewards, advantages and a
//     deterministic fixed-order reduction.
#include <cooperative_groups.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <type_traits>
#include <utility>

#include "kernels.cuh"
#include "ptx.cuh"
#include "token_math.cuh"
#include "fused_common.cuh"
#include "reduce.cuh"
#include "pair.cuh"

namespace cg = cooperative_groups;

namespace copris_b200 {

namespace {

// ---------------------------------------------------------------------------
// fused TMA / cluster kernel
// ---------------------------------------------------------------------------
constexpr int kPieceVec = 256;  // max 16-byte vectors per TMA piece (4 KB)
constexpr int kMaxPieces = 8;   // per warp
#ifndef COPRIS_PREFETCH_L2
#define COPRIS_PREFETCH_L2 1
#endif
constexpr bool kPrefetchL2 = COPRIS_PREFETCH_L2;

// Stores NP packed fp32 pairs (2*NP columns) as TOut at a 16-byte aligned address.
template <typename TOut, int NP>
__device__ __forceinline__ void store_pairs(TOut* p, const uint64_t* g, uint64_t pol) {
  if constexpr (sizeof(TOut) == 2) {
    if constexpr (NP == 4) {
      uint4 v{ptx::f2_to_bf16x2(g[0]), ptx::f2_to_bf16x2(g[1]), ptx::f2_to_bf16x2(g[2]),
              ptx::f2_to_bf16x2(g[3])};
      ptx::st_global_v4_hint(p, v, pol);
    } else {
      uint2 v{ptx::f2_to_bf16x2(g[0]), ptx::f2_to_bf16x2(g[1])};
      *reinterpret_cast<uint2*>(p) = v;
    }
  } else {
#pragma unroll
    for (int i = 0; i < NP; i += 2) {
      uint4 v{static_cast<uint32_t>(g[i]), static_cast<uint32_t>(g[i] >> 32),
              static_cast<uint32_t>(g[i + 1]), static_cast<uint32_t>(g[i + 1] >> 32)};
      ptx::st_global_v4_hint(p + 2 * i, v, pol);
    }
  }
}

template <typename TIn, typename TOut, int CL, int WARPS, bool ENT>
__global__ void __launch_bounds__(WARPS * 32, (WARPS == 8 && CL == 1) ? 3 : 1)
    fused_tma_kernel(const LossParams P, const int32_t E) {
  using VI = Vec<TIn>;
  using PB = PassB<TIn>;
  constexpr int VN = VI::N;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[WARPS * kMaxPieces];
  __shared__ __align__(8) uint64_t xbar[2];          // cluster exchange, per row parity
  __shared__ __align__(16) float slot[2][CL][8];     // (m, s, zy, -, u, a, -, -) per rank
  __shared__ Lse red[WARPS];
  __shared__ RowBroadcast bc;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CL > 1 ? ptx::cluster_ctarank() : 0u;
  const int64_t cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  const int32_t V = P.vocab;
  const int32_t col0 = static_cast<int32_t>(rank) * E;
  const int32_t ncols = max(0, min(E, V - col0));
  const int32_t nvec = ncols / VN;
  const int32_t wv0 = static_cast<int32_t>(static_cast<int64_t>(warp) * nvec / WARPS);
  const int32_t wv1 = static_cast<int32_t>(static_cast<int64_t>(warp + 1) * nvec / WARPS);
  const int32_t npieces = (wv1 - wv0 + kPieceVec - 1) / kPieceVec;
  const int32_t pv = npieces ? (wv1 - wv0 + npieces - 1) / npieces : 0;  // balanced pieces
  const uint32_t sbase = ptx::smem_u32(smem);
  const uint32_t barbase = ptx::smem_u32(bars) + warp * kMaxPieces * 8;
  const uint32_t xbar0 = ptx::smem_u32(xbar);
  const uint32_t slot0 = ptx::smem_u32(&slot[0][0][0]);
  const uint64_t pol = ptx::policy_evict_first();
  const uint64_t pol_keep = ptx::policy_evict_last();
  const TIn* logits = static_cast<const TIn*>(P.logits);

  if (lane == 0)
    for (int p = 0; p < npieces; ++p) ptx::mbar_init(&bars[warp * kMaxPieces + p], 1);
  if (CL > 1 && threadIdx.x == 0) {
    ptx::mbar_init(&xbar[0], CL - 1);
    ptx::mbar_init(&xbar[1], CL - 1);
  }
  if (threadIdx.x == 0 || lane == 0) ptx::fence_mbarrier_init();
  __syncthreads();
  if constexpr (CL > 1) ptx::cluster_sync_all();

  auto issue = [&](int64_t row, int p) {
    const int32_t v0 = wv0 + p * pv;
    const uint32_t bytes = static_cast<uint32_t>(min(pv, wv1 - v0)) * 16u;
    const uint32_t bar = barbase + p * 8;
    ptx::mbar_arrive_expect_tx_u32(bar, bytes);
    ptx::bulk_g2s_u32(sbase + v0 * 16, logits + row * P.ld + col0 + static_cast<int64_t>(v0) * VN,
                      bytes, bar, pol);
  };

  // Row schedule: the first two rows of each CTA are static (cid, cid + ncl);
  // every later row is CLAIMED from a per-launch counter (CL == 1), so CTAs
  // that run faster take more rows and all finish within about one row of
  // each other (a static stride left the slowest CTA ~20% behind the mean).
  // Thread 0 keeps the claim one row ahead: while row r runs, r1 (the next
  // row) is known to every thread and the claim for the row after r1 is in
  // flight. Cluster launches keep the static stride (all CTAs of a cluster
  // must walk the same rows).
  const bool dyn = CL == 1 && P.row_ctr != nullptr;
  __shared__ int64_t claim_sh;
  int64_t r = cid;
  int64_t r1 = cid + ncl;
  if (lane == 0 && r < P.n_rows)
    for (int p = 0; p < npieces; ++p) issue(r, p);
  // per-row metadata, loaded one row ahead
  int32_t y_next = r < P.n_rows ? P.target[P.row_base + r] : 0;
  RowMeta meta_next{};
  if (threadIdx.x == 0 && r < P.n_rows) meta_next = load_meta(P, P.row_base + r);

  PhaseTimer tm;
  tm.start(P.trace && threadIdx.x == 0 && blockIdx.x < kTraceCtas);
  for (uint32_t it = 0; r < P.n_rows; ++it) {
    const uint32_t par = it & 1u;
    const int64_t t = P.row_base + r;
    const int32_t y = y_next;
    RowMeta meta{};
    int64_t claim = 0;
    if (threadIdx.x == 0) {
      meta = meta_next;
      if (r1 < P.n_rows) {
        meta_next = load_meta(P, P.row_base + r1);
        claim = dyn ? 2 * ncl + static_cast<int64_t>(atomicAdd(P.row_ctr, 1ull)) : r1 + ncl;
      } else {
        claim = P.n_rows;
      }
    }
    const int32_t ycol = y - col0;
    // Pull the NEXT row's slice toward L2 now, so the HBM pipe stays busy
    // through the scalar phase and pass C's refills hit L2.
    if (kPrefetchL2 && lane == 0 && r1 < P.n_rows) {
      const TIn* nrow = logits + r1 * P.ld + col0;
      for (int p = 0; p < npieces; ++p) {
        const int32_t v0 = wv0 + p * pv;
        ptx::bulk_prefetch_l2(nrow + static_cast<int64_t>(v0) * VN,
                              static_cast<uint32_t>(min(pv, wv1 - v0)) * 16u, pol_keep);
      }
    }

    // ---- pass B: log-sum-exp of this warp's slice as its pieces land --------
    Lse st = lse_empty();
    if constexpr (ENT) {
      for (int p = 0; p < npieces; ++p) {
        ptx::mbar_wait_u32(barbase + p * 8, par);
        const int32_t v0 = wv0 + p * pv, v1 = min(wv1, v0 + pv);
        for (int32_t v = v0 + lane; v < v1; v += 32) {
          float x[VN];
          VI::unpack(ptx::lds_v4(sbase + v * 16), x);
          const int jt = ycol - v * VN;
          online_update<VN, true>(x, st, static_cast<uint32_t>(jt) < VN ? jt : -1);
        }
      }
    } else {
      // nml = -inf until a finite column is seen: an all -inf vector adds 2^-inf = 0
      float m = -INFINITY, nml = -INFINITY;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
      for (int p = 0; p < npieces; ++p) {
        ptx::mbar_wait_u32(barbase + p * 8, par);
        const int32_t v0 = wv0 + p * pv, v1 = min(wv1, v0 + pv);
        // does this piece hold the target column? (warp-uniform)
        const bool tpiece = static_cast<uint32_t>(ycol - v0 * VN) < static_cast<uint32_t>((v1 - v0) * VN);
        for (int32_t v = v0 + lane; v < v1; v += 64) {
          const bool two = v + 32 < v1;
          const uint4 a = ptx::lds_v4(sbase + v * 16);
          uint4 b;
          if (two) {
            b = ptx::lds_v4(sbase + (v + 32) * 16);
          } else {
            b = uint4{PB::kNegInfWord, PB::kNegInfWord, PB::kNegInfWord, PB::kNegInfWord};
          }
          const float vm = PB::vmax(a, b);
          if (vm > m) {
            const float rs = ptx::ex2((m - vm) * kLog2e);  // 0 while m = -inf
            s0 *= rs;
            s1 *= rs;
            s2 *= rs;
            s3 *= rs;
            m = vm;
            nml = -(m * kLog2e);
          }
          float xa[VN], xb[VN];
          VI::unpack(a, xa);
          VI::unpack(b, xb);
          if (tpiece) {  // keep the target column out of s (see Lse)
            const int ja = ycol - v * VN, jb = ja - 32 * VN;
#pragma unroll
            for (int q = 0; q < VN; ++q) {
              if (q == ja) xa[q] = -INFINITY;
              if (q == jb) xb[q] = -INFINITY;
            }
          }
#pragma unroll
          for (int q = 0; q < VN; q += 2) {
            s0 += ptx::ex2(fmaf(xa[q], kLog2e, nml));
            s1 += ptx::ex2(fmaf(xa[q + 1], kLog2e, nml));
            s2 += ptx::ex2(fmaf(xb[q], kLog2e, nml));
            s3 += ptx::ex2(fmaf(xb[q + 1], kLog2e, nml));
          }
        }
      }
      st.m = m;
      st.s = (s0 + s1) + (s2 + s3);
    }
    tm.mark(0);
    warp_lse<ENT>(st);
    if (lane == 0) red[warp] = st;
    if (threadIdx.x == 0) claim_sh = claim;
    __syncthreads();
    tm.mark(1);

    // the next row's target while the scalar phase runs
    const int64_t nxt = r1;
    const bool has_next = nxt < P.n_rows;
    if (has_next) y_next = P.target[P.row_base + nxt];
    const int64_t r2 = claim_sh;  // read before the barrier that ends the scalar phase

    // ---- scalar phase (warp 0): CTA total, cluster exchange, token math -----
    if (warp == 0) {
      Lse tot = lane < WARPS ? red[lane] : lse_empty();
      warp_lse<ENT, lse_width(WARPS)>(tot);  // lane 0 holds the CTA total
      if (lane == 0) {
        float zy = 0.f;
        if (static_cast<uint32_t>(ycol) < static_cast<uint32_t>(ncols)) {
          const uint32_t za = sbase + ycol * static_cast<uint32_t>(sizeof(TIn));
          zy = sizeof(TIn) == 2 ? __uint_as_float(ptx::lds_u16(za) << 16) : __uint_as_float(ptx::lds_u32(za));
        }
        if constexpr (CL > 1) {
          const uint32_t my = slot0 + ((par * CL + rank) * 8) * 4;
          slot[par][rank][0] = tot.m;
          slot[par][rank][1] = tot.s;
          slot[par][rank][2] = zy;
          slot[par][rank][4] = tot.u;
          slot[par][rank][5] = tot.a;
#pragma unroll
          for (uint32_t c = 0; c < CL; ++c) {
            if (c == rank) continue;
            const uint32_t rem = ptx::mapa(my, c);
            ptx::st_cluster_v4(rem, tot.m, tot.s, zy, 0.f);
            if (ENT) ptx::st_cluster_v4(rem + 16, tot.u, tot.a, 0.f, 0.f);
            ptx::mbar_arrive_remote(ptx::mapa(xbar0 + par * 8, c));
          }
          ptx::mbar_wait_acq_cluster(xbar0 + par * 8, (it >> 1) & 1u);
          tot = lse_empty();
#pragma unroll
          for (int c = 0; c < CL; ++c) {
            Lse o{slot[par][c][0], slot[par][c][1], slot[par][c][4], slot[par][c][5]};
            lse_merge<ENT>(tot, o);
          }
          const uint32_t owner = static_cast<uint32_t>(y) / static_cast<uint32_t>(E);
          zy = owner < static_cast<uint32_t>(CL) ? slot[par][owner][2] : 0.f;
        }
        bc = row_scalar_phase<ENT>(P, t, meta.y, meta.st, meta.blp, meta.rl, meta.adv, tot, zy,
                                   rank == 0, meta.keep);
      }
    }
    tm.mark(2);
    __syncthreads();
    tm.mark(3);

    // ---- pass C: dlogits from the shared-memory copy; each piece is refilled
    // with the next row as soon as this warp has consumed it -----------------
    const RowBroadcast b = bc;
    const bool zero_row = (b.coef == 0.f) && (!ENT || b.eg == 0.f);
    TOut* drow = P.dlogits ? static_cast<TOut*>(P.dlogits) + r * P.ld_d + col0 : nullptr;
    for (int p = 0; p < npieces; ++p) {
      const int32_t v0 = wv0 + p * pv, v1 = min(wv1, v0 + pv);
      if (drow) {
        if (zero_row) {
          float d[VN];
#pragma unroll
          for (int j = 0; j < VN; ++j) d[j] = 0.f;
          for (int32_t v = v0 + lane; v < v1; v += 32)
            store_vec<TOut, VN>(drow + static_cast<int64_t>(v) * VN, d, pol);
        } else if constexpr (ENT) {
          for (int32_t v = v0 + lane; v < v1; v += 32) {
            float x[VN], d[VN];
            VI::unpack(ptx::lds_v4(sbase + v * 16), x);
            row_grad<VN, ENT>(x, d, col0 + v * VN, b);
            store_vec<TOut, VN>(drow + static_cast<int64_t>(v) * VN, d, pol);
          }
        } else if constexpr (sizeof(TOut) == 2 && VN == 8) {
          // |coef| folded into the exponent, sign applied to the packed bf16
          // pair (as in p2_segment): d_k = sign * 2^(z_k log2(e) - c2)
          const bool tpiece = static_cast<uint32_t>(b.y - (col0 + v0 * VN)) < static_cast<uint32_t>((v1 - v0) * VN);
          const float sdy = b.smask ? -b.dy : b.dy;
          const uint64_t l2e = ptx::f2(kLog2e, kLog2e), nc22 = ptx::f2(-b.c2, -b.c2);
          for (int32_t v = v0 + lane; v < v1; v += 64) {
            const bool two = v + 32 < v1;
            const uint4 ra = ptx::lds_v4(sbase + v * 16);
            const uint4 rb = two ? ptx::lds_v4(sbase + (v + 32) * 16) : ra;
            uint64_t pa[4], pb[4];  // packed f32x2 FFMA, as in p2_segment
            PB::unpack2(ra, pa);
            PB::unpack2(rb, pb);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              pa[q] = ptx::ex2x2(ptx::ffma2(pa[q], l2e, nc22));
              pb[q] = ptx::ex2x2(ptx::ffma2(pb[q], l2e, nc22));
            }
            if (tpiece) {
              const int ja = b.y - (col0 + v * VN), jb = ja - 32 * VN;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                if (ja == 2 * q) pa[q] = ptx::f2(sdy, ptx::f2hi(pa[q]));
                if (ja == 2 * q + 1) pa[q] = ptx::f2(ptx::f2lo(pa[q]), sdy);
                if (jb == 2 * q) pb[q] = ptx::f2(sdy, ptx::f2hi(pb[q]));
                if (jb == 2 * q + 1) pb[q] = ptx::f2(ptx::f2lo(pb[q]), sdy);
              }
            }
            const uint32_t sm = b.smask;
            const uint4 wa{ptx::f2_to_bf16x2(pa[0]) ^ sm, ptx::f2_to_bf16x2(pa[1]) ^ sm,
                           ptx::f2_to_bf16x2(pa[2]) ^ sm, ptx::f2_to_bf16x2(pa[3]) ^ sm};
            ptx::st_global_v4_hint(drow + static_cast<int64_t>(v) * VN, wa, pol);
            if (two) {
              const uint4 wb{ptx::f2_to_bf16x2(pb[0]) ^ sm, ptx::f2_to_bf16x2(pb[1]) ^ sm,
                             ptx::f2_to_bf16x2(pb[2]) ^ sm, ptx::f2_to_bf16x2(pb[3]) ^ sm};
              ptx::st_global_v4_hint(drow + static_cast<int64_t>(v + 32) * VN, wb, pol);
            }
          }
        } else {
          // two vectors per iteration: both shared-memory loads issue first
          const bool tpiece = static_cast<uint32_t>(b.y - (col0 + v0 * VN)) < static_cast<uint32_t>((v1 - v0) * VN);
          for (int32_t v = v0 + lane; v < v1; v += 64) {
            const bool two = v + 32 < v1;
            const uint4 ra = ptx::lds_v4(sbase + v * 16);
            const uint4 rb = two ? ptx::lds_v4(sbase + (v + 32) * 16) : ra;
            float xa[VN], xb[VN], da[VN], db[VN];
            VI::unpack(ra, xa);
            VI::unpack(rb, xb);
#pragma unroll
            for (int q = 0; q < VN; ++q) {
              da[q] = ptx::ex2(fmaf(xa[q], kLog2e, -b.c1)) * -b.coef;
              db[q] = ptx::ex2(fmaf(xb[q], kLog2e, -b.c1)) * -b.coef;
            }
            if (tpiece) {
              const int ja = b.y - (col0 + v * VN), jb = ja - 32 * VN;
#pragma unroll
              for (int q = 0; q < VN; ++q) {
                if (q == ja) da[q] = b.dy;
                if (q == jb) db[q] = b.dy;
              }
            }
            store_vec<TOut, VN>(drow + static_cast<int64_t>(v) * VN, da, pol);
            if (two) store_vec<TOut, VN>(drow + static_cast<int64_t>(v + 32) * VN, db, pol);
          }
        }
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0 && has_next) issue(nxt, p);
    }
    tm.mark(4);
    tm.acc[5] += 1;
    r = r1;
    r1 = r2 < P.n_rows ? r2 : P.n_rows;
  }
  tm.flush(P.trace);
  // no CTA may exit while a peer can still address its shared memory
  if constexpr (CL > 1) ptx::cluster_sync_all();
  // the row buffer is free now: it holds the trees of the fused reduction; the
  // last CTA also rearms the claim counter
  const bool self_reset = dyn && P.red_scratch != nullptr;
  if (P.out4 || self_reset) end_of_launch(P, smem, self_reset);
}

// ---------------------------------------------------------------------------
// fused TMA-streaming kernel (warp-specialised): constants and ring position
// ---------------------------------------------------------------------------
constexpr int kStreamK = 4;  // 16-byte vectors per consumer thread per ring slot

template <typename TIn, typename TOut, int CW, int KV, bool ENT>
__global__ void __launch_bounds__((CW + 2) * 32, CW <= 8 ? 2 : 1)
    fused_stream_la_kernel(const LossParams P, const int nslots, const int look, const int resident) {
  constexpr int kSlotVec = CW * 32 * KV;
  using VI = Vec<TIn>;
  constexpr int VN = VI::N;
  constexpr int NC = CW * 32;
  constexpr int K = KV;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[32], empty[32], p1done[2], sdone[2];
  __shared__ Lse red[2][CW];
  __shared__ float zy_sh[2];
  __shared__ RowBroadcast bc[2];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int32_t V = P.vocab;
  const int32_t nvec = V / VN;
  const int32_t nseg = (nvec + kSlotVec - 1) / kSlotVec;
  const int32_t L = min(look, nseg);
  const uint32_t sbase = ptx::smem_u32(smem);
  const uint32_t fbase = ptx::smem_u32(full), ebase = ptx::smem_u32(empty);
  const uint32_t p1b = ptx::smem_u32(p1done), sdb = ptx::smem_u32(sdone);
  const int64_t G = gridDim.x;

  if (threadIdx.x == 0) {
    for (int i = 0; i < nslots; ++i) {
      ptx::mbar_init(&full[i], 1);
      ptx::mbar_init(&empty[i], CW);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&p1done[i], CW);
      ptx::mbar_init(&sdone[i], 1);
    }
    ptx::fence_mbarrier_init();
  }
  __syncthreads();

  if (warp == CW) {
    // ---------------- producer: same segment order as the consumers ----------
    if (lane == 0) {
      const uint64_t keep = ptx::policy_evict_last(), drop = ptx::policy_evict_first();
      Ring ring(nslots);
      auto issue = [&](const TIn* row, int32_t sg0, int32_t sg1, uint64_t pol) {
        for (int32_t sg = sg0; sg < sg1; ++sg, ring.next()) {
          const uint32_t slot = ring.slot, par = ring.ph;
          ptx::mbar_wait_u32(ebase + slot * 8, par ^ 1u);
          const int32_t v0 = sg * kSlotVec;
          const uint32_t bytes = static_cast<uint32_t>(min(kSlotVec, nvec - v0)) * 16u;
          ptx::mbar_arrive_expect_tx_u32(fbase + slot * 8, bytes);
          ptx::bulk_g2s_u32(sbase + slot * (kSlotVec * 16), row + static_cast<int64_t>(v0) * VN,
                            bytes, fbase + slot * 8, pol);
        }
      };
      auto rowp = [&](int64_t r) { return static_cast<const TIn*>(P.logits) + r * P.ld; };
      int64_t r = blockIdx.x;
      if (resident) {
        // rows stay in the ring between their two passes: one load per row
        for (; r < P.n_rows; r += G) issue(rowp(r), 0, nseg, drop);
        return;
      }
      if (r < P.n_rows) issue(rowp(r), 0, nseg, keep);
      for (; r < P.n_rows; r += G) {
        const bool nx = r + G < P.n_rows;
        if (nx) issue(rowp(r + G), 0, L, keep);
        if (P.dlogits) issue(rowp(r), 0, nseg, drop);
        if (nx) issue(rowp(r + G), L, nseg, keep);
      }
    }
    return;
  }

  if (warp == CW + 1) {
    // ---------------- scalar warp: merge partials, token math, broadcast -----
    MetaPipe mp;
    if (lane == 0) mp.init(P, blockIdx.x, G);
    uint32_t i = 0;
    for (int64_t r = blockIdx.x; r < P.n_rows; r += G, ++i) {
      RowMeta meta{};
      if (lane == 0) meta = mp.advance(P, r, G);
      const uint32_t bsel = i & 1u, par = (i >> 1) & 1u;
      ptx::mbar_wait_u32(p1b + bsel * 8, par);
      Lse tot = lane < CW ? red[bsel][lane] : lse_empty();
      warp_lse<ENT, lse_width(CW)>(tot);
      if (lane == 0) {
        const float zy = static_cast<uint32_t>(meta.y) < static_cast<uint32_t>(V) ? zy_sh[bsel] : 0.f;
        bc[bsel] = row_scalar_phase<ENT>(P, P.row_base + r, meta.y, meta.st, meta.blp, meta.rl,
                                         meta.adv, tot, zy, true, meta.keep);
        ptx::mbar_arrive_u32(sdb + bsel * 8);
      }
      __syncwarp();
    }
    return;
  }

  // ---------------- consumers ----------------
  const int tid = threadIdx.x;
  const uint64_t pol = ptx::policy_evict_first();
  // Resident mode (3 rows fit in the ring): pass 2 reads the row from the
  // segments pass 1 consumed, which stay allocated until pass 2 releases them;
  // `ring2` walks the same slot sequence one row behind `ring`.
  Ring ring(nslots), ring2(nslots);
  PhaseTimer tm;
  tm.start(P.trace && tid == 0 && blockIdx.x < kTraceCtas);

  auto run_p1 = [&](P1Acc& a, int32_t y, int32_t sg0, int32_t sg1) {
    for (int32_t sg = sg0; sg < sg1; ++sg, ring.next()) {
      const uint32_t slot = ring.slot, par = ring.ph;
      const int32_t v0 = sg * kSlotVec;
      const long long w0 = tm.on ? clock64() : 0;
      ptx::mbar_wait_u32(fbase + slot * 8, par);
      if (tm.on) tm.acc[6] += clock64() - w0;
      p1_segment<TIn, NC, K, kSlotVec, ENT>(a, sbase + slot * (kSlotVec * 16), v0,
                                            min(kSlotVec, nvec - v0), y, tid);
      __syncwarp();
      if (lane == 0 && !resident) ptx::mbar_arrive_u32(ebase + slot * 8);
    }
  };
  // hand row i's pass-1 partials to the scalar warp
  auto finish_p1 = [&](P1Acc& a, uint32_t i) {
    Lse st = a.st;
    if constexpr (!ENT) {
      st.m = a.m;
      st.s = (a.s0 + a.s1) + (a.s2 + a.s3);
    }
    warp_lse<ENT>(st);
    const uint32_t bsel = i & 1u;
    if (a.have_zy) zy_sh[bsel] = a.zy;  // exactly one consumer thread owns the target
    if (lane == 0) red[bsel][warp] = st;
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive_u32(p1b + bsel * 8);
  };

  int64_t r = blockIdx.x;
  uint32_t i = 0;
  if (r < P.n_rows) {
    P1Acc a0;
    run_p1(a0, P.target[P.row_base + r], 0, nseg);
    finish_p1(a0, 0);
  }
  tm.mark(0);
  for (; r < P.n_rows; r += G, ++i) {
    const int64_t rn = r + G;
    const bool nx = rn < P.n_rows;
    P1Acc an;
    const int32_t yn = nx ? P.target[P.row_base + rn] : 0;
    if (nx) run_p1(an, yn, 0, resident ? nseg : L);
    // resident: hand row i+1 over at once (its red/zy_sh buffer was freed by
    // row i-1's broadcast), so its scalar phase overlaps pass 2 of row i
    if (resident && nx) finish_p1(an, i + 1);
    tm.mark(0);
    const uint32_t bsel = i & 1u, par = (i >> 1) & 1u;
    ptx::mbar_wait_u32(sdb + bsel * 8, par);  // row i's broadcast (also frees red/zy_sh[bsel])
    tm.mark(2);
    if (resident) {
      // pass 2 of row i from its resident segments, then release them
      const RowBroadcast b = bc[bsel];
      const bool zero_row = (b.coef == 0.f) && (!ENT || b.eg == 0.f);
      TOut* drow = P.dlogits ? static_cast<TOut*>(P.dlogits) + r * P.ld_d : nullptr;
      for (int32_t sg = 0; sg < nseg; ++sg, ring2.next()) {
        const uint32_t slot = ring2.slot;
        const int32_t v0 = sg * kSlotVec;
        if (drow)
          p2_segment<TIn, TOut, NC, K, kSlotVec, ENT>(b, zero_row, sbase + slot * (kSlotVec * 16), v0,
                                                      min(kSlotVec, nvec - v0),
                                                      drow + static_cast<int64_t>(v0) * VN, tid, pol);
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_u32(ebase + slot * 8);
      }
      tm.mark(4);
      tm.acc[5] += 1;
      continue;
    }
    if (P.dlogits) {
      const RowBroadcast b = bc[bsel];
      const bool zero_row = (b.coef == 0.f) && (!ENT || b.eg == 0.f);
      TOut* drow = static_cast<TOut*>(P.dlogits) + r * P.ld_d;
      for (int32_t sg = 0; sg < nseg; ++sg, ring.next()) {
        const uint32_t slot = ring.slot, ph = ring.ph;
        const int32_t v0 = sg * kSlotVec;
        const long long w0 = tm.on ? clock64() : 0;
        ptx::mbar_wait_u32(fbase + slot * 8, ph);
        if (tm.on) tm.acc[7] += clock64() - w0;
        p2_segment<TIn, TOut, NC, K, kSlotVec, ENT>(b, zero_row, sbase + slot * (kSlotVec * 16), v0,
                                                    min(kSlotVec, nvec - v0),
                                                    drow + static_cast<int64_t>(v0) * VN, tid, pol);
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive_u32(ebase + slot * 8);
      }
    }
    tm.mark(4);
    if (nx) {
      run_p1(an, yn, L, nseg);
      finish_p1(an, i + 1);
    }
    tm.mark(0);
    tm.acc[5] += 1;
  }
  tm.flush(P.trace);
}

// ---------------------------------------------------------------------------
// generic fused kernel (any alignment / vocab): block per row, two L2 passes
// ---------------------------------------------------------------------------
template <typename TIn, typename TOut, bool ENT>
__global__ void __launch_bounds__(256) fused_generic_kernel(const LossParams P) {
  __shared__ Lse red[8];
  __shared__ RowBroadcast bc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int32_t V = P.vocab;
  for (int64_t r = blockIdx.x; r < P.n_rows; r += gridDim.x) {
    const int64_t t = P.row_base + r;
    const TIn* row = static_cast<const TIn*>(P.logits) + r * P.ld;
    RowMeta meta{};
    if (threadIdx.x == 0) meta = load_meta(P, t);
    const int32_t y = P.target[t];
    Lse st = lse_empty();
    for (int32_t k = threadIdx.x; k < V; k += blockDim.x) {
      float x = Vec<TIn>::load1(row + k);
      online_update<1, ENT>(&x, st, k == y ? 0 : -1);
    }
    warp_lse<ENT>(st);
    if (lane == 0) red[warp] = st;
    __syncthreads();
    if (threadIdx.x == 0) {
      Lse tot = lse_empty();
      for (int w = 0; w < nw; ++w) lse_merge<ENT>(tot, red[w]);
      const float zy = static_cast<uint32_t>(meta.y) < static_cast<uint32_t>(V)
                           ? Vec<TIn>::load1(row + meta.y) : 0.f;
      bc = row_scalar_phase<ENT>(P, t, meta.y, meta.st, meta.blp, meta.rl, meta.adv, tot, zy, true, meta.keep);
    }
    __syncthreads();
    const RowBroadcast b = bc;
    if (P.dlogits) {
      TOut* drow = static_cast<TOut*>(P.dlogits) + r * P.ld_d;
      const bool zero_row = (b.coef == 0.f) && (!ENT || b.eg == 0.f);
      for (int32_t k = threadIdx.x; k < V; k += blockDim.x) {
        float d = 0.f;
        if (!zero_row) {
          float x = Vec<TIn>::load1(row + k);
          row_grad<1, ENT>(&x, &d, k, b);
        }
        store1(drow + k, d);
      }
    }
    __syncthreads();  // red/bc reuse
  }
}

// ---------------------------------------------------------------------------
// K3 (unfused): dlogits from (cur_lp, lse, behav) in a second streaming pass
// ---------------------------------------------------------------------------
template <typename TIn, typename TOut, bool ENT, bool VECTOR>
__global__ void __launch_bounds__(256) bwd_kernel(const LossParams P) {
  using VI = Vec<TIn>;
  constexpr int VN = VI::N;
  __shared__ Lse red[8];
  __shared__ RowBroadcast bc;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int32_t V = P.vocab;
  const uint64_t pol = ptx::policy_evict_first();
  for (int64_t r = blockIdx.x; r < P.n_rows; r += gridDim.x) {
    const int64_t t = P.row_base + r;
    const TIn* row = static_cast<const TIn*>(P.logits) + r * P.ld;
    Lse tot = lse_empty();
    if (ENT) {  // the entropy term needs sum p*log p: one extra pass
      const int32_t yk = P.target[t];
      Lse st = lse_empty();
      for (int32_t k = threadIdx.x; k < V; k += blockDim.x) {
        float x = VI::load1(row + k);
        online_update<1, true>(&x, st, k == yk ? 0 : -1);
      }
      warp_lse<true>(st);
      if (lane == 0) red[warp] = st;
      __syncthreads();
      for (int w = 0; w < nw; ++w) lse_merge<true>(tot, red[w]);
    }
    if (threadIdx.x == 0) {
      const int32_t y = P.target[t];
      const uint32_t st = P.stage[t];
      const float cur = P.in_cur_lp[t];
      const float beh = P.in_behav[t];
      const double adv = P.adv[P.tok_traj[t]];
      const float rl = P.ref_lp ? P.ref_lp[t] : 0.f;
      const bool stale = st < static_cast<uint32_t>(P.cur_stage);
      float H = 0.f, ln_s = 0.f;
      if (ENT) {
        const bool ok = static_cast<uint32_t>(y) < static_cast<uint32_t>(V);
        const LogProb lp = finish_logprob(tot.m, tot.s, ok ? VI::load1(row + y) : 0.f, ok);
        ln_s = lp.ln_s;
        H = ln_s - tot.u / tot.a;
      }
      const bool keep = P.loss_mask ? P.loss_mask[t] != 0 : true;
      TokenResult tr = !keep ? TokenResult{0.0, 0.0, FLAG_MASKED, 0u}
                       : static_cast<uint32_t>(y) < static_cast<uint32_t>(V)
                           ? token_objective(P, cur, beh, adv, rl, stale, H, ENT)
                           : TokenResult{0.0, 0.0, static_cast<uint8_t>(stale ? FLAG_STALE : 0),
                                         ERR_TOKEN_OOV};
      if (tr.err) {
        atomicOr(P.err, tr.err);
        tr.obj = 0.0;
        tr.coef = 0.0;
      }
      P.obj[t] = tr.obj;
      if (P.coef) P.coef[t] = tr.coef;
      P.flags[t] = tr.flags;
      RowBroadcast b;
      b.coef = static_cast<float>(tr.coef);
      b.dy = tr.err ? 0.f : static_cast<float>(tr.coef) * -expm1f(cur);
      b.y = y;
      if (ENT) {
        b.m = tot.m;
        b.log2s = ln_s * kLog2e;
        b.k0 = H - ln_s;
        b.eg = tr.err ? 0.f : static_cast<float>(P.inv_t * P.entropy_coeff);
      } else {  // p = exp(z - lse): frame m = lse, log2 s = 0
        b.m = P.in_lse[t];
        b.log2s = 0.f;
        b.k0 = 0.f;
        b.eg = 0.f;
      }
      bc = b;
    }
    __syncthreads();
    const RowBroadcast b = bc;
    if (P.dlogits) {
      TOut* drow = static_cast<TOut*>(P.dlogits) + r * P.ld_d;
      const bool zero_row = (b.coef == 0.f) && (!ENT || b.eg == 0.f);
      if constexpr (VECTOR) {
        const int32_t nvec = V / VN;
        const uint4* rv = reinterpret_cast<const uint4*>(row);
        for (int32_t v = threadIdx.x; v < nvec; v += blockDim.x) {
          float d[VN];
          if (zero_row) {
#pragma unroll
            for (int j = 0; j < VN; ++j) d[j] = 0.f;
          } else {
            float x[VN];
            VI::unpack(ptx::ld_global_nc_v4(rv + v), x);
            row_grad<VN, ENT>(x, d, v * VN, b);
          }
          store_vec<TOut, VN>(drow + static_cast<int64_t>(v) * VN, d, pol);
        }
      } else {
        for (int32_t k = threadIdx.x; k < V; k += blockDim.x) {
          float d = 0.f;
          if (!zero_row) {
            float x = VI::load1(row + k);
            row_grad<1, ENT>(&x, &d, k, b);
          }
          store1(drow + k, d);
        }
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// small kernels
// ---------------------------------------------------------------------------
// VEC (every pointer 16-byte aligned, flags 4-byte): 4 tokens per thread with
// 16-byte loads/stores and one 4-byte flag store; the remaining n % 4 tokens
// scalar. Same per-token select either way (bit-exact).
template <bool VEC>
__global__ void behaviour_kernel(const uint32_t* __restrict__ stage, uint32_t cur_stage,
                                 const float* __restrict__ blp, const float* __restrict__ cur,
                                 int is_enabled, int behav_mode, int64_t n, float* __restrict__ out,
                                 uint8_t* __restrict__ flags) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  int64_t tail = 0;
  if constexpr (VEC) {
    const int64_t nq = n / 4;
    for (int64_t q = i0; q < nq; q += stride) {
      const uint4 s = reinterpret_cast<const uint4*>(stage)[q];
      const float4 b = reinterpret_cast<const float4*>(blp)[q];
      const float4 c = reinterpret_cast<const float4*>(cur)[q];
      float4 r;
      r.x = select_behaviour(s.x, cur_stage, b.x, c.x, is_enabled, behav_mode);
      r.y = select_behaviour(s.y, cur_stage, b.y, c.y, is_enabled, behav_mode);
      r.z = select_behaviour(s.z, cur_stage, b.z, c.z, is_enabled, behav_mode);
      r.w = select_behaviour(s.w, cur_stage, b.w, c.w, is_enabled, behav_mode);
      reinterpret_cast<float4*>(out)[q] = r;
      if (flags) {
        const uint32_t f = (s.x < cur_stage ? FLAG_STALE : 0u) | (s.y < cur_stage ? FLAG_STALE : 0u) << 8 |
                           (s.z < cur_stage ? FLAG_STALE : 0u) << 16 | (s.w < cur_stage ? FLAG_STALE : 0u) << 24;
        reinterpret_cast<uint32_t*>(flags)[q] = f;
      }
    }
    tail = nq * 4;
  }
  for (int64_t t = tail + i0; t < n; t += stride) {
    const uint32_t st = stage[t];
    out[t] = select_behaviour(st, cur_stage, blp[t], cur[t], is_enabled, behav_mode);
    if (flags) flags[t] = st < cur_stage ? FLAG_STALE : 0;
  }
}

// one warp per segment / trajectory: fill [off[i], off[i+1]) with val(i)
__global__ void expand_u32_kernel(const int64_t* __restrict__ off, const uint32_t* __restrict__ val,
                                  int64_t n, uint32_t* __restrict__ out) {
  const int64_t w = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= n) return;
  const uint32_t v = val ? val[w] : static_cast<uint32_t>(w);
  const int64_t a = off[w], b = off[w + 1];
  // head up to a 16-byte boundary, 16-byte body, tail (out is 4-byte aligned)
  int64_t a4 = a + ((4 - static_cast<int64_t>((reinterpret_cast<uintptr_t>(out) / 4 + a) & 3)) & 3);
  if (a4 > b) a4 = b;
  const int64_t b4 = a4 + ((b - a4) & ~int64_t{3});
  for (int64_t t = a + lane; t < a4; t += 32) out[t] = v;
  const uint4 vv{v, v, v, v};
  for (int64_t t = a4 + 4 * lane; t < b4; t += 128) *reinterpret_cast<uint4*>(out + t) = vv;
  for (int64_t t = b4 + lane; t < b; t += 32) out[t] = v;
}

__global__ void terminal_rewards_kernel(const int32_t* __restrict__ tokens,
                                        const int64_t* __restrict__ tok_off, int64_t n_traj,
                                        const uint8_t* __restrict__ terminated,
                                        const int32_t* __restrict__ answer_target, int32_t eos,
                                        double* __restrict__ out, uint32_t* err) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n_traj;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = tok_off[i], n = tok_off[i + 1] - b;
    if (!terminated[i] || n == 0) {  // grpo.hpp:36,38 (two different messages)
      atomicOr(err, terminated[i] ? ERR_EMPTY_TERMINATED : ERR_NOT_TERMINATED);
      out[i] = 0.0;
      continue;
    }
    int32_t answer;
    if (tokens[b + n - 1] == eos) {
      if (n < 2) {  // bare EOS, grpo.hpp:40
        out[i] = 0.0;
        continue;
      }
      answer = tokens[b + n - 2];
    } else {
      answer = tokens[b + n - 1];  // truncated at the horizon
    }
    out[i] = answer == answer_target[i] ? 1.0 : 0.0;
  }
}

// grpo.hpp:51-65, one thread per group, fp64 with the reference's order and
// explicitly unfused multiply/add so the result is bit-identical.
__global__ void group_advantages_kernel(const double* __restrict__ r, const int64_t* __restrict__ goff,
                                        int64_t n_groups, double eps, double* __restrict__ adv) {
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < n_groups;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = goff[g], e = goff[g + 1];
    const double n = static_cast<double>(e - b);
    double mean = 0.0;
    for (int64_t i = b; i < e; ++i) mean = __dadd_rn(mean, r[i]);
    mean = __ddiv_rn(mean, n);
    double var = 0.0;
    for (int64_t i = b; i < e; ++i) {
      const double d = __dadd_rn(r[i], -mean);
      var = __dadd_rn(var, __dmul_rn(d, d));
    }
    var = __ddiv_rn(var, n);
    const double denom = __dadd_rn(__dsqrt_rn(var), eps);
    for (int64_t i = b; i < e; ++i) adv[i] = __ddiv_rn(__dadd_rn(r[i], -mean), denom);
  }
}

// AdamOptimizer::update (grpo.hpp:209-227) per element in fp64, unfused and in
// the reference's order so the result is bit-identical.
__global__ void adam_kernel(double* __restrict__ p, const double* __restrict__ g,
                            double* __restrict__ m, double* __restrict__ v, int64_t n, double lr,
                            double b1, double b2, double eps, double wd, double bc1, double bc2) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double gi = g[i];
    const double mi = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(__dadd_rn(1.0, -b1), gi));
    const double vi = __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(__dmul_rn(__dadd_rn(1.0, -b2), gi), gi));
    m[i] = mi;
    v[i] = vi;
    const double mhat = __ddiv_rn(mi, bc1);
    const double vhat = __ddiv_rn(vi, bc2);
    const double pi = p[i];
    const double upd = __dadd_rn(__ddiv_rn(mhat, __dadd_rn(__dsqrt_rn(vhat), eps)), __dmul_rn(wd, pi));
    p[i] = __dadd_rn(pi, -__dmul_rn(lr, upd));
  }
}

template <bool VEC>
__global__ void __launch_bounds__(kReduceThreads)
    reduce_kernel(const double* __restrict__ obj, const uint8_t* __restrict__ flags, int64_t n,
                  double* __restrict__ out4, ReduceScratch* sc) {
  __shared__ ReduceSmem sm;
  __shared__ bool last;
  const int64_t tile = reduce_tile(n), ntiles = (n + tile - 1) / tile;
  for (int64_t k = blockIdx.x; k < ntiles; k += gridDim.x) {
    double po;
    unsigned long long ps, pc;
    reduce_tile_partial<VEC>(obj, flags, n, tile, k, sm, threadIdx.x, po, ps, pc);
    if (threadIdx.x == 0) {
      sc->obj[k] = po;
      sc->stale[k] = ps;
      sc->clipped[k] = pc;
    }
  }
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&sc->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {
    __threadfence();
    reduce_final(n, ntiles, out4, sm, threadIdx.x,
                 [&](int64_t i, double& o, unsigned long long& s, unsigned long long& c) {
                   scratch_part(sc, i, o, s, c);
                 });
    if (threadIdx.x == 0) sc->ticket = 0;
  }
}

// ---------------------------------------------------------------------------
// host-side dispatch helpers
// ---------------------------------------------------------------------------
template <typename K>
cudaError_t set_smem(K kernel, int bytes) {
  return allow_dyn_smem(reinterpret_cast<const void*>(kernel), bytes);
}

int grid_rows(int64_t n_rows, int num_sms, int per_sm) {
  int64_t g = static_cast<int64_t>(num_sms) * per_sm;
  if (n_rows < g) g = n_rows;
  return static_cast<int>(g < 1 ? 1 : g);
}

template <typename TIn, typename TOut, int WARPS, bool ENT>
cudaError_t launch_tma(const LossParams& p, int32_t E, int num_sms, cudaStream_t stream,
                       LaunchInfo* info) {
  constexpr int VN = Vec<TIn>::N;
  constexpr int CL = 1;
  auto kernel = fused_tma_kernel<TIn, TOut, CL, WARPS, ENT>;
  const int smem = ((E / VN) * 16 + 127) / 128 * 128;
  cudaError_t e = set_smem(kernel, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, WARPS * 32, smem);
  if (e != cudaSuccess) return e;
  const int64_t resident = static_cast<int64_t>(per_sm) * num_sms;
  if (resident < 1) return cudaErrorInvalidConfiguration;
  const int64_t grid = p.n_rows < resident ? p.n_rows : resident;
  // fused reduction for small steps (<= kFuseReduceTiles tiles): the last CTA
  // reduces in its row buffer; larger steps keep the separate reduce launch
  LossParams q = p;
  const bool fuse = fuse_reduce_ok(p, smem);
  if (!fuse) q.out4 = nullptr;
  if (info) {
    info->cluster = CL;
    info->grid = static_cast<int>(grid);
    info->kernel = "fused_tma_kernel";
    info->reduced = fuse ? 1 : 0;
  }
  // without the reduction scratch (its ticket) the kernel cannot rearm the claim
  // counter itself: zero it here
  if (p.row_ctr && (CL != 1 || !p.red_scratch)) {
    e = cudaMemsetAsync(p.row_ctr, 0, sizeof(unsigned long long), stream);
    if (e != cudaSuccess) return e;
  }
  kernel<<<static_cast<unsigned>(grid), WARPS * 32, smem, stream>>>(q, E);
  return cudaGetLastError();
}

template <typename TIn, typename TOut, bool ENT>
cudaError_t launch_stream(const LossParams& p, int num_sms, const Tuning& tu, cudaStream_t stream,
                          LaunchInfo* info) {
  constexpr int CW = 16, KV = kStreamK;
  auto kernel = fused_stream_la_kernel<TIn, TOut, CW, KV, ENT>;
  constexpr int slot_bytes = CW * 32 * KV * 16;
  const int nslots = tu.slots > 0 ? tu.slots : 196608 / slot_bytes;
  if (nslots > 32 || nslots < 2) return cudaErrorInvalidValue;
  const int smem = nslots * slot_bytes;
  cudaError_t e = set_smem(kernel, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, (CW + 2) * 32, smem);
  if (e != cudaSuccess) return e;
  const int grid = grid_rows(p.n_rows, num_sms, per_sm < 1 ? 1 : per_sm);
  // resident rows: three whole rows fit in the ring (pass 2 reuses pass 1's
  // segments instead of re-reading the row from L2)
  const int64_t nseg = (p.vocab / Vec<TIn>::N + CW * 32 * KV - 1) / (CW * 32 * KV);
  const int resident = tu.resident && p.dlogits != nullptr && 3 * nseg <= nslots;
  if (info) {
    info->cluster = 1;
    info->grid = grid;
    info->kernel = resident ? "fused_stream_la_kernel[resident]" : "fused_stream_la_kernel";
  }
  kernel<<<grid, (CW + 2) * 32, smem, stream>>>(p, nslots, tu.lookahead < 0 ? 0 : tu.lookahead,
                                                 resident);
  return cudaGetLastError();
}

// Fused-kernel selection (ctx tuning `fused_impl`: 0 auto, 1 stream, 2 tma):
//   rows <= 72 KB : fused_tma_kernel, whole row in shared memory, several
//                   CTAs per SM (independent rows overlap their sync phases);
//   larger rows   : fused_stream_la_kernel (TMA ring + L2 re-read, 1 CTA/SM);
//   unaligned     : fused_generic_kernel.
template <typename TIn, typename TOut, bool ENT>
cudaError_t dispatch_fused(const LossParams& p, int num_sms, const Tuning& tu, cudaStream_t stream,
                           LaunchInfo* info) {
  constexpr int VN = Vec<TIn>::N;
  constexpr int64_t kMaxTmaRowBytes = 200 * 1024;
  const int64_t row_bytes = static_cast<int64_t>(p.vocab) * sizeof(TIn);
  const bool aligned = (p.vocab % VN == 0) && ((p.ld * sizeof(TIn)) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(p.logits) % 16 == 0) &&
                       (p.dlogits == nullptr ||
                        (((p.ld_d * sizeof(TOut)) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(p.dlogits) % 16 == 0))) &&
                       p.vocab >= 32 * VN;
  if (aligned) {
    int impl = tu.fused_impl;
    if (impl == 2 && row_bytes > kMaxTmaRowBytes) impl = 1;
    if (impl == 0) impl = row_bytes <= 72 * 1024 ? 2 : 1;
    if (impl == 2) {
      const int32_t E = static_cast<int32_t>((p.vocab + VN - 1) / VN * VN);
      if (row_bytes <= 72 * 1024) return launch_tma<TIn, TOut, 8, ENT>(p, E, num_sms, stream, info);
      return launch_tma<TIn, TOut, 16, ENT>(p, E, num_sms, stream, info);
    }
    return launch_stream<TIn, TOut, ENT>(p, num_sms, tu, stream, info);
  }
  if (info) {
    info->cluster = 1;
    info->grid = grid_rows(p.n_rows, num_sms, 8);
    info->kernel = "fused_generic_kernel";
  }
  fused_generic_kernel<TIn, TOut, ENT><<<grid_rows(p.n_rows, num_sms, 8), 256, 0, stream>>>(p);
  return cudaGetLastError();
}

template <typename TIn, typename TOut, bool ENT>
cudaError_t dispatch_bwd(const LossParams& p, int num_sms, cudaStream_t stream, LaunchInfo* info) {
  constexpr int VN = Vec<TIn>::N;
  const bool aligned = (p.vocab % VN == 0) && ((p.ld * sizeof(TIn)) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(p.logits) % 16 == 0) &&
                       (p.dlogits == nullptr ||
                        (((p.ld_d * sizeof(TOut)) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(p.dlogits) % 16 == 0)));
  const int grid = grid_rows(p.n_rows, num_sms, 8);
  if (info) {
    info->cluster = 1;
    info->grid = grid;
    info->kernel = "bwd_kernel";
  }
  if (aligned)
    bwd_kernel<TIn, TOut, ENT, true><<<grid, 256, 0, stream>>>(p);
  else
    bwd_kernel<TIn, TOut, ENT, false><<<grid, 256, 0, stream>>>(p);
  return cudaGetLastError();
}

template <bool ENT>
cudaError_t by_types(bool bwd, const LossParams& p, DType in, DType out, int num_sms,
                     const Tuning& tu, cudaStream_t stream, LaunchInfo* info) {
  using bf16 = __nv_bfloat16;
  if (in == DType::BF16 && out == DType::BF16)
    return bwd ? dispatch_bwd<bf16, bf16, ENT>(p, num_sms, stream, info)
               : dispatch_fused<bf16, bf16, ENT>(p, num_sms, tu, stream, info);
  if (in == DType::BF16 && out == DType::F32)
    return bwd ? dispatch_bwd<bf16, float, ENT>(p, num_sms, stream, info)
               : dispatch_fused<bf16, float, ENT>(p, num_sms, tu, stream, info);
  if (in == DType::F32 && out == DType::BF16)
    return bwd ? dispatch_bwd<float, bf16, ENT>(p, num_sms, stream, info)
               : dispatch_fused<float, bf16, ENT>(p, num_sms, tu, stream, info);
  return bwd ? dispatch_bwd<float, float, ENT>(p, num_sms, stream, info)
             : dispatch_fused<float, float, ENT>(p, num_sms, tu, stream, info);
}

}  // namespace

cudaError_t launch_fused_kernel(const LossParams& p, DType in, DType out, int num_sms,
                                const Tuning& tu, cudaStream_t stream, LaunchInfo* info);

cudaError_t launch_fused(const LossParams& p, DType in, DType out, int num_sms, const Tuning& tu,
                         cudaStream_t stream, LaunchInfo* info) {
  LaunchInfo li{};
  cudaError_t e = launch_fused_kernel(p, in, out, num_sms, tu, stream, &li);
  li.num_sms = num_sms;
  if (e == cudaSuccess && p.out4 && !li.reduced)
    e = launch_reduce(p.obj, p.flags, p.red_n, p.out4, p.red_scratch, num_sms, stream);
  if (info) *info = li;
  return e;
}

cudaError_t launch_fused_kernel(const LossParams& p, DType in, DType out, int num_sms,
                                const Tuning& tu, cudaStream_t stream, LaunchInfo* info) {
  if (p.n_rows == 0) return cudaSuccess;
  // bf16 rows, by size (fused_impl 0; 3 forces the pair kernel, 4 the solo):
  //   4 KB .. 112 KB (V 2,048 .. 57,344, e.g. 32,000 / 50,304): the solo
  //     kernel — one CTA per row, two 8-warp CTAs per SM;
  //   above (e.g. 65,536 .. 229,376): the CTA-pair kernel, with 8-warp CTAs
  //     (two per SM) while the half row fits them (V <= 114,688), else 16;
  //   below, unaligned or with the entropy term: the TMA / ring / generic kernels.
  // K1 (gather-only) takes the same shape as the loss at its vocabulary: its
  // log-probs are bitwise the loss kernel's recomputation.
  // Same-box A/B in profiles/r02_vocab_sweep.txt (solo at V = 50,304: 0.92 vs
  // 0.74 for the 16-warp pair; V = 32,000 sustained: solo 0.90 vs pair 0.86;
  // solo vs the TMA kernel at V = 2,048 / 8,192 / 16,384 / 24,576: 136 / 128 /
  // 91 / 57 M rows/s vs 119 / 97 / 71 / 52).
  const bool ent = p.entropy_coeff != 0.0;
  const int64_t row_bytes = static_cast<int64_t>(p.vocab) * 2;
  const bool solo_auto = tu.fused_impl == 0 && row_bytes >= 4 * 1024 && pair_fits(p.vocab, 1, 8);
  if ((tu.fused_impl == 4 || solo_auto) && pair_supported(p, in, out, ent, 1))
    return launch_pair(p, out, 1, num_sms, tu, stream, info);
  if ((tu.fused_impl == 3 || (tu.fused_impl == 0 && row_bytes > 72 * 1024)) &&
      pair_supported(p, in, out, ent, 2))
    return launch_pair(p, out, 2, num_sms, tu, stream, info);
  return p.entropy_coeff != 0.0 ? by_types<true>(false, p, in, out, num_sms, tu, stream, info)
                                : by_types<false>(false, p, in, out, num_sms, tu, stream, info);
}

cudaError_t launch_bwd(const LossParams& p, DType in, DType out, int num_sms,
                       cudaStream_t stream, LaunchInfo* info) {
  if (info) info->num_sms = num_sms;
  cudaError_t e = cudaSuccess;
  if (p.n_rows > 0) {
    const Tuning tu{};
    e = p.entropy_coeff != 0.0 ? by_types<true>(true, p, in, out, num_sms, tu, stream, info)
                               : by_types<false>(true, p, in, out, num_sms, tu, stream, info);
  }
  if (e == cudaSuccess && p.out4)
    e = launch_reduce(p.obj, p.flags, p.red_n, p.out4, p.red_scratch, num_sms, stream);
  return e;
}

// K1 = the fused kernels in gather-only mode: the same TMA/shared-memory
// staged row stream and online LSE as the loss pass (and therefore bitwise the
// same cur_lp/lse as the loss kernel recomputes, the GPU form of
// test_policy.cpp:157-172), without metadata, objective or dlogits.
cudaError_t launch_logprob_gather(const void* logits, int64_t ld, DType in, const int32_t* target,
                                  int64_t n_tok, int32_t vocab, float* out_lp, float* out_lse,
                                  uint32_t* err, unsigned long long* row_ctr, void* red_scratch,
                                  int num_sms, const Tuning& tu, cudaStream_t stream) {
  if (n_tok == 0) return cudaSuccess;
  LossParams p{};
  p.logits = logits;
  p.ld = ld;
  p.vocab = vocab;
  p.n_rows = n_tok;
  p.row_base = 0;
  p.target = target;
  p.cur_lp = out_lp;
  p.lse = out_lse;
  p.err = err;
  p.row_ctr = row_ctr;
  p.red_scratch = red_scratch;  // its ticket lets the last CTA rearm row_ctr
  p.gather_only = 1;
  p.clamp_lo = 0.8;
  p.clamp_hi = 1.28;
  p.inv_t = 1.0;
  return launch_fused(p, in, DType::BF16, num_sms, tu, stream, nullptr);
}

// ---------------------------------------------------------------------------
// per-context tuning (read from the environment once, at context creation)
// ---------------------------------------------------------------------------
namespace {
using I32Field = int Tuning::*;
using I64Field = int64_t Tuning::*;
struct TuneField {
  const char* name;  // option name (copris_ctx_set_option)
  const char* env;   // COPRIS_* variable read by tuning_from_env
  int64_t lo, hi;
  I32Field i32;
  I64Field i64;
};
const TuneField kFields[] = {
    {"fused_impl", "COPRIS_FUSED_IMPL", 0, 4, &Tuning::fused_impl, nullptr},
    {"lookahead", "COPRIS_TUNE_LOOKAHEAD", 0, 16, &Tuning::lookahead, nullptr},
    {"slots", "COPRIS_TUNE_SLOTS", 0, 32, &Tuning::slots, nullptr},
    {"resident", "COPRIS_TUNE_RESIDENT", 0, 1, &Tuning::resident, nullptr},
    {"pair_lookahead", "COPRIS_PAIR_LOOKAHEAD", 0, 7, &Tuning::pair_lookahead, nullptr},
    {"pair_st256", "COPRIS_PAIR_ST256", 0, 1, &Tuning::pair_st256, nullptr},
    {"pair_bf16_stage", "COPRIS_PAIR_BF16_STAGE", 0, 1, &Tuning::pair_bf16_stage, nullptr},
    {"pair_pw8", "COPRIS_PAIR_PW8", 0, 1, &Tuning::pair_pw8, nullptr},
    {"pair_dynamic", "COPRIS_PAIR_DYNAMIC", 0, 1, &Tuning::pair_dynamic, nullptr},
    {"lmhead_impl", "COPRIS_LMHEAD_IMPL", 0, 1, &Tuning::lmhead_impl, nullptr},
    {"lmhead_group", "COPRIS_LMHEAD_GROUP", 1, 1 << 20, &Tuning::lmhead_group, nullptr},
    {"lmhead_tma_store", "COPRIS_LMHEAD_TMA_STORE", 0, 1, &Tuning::lmhead_tma_store, nullptr},
    {"gemm_wide", "COPRIS_GEMM_WIDE", 0, 1, &Tuning::gemm_wide, nullptr},
    {"gemm_mc", "COPRIS_GEMM_MC", 0, 1, &Tuning::gemm_mc, nullptr},
    {"gemm_splits", "COPRIS_GEMM_SPLITS", 0, 64, &Tuning::gemm_splits, nullptr},
    {"gemm_a_evict_first", "COPRIS_GEMM_A_EVICT_FIRST", 0, 3, &Tuning::gemm_a_evict_first, nullptr},
    {"dw_group", "COPRIS_DW_GROUP", 1, 1 << 20, &Tuning::dw_group, nullptr},
    {"dw_policy", "COPRIS_DW_POLICY", 0, 3, &Tuning::dw_policy, nullptr},
    {"dw_kchunk", "COPRIS_DW_KCHUNK", 64, int64_t(1) << 40, nullptr, &Tuning::dw_kchunk},
    {"trace", "COPRIS_TRACE", 0, 1, &Tuning::trace, nullptr},
};

// fused_impl and lmhead_impl also accept their names in the environment
int64_t parse_env(const TuneField& f, const char* v) {
  if (!strcmp(f.name, "fused_impl")) {
    if (!strcmp(v, "auto") || !*v) return 0;
    if (!strcmp(v, "stream")) return 1;
    if (!strcmp(v, "tma")) return 2;
    if (!strcmp(v, "pair")) return 3;
    if (!strcmp(v, "solo")) return 4;
  }
  if (!strcmp(f.name, "lmhead_impl")) {
    if (!strcmp(v, "1sm")) return 1;
    if (!strcmp(v, "pair")) return 0;
  }
  if (!strcmp(f.name, "trace")) return 1;  // any value turns tracing on
  return atoll(v);
}
}  // namespace

bool tuning_set(Tuning& t, const char* name, int64_t value) {
  if (!name) return false;
  for (const TuneField& f : kFields) {
    if (strcmp(f.name, name) != 0) continue;
    if (value < f.lo || value > f.hi) return false;
    if (f.i32) t.*(f.i32) = static_cast<int>(value);
    else t.*(f.i64) = value;
    return true;
  }
  return false;
}

bool tuning_get(const Tuning& t, const char* name, int64_t* value) {
  if (!name || !value) return false;
  for (const TuneField& f : kFields) {
    if (strcmp(f.name, name) != 0) continue;
    *value = f.i32 ? static_cast<int64_t>(t.*(f.i32)) : t.*(f.i64);
    return true;
  }
  return false;
}

Tuning tuning_from_env() {
  Tuning t;
  for (const TuneField& f : kFields) {
    const char* v = getenv(f.env);
    if (v) tuning_set(t, f.name, parse_env(f, v));  // out-of-range values keep the default
  }
  return t;
}


cudaError_t launch_expand_segments(const int64_t* seg_off, const uint32_t* seg_ver, int64_t n_seg,
                                   uint32_t* out_stage, cudaStream_t stream) {
  if (n_seg == 0) return cudaSuccess;
  const int64_t threads = n_seg * 32;
  expand_u32_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, stream>>>(
      seg_off, seg_ver, n_seg, out_stage);
  return cudaGetLastError();
}

cudaError_t launch_token_traj(const int64_t* tok_off, int64_t n_traj, int32_t* out,
                              cudaStream_t stream) {
  if (n_traj == 0) return cudaSuccess;
  const int64_t threads = n_traj * 32;
  expand_u32_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, stream>>>(
      tok_off, nullptr, n_traj, reinterpret_cast<uint32_t*>(out));
  return cudaGetLastError();
}

cudaError_t launch_behaviour(const uint32_t* stage, uint32_t cur_stage, const float* blp,
                             const float* cur_lp, int is_enabled, int behav_mode, int64_t n_tok,
                             float* out_behav, uint8_t* out_flags, cudaStream_t stream) {
  if (n_tok == 0) return cudaSuccess;
  auto a16 = [](const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; };
  const bool vec = a16(stage) && a16(blp) && a16(cur_lp) && a16(out_behav) &&
                   reinterpret_cast<uintptr_t>(out_flags) % 4 == 0;
  const int64_t per = vec ? 4 : 1;
  int64_t blocks = (n_tok / per + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 65535) blocks = 65535;
  if (vec)
    behaviour_kernel<true><<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
        stage, cur_stage, blp, cur_lp, is_enabled, behav_mode, n_tok, out_behav, out_flags);
  else
    behaviour_kernel<false><<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
        stage, cur_stage, blp, cur_lp, is_enabled, behav_mode, n_tok, out_behav, out_flags);
  return cudaGetLastError();
}

cudaError_t launch_terminal_rewards(const int32_t* tokens, const int64_t* tok_off,
                                        int64_t n_traj, const uint8_t* terminated,
                                        const int32_t* answer_target, int32_t eos, double* out,
                                        uint32_t* err, cudaStream_t stream) {
  if (n_traj == 0) return cudaSuccess;
  const int64_t blocks = (n_traj + 255) / 256;
  terminal_rewards_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
      tokens, tok_off, n_traj, terminated, answer_target, eos, out, err);
  return cudaGetLastError();
}

cudaError_t launch_group_advantages(const double* rewards, const int64_t* group_off,
                                    int64_t n_groups, double eps, double* out_adv,
                                    cudaStream_t stream) {
  if (n_groups == 0) return cudaSuccess;
  const int64_t blocks = (n_groups + 127) / 128;
  group_advantages_kernel<<<static_cast<unsigned>(blocks), 128, 0, stream>>>(rewards, group_off,
                                                                             n_groups, eps, out_adv);
  return cudaGetLastError();
}

size_t reduce_scratch_bytes() { return sizeof(ReduceScratch); }

cudaError_t launch_adam(double* p, const double* g, double* m, double* v, int64_t n, double lr,
                        double b1, double b2, double eps, double wd, double bc1, double bc2,
                        int num_sms, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, static_cast<int64_t>(num_sms) * 8);
  adam_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(p, g, m, v, n, lr, b1, b2, eps, wd,
                                                                 bc1, bc2);
  return cudaGetLastError();
}

cudaError_t launch_reduce(const double* obj, const uint8_t* flags, int64_t n_tok, double* out4,
                          void* scratch, int num_sms, cudaStream_t stream) {
  (void)num_sms;
  if (n_tok == 0) {
    // an empty batch: zeros (a tile-less reduce would still reset the tickets)
    return cudaMemsetAsync(out4, 0, 4 * sizeof(double), stream);
  }
  const int64_t tile = reduce_tile(n_tok), ntiles = (n_tok + tile - 1) / tile;
  int64_t nb = ntiles < kReduceBlocks ? ntiles : kReduceBlocks;
  const bool vec = (reinterpret_cast<uintptr_t>(obj) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(flags) % 4 == 0);
  if (vec)
    reduce_kernel<true><<<static_cast<unsigned>(nb), kReduceThreads, 0, stream>>>(
        obj, flags, n_tok, out4, static_cast<ReduceScratch*>(scratch));
  else
    reduce_kernel<false><<<static_cast<unsigned>(nb), kReduceThreads, 0, stream>>>(
        obj, flags, n_tok, out4, static_cast<ReduceScratch*>(scratch));
  return cudaGetLastError();
}

cudaError_t allow_dyn_smem(const void* func, int bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> raised;
  std::lock_guard<std::mutex> lock(mu);
  if (raised.count({func, dev})) return cudaSuccess;
  cudaFuncAttributes fa{};
  e = cudaFuncGetAttributes(&fa, func);
  if (e != cudaSuccess) return e;
  int optin = 0;
  e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  const int max_dyn = optin - static_cast<int>(fa.sharedSizeBytes);
  if (bytes > max_dyn) return cudaErrorInvalidValue;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, max_dyn);
  if (e == cudaSuccess) raised.insert({func, dev});
  return e;
}

}  // namespace copris_b200
