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
//   fused_generic_kernel  same arithmetic for rows that are not 16-byte
//                         aligned (tiny/odd vocab); two passes through L2.
//   logprob_gather_kernel K1: streaming log-softmax + gather (cur_lp, lse).
//   bwd_kernel            unfused K3: second streaming pass from lse.
//   + behaviour select (K2), segment expansion, rewards, advantages and a
//     deterministic fixed-order reduction.
#include <cooperative_groups.h>
#include <cuda_bf16.h>

#include <cmath>
#include <cstdint>

#include "kernels.cuh"
#include "ptx.cuh"
#include "token_math.cuh"

namespace cg = cooperative_groups;

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
  if (jt < 0) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const float d = x[j] - st.m;
      const float e = ptx::ex2(d * kLog2e);
      st.s += e;
      if (ENT) {
        st.u = fmaf(e, d, st.u);
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
        st.u = fmaf(e, d, st.u);
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

template <bool ENT>
__device__ __forceinline__ void warp_lse(Lse& st) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    Lse o;
    o.m = __shfl_xor_sync(0xffffffffu, st.m, off);
    o.s = __shfl_xor_sync(0xffffffffu, st.s, off);
    o.u = ENT ? __shfl_xor_sync(0xffffffffu, st.u, off) : 0.f;
    o.a = ENT ? __shfl_xor_sync(0xffffffffu, st.a, off) : 0.f;
    lse_merge<ENT>(st, o);
  }
}

// Per-token metadata of one row, loaded by one thread early in the row.
struct RowMeta {
  int32_t y;
  uint32_t st;
  float blp, rl;
  double adv;
};

__device__ __forceinline__ RowMeta load_meta(const LossParams& P, int64_t t) {
  RowMeta m;
  m.y = P.target[t];
  m.st = P.stage[t];
  m.blp = P.buffered_lp[t];
  m.rl = P.ref_lp ? P.ref_lp[t] : 0.f;
  m.adv = P.adv[P.tok_traj[t]];
  return m;
}

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
    if (ENT) v = fmaf(b.eg * p, xm + b.k0, v);
    d[j] = v;
  }
}

// ---------------------------------------------------------------------------
// fused TMA / cluster kernel
// ---------------------------------------------------------------------------
constexpr int kPieceVec = 256;  // 16-byte vectors per TMA piece (4 KB)
constexpr int kMaxPieces = 8;   // per warp

template <typename TIn, typename TOut, int CL, int WARPS, bool ENT>
__global__ void __launch_bounds__(WARPS * 32, 1)
    fused_tma_kernel(const LossParams P, const int32_t E) {
  using VI = Vec<TIn>;
  constexpr int VN = VI::N;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[WARPS * kMaxPieces];
  __shared__ Lse red[WARPS];
  __shared__ Lse slot[2][CL];
  __shared__ float slot_zy[2][CL];
  __shared__ RowBroadcast bc;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int rank = 0;
  if constexpr (CL > 1) rank = static_cast<int>(cg::this_cluster().block_rank());
  const int64_t cid = blockIdx.x / CL, ncl = gridDim.x / CL;
  const int32_t V = P.vocab;
  const int32_t col0 = rank * E;
  const int32_t ncols = max(0, min(E, V - col0));
  const int32_t nvec = ncols / VN;
  const int32_t wv0 = static_cast<int32_t>(static_cast<int64_t>(warp) * nvec / WARPS);
  const int32_t wv1 = static_cast<int32_t>(static_cast<int64_t>(warp + 1) * nvec / WARPS);
  const int32_t npieces = (wv1 - wv0 + kPieceVec - 1) / kPieceVec;
  uint64_t* mybars = bars + warp * kMaxPieces;
  const uint64_t pol = ptx::policy_evict_first();
  const TIn* logits = static_cast<const TIn*>(P.logits);

  if (lane == 0) {
    for (int p = 0; p < npieces; ++p) ptx::mbar_init(&mybars[p], 1);
    ptx::fence_mbarrier_init();
  }
  __syncthreads();
  if constexpr (CL > 1) cg::this_cluster().sync();

  auto issue = [&](int64_t row, int p) {
    const int32_t v0 = wv0 + p * kPieceVec;
    const uint32_t bytes = static_cast<uint32_t>(min(kPieceVec, wv1 - v0)) * 16u;
    ptx::mbar_arrive_expect_tx(&mybars[p], bytes);
    ptx::bulk_g2s(smem + static_cast<size_t>(v0) * 16,
                  logits + row * P.ld + col0 + static_cast<int64_t>(v0) * VN, bytes, &mybars[p],
                  pol);
  };

  int64_t r = cid;
  if (lane == 0 && r < P.n_rows)
    for (int p = 0; p < npieces; ++p) issue(r, p);

  for (uint32_t it = 0; r < P.n_rows; r += ncl, ++it) {
    const uint32_t par = it & 1u;
    const int64_t t = P.row_base + r;
    RowMeta meta{};
    if (threadIdx.x == 0) meta = load_meta(P, t);
    const int32_t ycol = P.target[t] - col0;  // target column relative to this chunk

    // pass B: online log-sum-exp over this warp's slice as its pieces land
    Lse st = lse_empty();
    for (int p = 0; p < npieces; ++p) {
      ptx::mbar_wait(&mybars[p], par);
      const int32_t v0 = wv0 + p * kPieceVec, v1 = min(wv1, v0 + kPieceVec);
      for (int32_t v = v0 + lane; v < v1; v += 32) {
        float x[VN];
        VI::unpack(ptx::ld_shared_v4(smem + static_cast<size_t>(v) * 16), x);
        const int jt = ycol - v * VN;
        online_update<VN, ENT>(x, st, static_cast<uint32_t>(jt) < VN ? jt : -1);
      }
    }
    warp_lse<ENT>(st);
    if (lane == 0) red[warp] = st;
    __syncthreads();

    Lse tot = lse_empty();
    float zy = 0.f;
    if (threadIdx.x == 0) {
      for (int w = 0; w < WARPS; ++w) lse_merge<ENT>(tot, red[w]);
      if (static_cast<uint32_t>(meta.y - col0) < static_cast<uint32_t>(ncols))
        zy = VI::load1(smem + static_cast<size_t>(meta.y - col0) * sizeof(TIn));
      if constexpr (CL > 1) {
        cg::cluster_group cl = cg::this_cluster();
        for (int c = 0; c < CL; ++c) {
          *cl.map_shared_rank(&slot[par][rank], c) = tot;
          *cl.map_shared_rank(&slot_zy[par][rank], c) = zy;
        }
      }
    }
    if constexpr (CL > 1) cg::this_cluster().sync();
    if (threadIdx.x == 0) {
      if constexpr (CL > 1) {
        tot = lse_empty();
        for (int c = 0; c < CL; ++c) lse_merge<ENT>(tot, slot[par][c]);
        const uint32_t owner = static_cast<uint32_t>(meta.y) / static_cast<uint32_t>(E);
        zy = owner < static_cast<uint32_t>(CL) ? slot_zy[par][owner] : 0.f;
      }
      bc = row_scalar_phase<ENT>(P, t, meta.y, meta.st, meta.blp, meta.rl, meta.adv, tot, zy,
                                 rank == 0);
    }
    __syncthreads();

    // pass C: dlogits from the shared-memory copy; refill each piece with the
    // next row as soon as this warp has consumed it.
    const RowBroadcast b = bc;
    const bool zero_row = (b.coef == 0.f) && (!ENT || b.eg == 0.f);
    const int64_t nxt = r + ncl;
    const bool has_next = nxt < P.n_rows;
    TOut* drow = P.dlogits ? static_cast<TOut*>(P.dlogits) + r * P.ld_d + col0 : nullptr;
    for (int p = 0; p < npieces; ++p) {
      const int32_t v0 = wv0 + p * kPieceVec, v1 = min(wv1, v0 + kPieceVec);
      if (drow) {
        for (int32_t v = v0 + lane; v < v1; v += 32) {
          float d[VN];
          if (zero_row) {
#pragma unroll
            for (int j = 0; j < VN; ++j) d[j] = 0.f;
          } else {
            float x[VN];
            VI::unpack(ptx::ld_shared_v4(smem + static_cast<size_t>(v) * 16), x);
            row_grad<VN, ENT>(x, d, col0 + v * VN, b);
          }
          store_vec<TOut, VN>(drow + static_cast<int64_t>(v) * VN, d, pol);
        }
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0 && has_next) issue(nxt, p);
    }
  }
  // no CTA may exit while a peer can still write its DSMEM slots
  if constexpr (CL > 1) cg::this_cluster().sync();
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
      bc = row_scalar_phase<ENT>(P, t, meta.y, meta.st, meta.blp, meta.rl, meta.adv, tot, zy, true);
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
// K1: streaming log-softmax + gather
// ---------------------------------------------------------------------------
template <typename TIn, bool VECTOR>
__global__ void __launch_bounds__(256)
    logprob_gather_kernel(const TIn* __restrict__ logits, int64_t ld, const int32_t* __restrict__ target,
                          int64_t n_tok, int32_t V, float* __restrict__ out_lp,
                          float* __restrict__ out_lse, uint32_t* err) {
  using VI = Vec<TIn>;
  constexpr int VN = VI::N;
  constexpr int UNROLL = 4;
  __shared__ Lse red[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  for (int64_t r = blockIdx.x; r < n_tok; r += gridDim.x) {
    const TIn* row = logits + r * ld;
    const int32_t y = target[r];
    Lse st = lse_empty();
    if constexpr (VECTOR) {
      const int32_t nvec = V / VN;
      const uint4* rv = reinterpret_cast<const uint4*>(row);
      for (int32_t v = threadIdx.x; v < nvec; v += UNROLL * blockDim.x) {
        uint4 buf[UNROLL];
#pragma unroll
        for (int k = 0; k < UNROLL; ++k) {
          const int32_t vi = v + k * blockDim.x;
          if (vi < nvec) buf[k] = ptx::ld_global_nc_v4(rv + vi);
        }
#pragma unroll
        for (int k = 0; k < UNROLL; ++k) {
          const int32_t vi = v + k * static_cast<int32_t>(blockDim.x);
          if (vi < nvec) {
            float x[VN];
            VI::unpack(buf[k], x);
            const int jt = y - vi * VN;
            online_update<VN, false>(x, st, static_cast<uint32_t>(jt) < VN ? jt : -1);
          }
        }
      }
    } else {
      for (int32_t k = threadIdx.x; k < V; k += blockDim.x) {
        float x = VI::load1(row + k);
        online_update<1, false>(&x, st, k == y ? 0 : -1);
      }
    }
    warp_lse<false>(st);
    if (lane == 0) red[warp] = st;
    __syncthreads();
    if (threadIdx.x == 0) {
      Lse tot = lse_empty();
      for (int w = 0; w < nw; ++w) lse_merge<false>(tot, red[w]);
      const bool ok = static_cast<uint32_t>(y) < static_cast<uint32_t>(V);
      const float zy = ok ? VI::load1(row + y) : 0.f;
      const LogProb lp = finish_logprob(tot.m, tot.s, zy, ok);
      if (!ok) atomicOr(err, ERR_TOKEN_OOV);
      out_lp[r] = lp.cur;
      if (out_lse) out_lse[r] = static_cast<float>(lp.lse);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// unfused K3: per-token objective from (cur_lp, lse, behav) + dlogits pass
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
      double H = 0.0, ln_s = 0.0;
      if (ENT) {
        const bool ok = static_cast<uint32_t>(y) < static_cast<uint32_t>(V);
        const double Sd = static_cast<double>(tot.s) +
                          (ok ? exp(static_cast<double>(VI::load1(row + y)) - static_cast<double>(tot.m)) : 0.0);
        ln_s = log(Sd);
        H = ln_s - static_cast<double>(tot.u) / static_cast<double>(tot.a);
      }
      TokenResult tr = static_cast<uint32_t>(y) < static_cast<uint32_t>(V)
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
      b.dy = tr.err ? 0.f : static_cast<float>(tr.coef * -expm1(static_cast<double>(cur)));
      b.y = y;
      if (ENT) {
        b.m = tot.m;
        b.log2s = static_cast<float>(ln_s * kLog2eD);
        b.k0 = static_cast<float>(H - ln_s);
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
__global__ void behaviour_kernel(const uint32_t* __restrict__ stage, uint32_t cur_stage,
                                 const float* __restrict__ blp, const float* __restrict__ cur,
                                 int is_enabled, int behav_mode, int64_t n, float* __restrict__ out,
                                 uint8_t* __restrict__ flags) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
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
  for (int64_t t = off[w] + lane; t < off[w + 1]; t += 32) out[t] = v;
}

__global__ void terminal_rewards_kernel(const int32_t* __restrict__ tokens,
                                        const int64_t* __restrict__ tok_off, int64_t n_traj,
                                        const uint8_t* __restrict__ terminated,
                                        const int32_t* __restrict__ answer_target, int32_t eos,
                                        double* __restrict__ out, uint32_t* err) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n_traj;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = tok_off[i], n = tok_off[i + 1] - b;
    if (!terminated[i] || n == 0) {  // grpo.hpp:36,38
      atomicOr(err, ERR_NOT_TERMINATED);
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

// Deterministic two-level reduction: fixed block partition, fixed in-block
// tree, and the last block sums block partials in index order.
constexpr int kReduceBlocks = 512;
constexpr int kReduceThreads = 256;
struct ReduceScratch {
  double obj[kReduceBlocks];
  unsigned long long stale[kReduceBlocks];
  unsigned long long clipped[kReduceBlocks];
  unsigned int ticket;
};

__global__ void __launch_bounds__(kReduceThreads)
    reduce_kernel(const double* __restrict__ obj, const uint8_t* __restrict__ flags, int64_t n,
                  double* __restrict__ out4, ReduceScratch* sc) {
  __shared__ double so[kReduceThreads];
  __shared__ unsigned long long ss[kReduceThreads], sk[kReduceThreads];
  __shared__ bool last;
  const int64_t nb = gridDim.x;
  const int64_t b0 = n * blockIdx.x / nb, b1 = n * (blockIdx.x + 1) / nb;
  double o = 0.0;
  unsigned long long st = 0, cl = 0;
  for (int64_t t = b0 + threadIdx.x; t < b1; t += blockDim.x) {
    o += obj[t];
    const uint8_t f = flags[t];
    st += f & FLAG_STALE;
    cl += (f >> 1) & 1u;
  }
  so[threadIdx.x] = o;
  ss[threadIdx.x] = st;
  sk[threadIdx.x] = cl;
  __syncthreads();
  for (int h = blockDim.x / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h) {
      so[threadIdx.x] += so[threadIdx.x + h];
      ss[threadIdx.x] += ss[threadIdx.x + h];
      sk[threadIdx.x] += sk[threadIdx.x + h];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    sc->obj[blockIdx.x] = so[0];
    sc->stale[blockIdx.x] = ss[0];
    sc->clipped[blockIdx.x] = sk[0];
    __threadfence();
    last = atomicAdd(&sc->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double O = 0.0;
    unsigned long long Sx = 0, Cx = 0;
    for (int i = 0; i < gridDim.x; ++i) {
      O += *reinterpret_cast<volatile double*>(&sc->obj[i]);
      Sx += *reinterpret_cast<volatile unsigned long long*>(&sc->stale[i]);
      Cx += *reinterpret_cast<volatile unsigned long long*>(&sc->clipped[i]);
    }
    out4[0] = O;
    out4[1] = static_cast<double>(n);
    out4[2] = static_cast<double>(Sx);
    out4[3] = static_cast<double>(Cx);
    sc->ticket = 0;
  }
}

// ---------------------------------------------------------------------------
// host-side dispatch helpers
// ---------------------------------------------------------------------------
template <typename K>
cudaError_t set_smem(K kernel, int bytes) {
  return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

int grid_rows(int64_t n_rows, int num_sms, int per_sm) {
  int64_t g = static_cast<int64_t>(num_sms) * per_sm;
  if (n_rows < g) g = n_rows;
  return static_cast<int>(g < 1 ? 1 : g);
}

template <typename TIn, typename TOut, int CL, int WARPS, bool ENT>
cudaError_t launch_tma(const LossParams& p, int32_t E, int num_sms, cudaStream_t stream,
                       LaunchInfo* info) {
  constexpr int VN = Vec<TIn>::N;
  auto kernel = fused_tma_kernel<TIn, TOut, CL, WARPS, ENT>;
  const int smem = ((E / VN) * 16 + 127) / 128 * 128;
  cudaError_t e = set_smem(kernel, smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  cfg.blockDim = dim3(WARPS * 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  int resident = 0;
  if (CL > 1) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(CL * num_sms);
    int ncl = 0;
    e = cudaOccupancyMaxActiveClusters(&ncl, kernel, &cfg);
    if (e != cudaSuccess) return e;
    resident = ncl;
  } else {
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, WARPS * 32, smem);
    if (e != cudaSuccess) return e;
    resident = per_sm * num_sms;
  }
  if (resident < 1) return cudaErrorInvalidConfiguration;
  int64_t ncl = resident;
  if (p.n_rows < ncl) ncl = p.n_rows;
  cfg.gridDim = dim3(static_cast<unsigned>(ncl * CL));
  if (info) {
    info->cluster = CL;
    info->grid = static_cast<int>(ncl * CL);
    info->kernel = "fused_tma_kernel";
  }
  return cudaLaunchKernelEx(&cfg, kernel, p, E);
}

template <typename TIn, typename TOut, bool ENT>
cudaError_t dispatch_fused(const LossParams& p, int num_sms, cudaStream_t stream, LaunchInfo* info) {
  constexpr int VN = Vec<TIn>::N;
  constexpr int64_t kMaxChunkBytes = 200 * 1024;
  const int64_t row_bytes = static_cast<int64_t>(p.vocab) * sizeof(TIn);
  const bool aligned = (p.vocab % VN == 0) && ((p.ld * sizeof(TIn)) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(p.logits) % 16 == 0) &&
                       (p.dlogits == nullptr ||
                        (((p.ld_d * sizeof(TOut)) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(p.dlogits) % 16 == 0))) &&
                       p.vocab >= 32 * VN;
  if (aligned) {
    auto chunk = [&](int cl) {
      const int64_t per = (p.vocab + cl - 1) / cl;
      return static_cast<int32_t>((per + VN - 1) / VN * VN);
    };
    if (row_bytes <= 72 * 1024) {
      return launch_tma<TIn, TOut, 1, 8, ENT>(p, chunk(1), num_sms, stream, info);
    } else if (row_bytes <= kMaxChunkBytes) {
      return launch_tma<TIn, TOut, 1, 16, ENT>(p, chunk(1), num_sms, stream, info);
    } else if (row_bytes <= 2 * kMaxChunkBytes) {
      return launch_tma<TIn, TOut, 2, 16, ENT>(p, chunk(2), num_sms, stream, info);
    } else if (row_bytes <= 4 * kMaxChunkBytes) {
      return launch_tma<TIn, TOut, 4, 16, ENT>(p, chunk(4), num_sms, stream, info);
    }
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
                     cudaStream_t stream, LaunchInfo* info) {
  using bf16 = __nv_bfloat16;
  if (in == DType::BF16 && out == DType::BF16)
    return bwd ? dispatch_bwd<bf16, bf16, ENT>(p, num_sms, stream, info)
               : dispatch_fused<bf16, bf16, ENT>(p, num_sms, stream, info);
  if (in == DType::BF16 && out == DType::F32)
    return bwd ? dispatch_bwd<bf16, float, ENT>(p, num_sms, stream, info)
               : dispatch_fused<bf16, float, ENT>(p, num_sms, stream, info);
  if (in == DType::F32 && out == DType::BF16)
    return bwd ? dispatch_bwd<float, bf16, ENT>(p, num_sms, stream, info)
               : dispatch_fused<float, bf16, ENT>(p, num_sms, stream, info);
  return bwd ? dispatch_bwd<float, float, ENT>(p, num_sms, stream, info)
             : dispatch_fused<float, float, ENT>(p, num_sms, stream, info);
}

}  // namespace

cudaError_t launch_fused(const LossParams& p, DType in, DType out, int num_sms,
                         cudaStream_t stream, LaunchInfo* info) {
  if (info) info->num_sms = num_sms;
  if (p.n_rows == 0) return cudaSuccess;
  return p.entropy_coeff != 0.0 ? by_types<true>(false, p, in, out, num_sms, stream, info)
                                : by_types<false>(false, p, in, out, num_sms, stream, info);
}

cudaError_t launch_bwd(const LossParams& p, DType in, DType out, int num_sms,
                       cudaStream_t stream, LaunchInfo* info) {
  if (info) info->num_sms = num_sms;
  if (p.n_rows == 0) return cudaSuccess;
  return p.entropy_coeff != 0.0 ? by_types<true>(true, p, in, out, num_sms, stream, info)
                                : by_types<false>(true, p, in, out, num_sms, stream, info);
}

cudaError_t launch_logprob_gather(const void* logits, int64_t ld, DType in, const int32_t* target,
                                  int64_t n_tok, int32_t vocab, float* out_lp, float* out_lse,
                                  uint32_t* err, int num_sms, cudaStream_t stream) {
  if (n_tok == 0) return cudaSuccess;
  const int grid = grid_rows(n_tok, num_sms, 8);
  const size_t es = in == DType::BF16 ? 2 : 4;
  const int vn = in == DType::BF16 ? 8 : 4;
  const bool aligned = (vocab % vn == 0) && ((ld * es) % 16 == 0) &&
                       (reinterpret_cast<uintptr_t>(logits) % 16 == 0);
  if (in == DType::BF16) {
    auto lg = static_cast<const __nv_bfloat16*>(logits);
    if (aligned)
      logprob_gather_kernel<__nv_bfloat16, true><<<grid, 256, 0, stream>>>(lg, ld, target, n_tok, vocab, out_lp, out_lse, err);
    else
      logprob_gather_kernel<__nv_bfloat16, false><<<grid, 256, 0, stream>>>(lg, ld, target, n_tok, vocab, out_lp, out_lse, err);
  } else {
    auto lg = static_cast<const float*>(logits);
    if (aligned)
      logprob_gather_kernel<float, true><<<grid, 256, 0, stream>>>(lg, ld, target, n_tok, vocab, out_lp, out_lse, err);
    else
      logprob_gather_kernel<float, false><<<grid, 256, 0, stream>>>(lg, ld, target, n_tok, vocab, out_lp, out_lse, err);
  }
  return cudaGetLastError();
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
  const int64_t blocks = (n_tok + 255) / 256;
  behaviour_kernel<<<static_cast<unsigned>(blocks < 65535 ? blocks : 65535), 256, 0, stream>>>(
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

cudaError_t launch_reduce(const double* obj, const uint8_t* flags, int64_t n_tok, double* out4,
                          void* scratch, int num_sms, cudaStream_t stream) {
  (void)num_sms;
  int64_t nb = (n_tok + 4 * kReduceThreads - 1) / (4 * kReduceThreads);
  if (nb > kReduceBlocks) nb = kReduceBlocks;
  if (nb < 1) nb = 1;
  reduce_kernel<<<static_cast<unsigned>(nb), kReduceThreads, 0, stream>>>(
      obj, flags, n_tok, out4, static_cast<ReduceScratch*>(scratch));
  return cudaGetLastError();
}

}  // namespace copris_b200
