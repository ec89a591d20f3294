// token_math.cuh — per-token scalar semantics shared by every loss kernel, so
// the fused, generic and unfused paths agree on branch selection and rounding.
//
// Restates grpo.hpp:147-181 (ratio, asymmetric clip, KL, entropy objective)
// and the scale of policy.hpp:180-196 for ONE token, in fp64, with the
// reference's operation order. The V-length work stays in the kernels.
#pragma once

#include <cstdint>

#include "kernels.cuh"

namespace copris_b200 {

constexpr float kLog2e = 1.4426950408889634f;
constexpr double kLog2eD = 1.4426950408889634;

enum : uint8_t { FLAG_STALE = 1, FLAG_CLIPPED = 2, FLAG_MASKED = 4 };

// trajectory.hpp:69-75 (concat_segments) + trainer.hpp:149 (IS off) for one
// token. A select, never arithmetic: bit-exact by construction.
__device__ __forceinline__ float select_behaviour(uint32_t stage, uint32_t cur_stage, float blp,
                                                  float cur, int is_enabled, int behav_mode) {
  return (is_enabled && (stage < cur_stage || behav_mode == 1)) ? blp : cur;
}

struct TokenResult {
  double obj;    // this token's objective contribution
  double coef;   // dlogits row scale: -w/T (policy.hpp:188 with scale -inv_t)
  uint8_t flags;
  uint32_t err;
};

// grpo.hpp:147-162 (+ 170-171 when `ent`): cur/beh are the f32 log-probs,
// H the row entropy in nats (only read when ent). The ratio and the KL
// exponential are fp32 expf (fp64 exp beyond |x| >= 80, where expf would
// overflow), and the products and sums that decide the branch and form w, obj
// and coef are fp64 in the reference's order, so a current-stage token (ratio
// exactly 1) gets w = A and coef = -A/T bit for bit.
__device__ __forceinline__ TokenResult token_objective(const LossParams& P, float cur, float beh,
                                                       double adv, float ref, bool stale,
                                                       float H, bool ent) {
  TokenResult r{0.0, 0.0, static_cast<uint8_t>(stale ? FLAG_STALE : 0), 0u};
  if (!isfinite(adv)) {
    r.err = ERR_NONFINITE_ADV;
    return r;
  }
  if (!isfinite(cur) || !isfinite(beh)) {  // grpo.hpp:69-70 token_ratio
    r.err = ERR_NONFINITE_LP;
    return r;
  }
  // exp in fp32 (<= 2 ulp, on the scalar phase's critical path) unless the token
  // is far off policy (|cur - beh| >= 80, where expf would overflow at 88): then
  // fp64, as the reference (grpo.hpp:71), finite up to e^709, so the objective
  // and the fp64 coef keep the reference's values; cur == beh gives exactly 1
  const float dr = cur - beh;
  const double ratio = fabsf(dr) < 80.f ? static_cast<double>(expf(dr))
                                        : exp(static_cast<double>(cur) - static_cast<double>(beh));
  // std::clamp(ratio, 1 - clip_low, 1 + clip_high), grpo.hpp:149
  const double clamped = ratio < P.clamp_lo ? P.clamp_lo : (P.clamp_hi < ratio ? P.clamp_hi : ratio);
  const double unclipped = __dmul_rn(ratio, adv);
  const double clipped = __dmul_rn(clamped, adv);
  double obj, w = 0.0;
  if (unclipped <= clipped) {  // ties take the unclipped branch (grpo.hpp:152)
    obj = unclipped;
    w = __dmul_rn(ratio, adv);
  } else {
    obj = clipped;  // binding clamp: zero gradient
    r.flags |= FLAG_CLIPPED;
  }
  if (P.kl_coeff > 0.0) {  // grpo.hpp:158-162
    const float df = ref - cur;
    const double d = static_cast<double>(df);
    const double ed = fabsf(df) < 80.f ? static_cast<double>(expf(df))
                                       : exp(static_cast<double>(ref) - static_cast<double>(cur));
    obj = __dadd_rn(obj, -__dmul_rn(P.kl_coeff, __dadd_rn(__dadd_rn(ed, -d), -1.0)));
    w = __dadd_rn(w, __dmul_rn(P.kl_coeff, __dadd_rn(ed, -1.0)));
  }
  if (ent) obj = __dadd_rn(obj, __dmul_rn(P.entropy_coeff, static_cast<double>(H)));
  r.obj = obj;
  r.coef = __dmul_rn(-P.inv_t, w);
  return r;
}

// log-prob and log-sum-exp of one row from the online state (m, s = sum over
// the NON-target columns of e^(z-m)) and the target logit z_y. With
// dz = z_y - m and r = s e^(-dz) = sum_{k!=y} p_k / p_y:
//   cur = log p_y = -log1p(r),  ln S = dz + log1p(r),  lse = m + ln S.
// log1p keeps cur accurate when the target saturates the row (p_y -> 1),
// where log(e^dz + s) would lose r to the rounding of 1 + r. fp64: O(1) work.
struct LogProb {
  float cur;
  double lse;
  float ln_s;
  float S;
};

__device__ __forceinline__ LogProb finish_logprob(float M, float s_excl, float zy, bool ok) {
  LogProb q;
  if (!ok) {
    q.ln_s = logf(s_excl);
    q.S = s_excl;
    q.lse = static_cast<double>(M) + q.ln_s;
    q.cur = __int_as_float(0x7fc00000);
    return q;
  }
  if (M == -INFINITY) {  // every other column is -inf (masked vocabulary): p_y = 1
    M = zy;
    s_excl = 0.f;
  }
  const float dz = zy - M;
  if (dz < -64.f) {
    // target far below the row maximum (p_y < e^-64): s_excl e^-dz would
    // overflow fp32; s_excl >= 1 (it holds the max column's e^0), so
    // ln S = ln s_excl + log1p(e^dz / s_excl) is exact to rounding
    const float ey = expf(dz);
    q.ln_s = logf(s_excl) + log1pf(ey / s_excl);
    q.cur = dz - q.ln_s;
    q.S = s_excl + ey;
    q.lse = static_cast<double>(M) + static_cast<double>(q.ln_s);
    return q;
  }
  const float r = s_excl * expf(-dz);
  const float l1 = log1pf(r);
  q.cur = -l1;
  q.ln_s = dz + l1;
  q.S = s_excl + expf(dz);
  q.lse = static_cast<double>(M) + static_cast<double>(q.ln_s);
  return q;
}

// Values pass C of a row needs, broadcast from the scalar phase.
struct RowBroadcast {
  float coef;    // dlogits scale of the one-hot/softmax term
  float dy;      // dlogits of the target column: coef * (1 - p_y)
  float m;       // row max (pass-B frame)
  float log2s;   // log2(sum exp(z - m))
  float c1;      // m*log2(e) + log2(S): p_k = 2^(z_k log2(e) - c1)
  int32_t y;     // target column
  float eg;      // entropy gradient scale c_H/T (0 when off or on error)
  float k0;      // H - ln(S): log p + H = (z - m) + k0
  float c2;      // c1 - log2|coef|: |dlogits_k| = 2^(z_k log2(e) - c2) off the target
  uint32_t smask;  // bf16x2 sign mask of -coef (0x80008000 when coef > 0)
};

// The scalar phase of one row: given the row's (max, sum exp(z-m), sum
// exp(z-m)(z-m)) and the target logit, produce cur_lp, behaviour, objective and
// the dlogits coefficients; write the per-token outputs when `write`.
template <bool ENT, typename LseT>
__device__ __forceinline__ RowBroadcast row_scalar_phase(const LossParams& P, int64_t t, int32_t y,
                                                         uint32_t st, float blp, float rl,
                                                         double adv, const LseT& tot, float zy,
                                                         bool write, bool keep = true) {
  const bool oov = static_cast<uint32_t>(y) >= static_cast<uint32_t>(P.vocab);
  const float M = tot.m;
  const LogProb lp = finish_logprob(M, tot.s, zy, !oov);
  if (P.gather_only) {  // K1 (sequence_logprobs): the log-prob and LSE only
    if (oov) atomicOr(P.err, ERR_TOKEN_OOV);  // policy.hpp:169
    if (write) {
      P.cur_lp[t] = lp.cur;
      if (P.lse) P.lse[t] = static_cast<float>(lp.lse);
    }
    RowBroadcast z{};
    return z;
  }
  const float ln_s = lp.ln_s;
  const double lse = lp.lse;
  const float cur = lp.cur;
  const bool stale = st < static_cast<uint32_t>(P.cur_stage);
  const float beh = select_behaviour(st, static_cast<uint32_t>(P.cur_stage), blp, cur, P.is_enabled,
                                     P.behav_mode);
  float H = 0.f;
  if (ENT) H = ln_s - tot.u / tot.a;
  TokenResult tr;
  if (!keep) {  // masked token: out of the loss as if absent from the batch
    tr = TokenResult{0.0, 0.0, FLAG_MASKED, 0u};
  } else if (oov) {
    tr = TokenResult{0.0, 0.0, static_cast<uint8_t>(stale ? FLAG_STALE : 0), ERR_TOKEN_OOV};
  } else {
    tr = token_objective(P, cur, beh, adv, rl, stale, H, ENT);
  }
  if (tr.err) {
    atomicOr(P.err, tr.err);
    tr.obj = 0.0;
    tr.coef = 0.0;
  }
  if (write) {
    P.cur_lp[t] = cur;
    if (P.lse) P.lse[t] = static_cast<float>(lse);
    if (P.behav) P.behav[t] = beh;
    P.obj[t] = tr.obj;
    if (P.coef) P.coef[t] = tr.coef;
    P.flags[t] = tr.flags;
  }
  RowBroadcast b;
  b.coef = static_cast<float>(tr.coef);
  b.dy = tr.err ? 0.f : static_cast<float>(tr.coef) * -expm1f(cur);  // coef*(1-p_y)
  b.m = M;
  b.log2s = ln_s * kLog2e;
  b.c1 = static_cast<float>(static_cast<double>(M) * kLog2eD + static_cast<double>(ln_s) * kLog2eD);
  b.y = y;
  b.eg = (ENT && !tr.err) ? static_cast<float>(P.inv_t * P.entropy_coeff) : 0.f;
  b.k0 = ENT ? H - ln_s : 0.f;
  // log2|coef| in fp32 (MUFU lg2, ~1 ulp of |log2| <= ~40, i.e. <= 2^-18 in the
  // exponent of a bf16 output) instead of a fp64 log2 on every row's critical path
  const float ac = fabsf(b.coef);
  b.c2 = ac > 0.f ? static_cast<float>(static_cast<double>(M) * kLog2eD +
                                       static_cast<double>(ln_s) * kLog2eD -
                                       static_cast<double>(log2f(ac)))
                  : 0.f;
  b.smask = b.coef > 0.f ? 0x80008000u : 0u;
  return b;
}

}  // namespace copris_b200
