/*
 * copris_oracle.c — TEST INFRASTRUCTURE ONLY (see copris_oracle.h).
 *
 * fp64 restatement of the reference hot path, operation order preserved so
 * the results are bit-identical to /root/reference/proj/include/copris on
 * log-probs and loss. Build with -ffp-contract=off (oracle/Makefile).
 */
#include "copris_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local const char* g_err = "";

const char* oracle_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  g_err = msg;
  return code;
}

/* policy.hpp:114-120 token_distribution_into: max, exp(z - max), sum, divide. */
static void softmax_row(const double* row, int32_t v, double* out) {
  double mx = row[0];
  for (int32_t k = 1; k < v; ++k)
    if (row[k] > mx) mx = row[k]; /* std::max_element keeps the first max */
  double sum = 0.0;
  for (int32_t k = 0; k < v; ++k) {
    out[k] = exp(row[k] - mx);
    sum += out[k];
  }
  for (int32_t k = 0; k < v; ++k) out[k] /= sum;
}

int oracle_logprob_gather(const double* logits, int64_t ld, const int32_t* target,
                          int64_t n_tok, int32_t vocab, double* out_lp) {
  if (n_tok == 0) return ORACLE_OK; /* test_policy.cpp:151-155: empty -> empty */
  double* probs = (double*)malloc(sizeof(double) * (size_t)vocab);
  for (int64_t t = 0; t < n_tok; ++t) {
    softmax_row(logits + t * ld, vocab, probs);
    int32_t tok = target[t];
    if (tok < 0 || tok >= vocab) { /* policy.hpp:169 */
      free(probs);
      return fail(ORACLE_E_CONTRACT, "token out of vocabulary");
    }
    out_lp[t] = log(probs[tok]); /* policy.hpp:170 */
  }
  free(probs);
  return ORACLE_OK;
}

void oracle_behaviour(const uint32_t* stage, uint32_t cur_stage, const double* buffered_lp,
                      const double* cur_lp, int is_enabled, int behav_mode, int64_t n_tok,
                      double* out_behav, int64_t* out_stale) {
  int64_t stale = 0;
  for (int64_t t = 0; t < n_tok; ++t) {
    int old = stage[t] < cur_stage; /* rollout.hpp:105 */
    stale += old;
    /* trajectory.hpp:69-75 + trainer.hpp:149 (IS off -> current_lp). Mode 1
     * (recorded) is concat_segments verbatim for every token. */
    out_behav[t] = (is_enabled && (old || behav_mode == 1)) ? buffered_lp[t] : cur_lp[t];
  }
  if (out_stale) *out_stale = stale;
}

int oracle_advantages(const double* rewards, const int64_t* group_off, int64_t n_groups,
                      double adv_epsilon, double* out_adv) {
  for (int64_t g = 0; g < n_groups; ++g) {
    const int64_t b = group_off[g], e = group_off[g + 1];
    const int64_t n = e - b;
    if (n < 2) return fail(ORACLE_E_CONFIG, "advantage group size must be >= 2"); /* :54 */
    double mean = 0.0;
    for (int64_t i = b; i < e; ++i) mean += rewards[i];
    mean /= (double)n;
    double var = 0.0;
    for (int64_t i = b; i < e; ++i) var += (rewards[i] - mean) * (rewards[i] - mean);
    var /= (double)n;
    double denom = sqrt(var) + adv_epsilon;
    for (int64_t i = b; i < e; ++i) out_adv[i] = (rewards[i] - mean) / denom;
  }
  return ORACLE_OK;
}

int oracle_terminal_rewards(const int32_t* tokens, const int64_t* tok_off, int64_t n_traj,
                            const uint8_t* terminated, const int32_t* answer_target,
                            int32_t eos_token, double* out_reward) {
  for (int64_t i = 0; i < n_traj; ++i) {
    const int64_t b = tok_off[i], n = tok_off[i + 1] - tok_off[i];
    if (!terminated[i])
      return fail(ORACLE_E_CONTRACT, "terminal_reward requires a terminated trajectory");
    if (n == 0) return fail(ORACLE_E_CONTRACT, "terminated trajectory cannot be empty");
    int32_t answer;
    if (tokens[b + n - 1] == eos_token) {
      if (n < 2) { /* bare EOS, grpo.hpp:40 */
        out_reward[i] = 0.0;
        continue;
      }
      answer = tokens[b + n - 2];
    } else {
      answer = tokens[b + n - 1]; /* truncated at horizon, grpo.hpp:43 */
    }
    out_reward[i] = answer == answer_target[i] ? 1.0 : 0.0;
  }
  return ORACLE_OK;
}

int oracle_is_loss(const oracle_batch* b, const oracle_clip_cfg* cfg, oracle_result* out) {
  /* grpo.hpp:120-133 validation, in the reference's order */
  if (b->n_traj == 0) return fail(ORACLE_E_CONFIG, "grpo_step_loss requires a non-empty batch");
  int64_t total = 0;
  for (int64_t i = 0; i < b->n_traj; ++i) {
    if (cfg->kl_coeff != 0.0 && b->ref_lp == NULL)
      return fail(ORACLE_E_CONTRACT, "reference log-probs required when kl_coeff > 0");
    if (!isfinite(b->adv[i])) return fail(ORACLE_E_CONTRACT, "advantage must be finite");
    total += b->tok_off[i + 1] - b->tok_off[i];
  }
  if (total == 0) return fail(ORACLE_E_CONFIG, "grpo_step_loss batch has no tokens");

  const int32_t V = b->vocab;
  double* cur = (double*)malloc(sizeof(double) * (size_t)total);
  double* behav = (double*)malloc(sizeof(double) * (size_t)total);
  double* w = (double*)calloc((size_t)total, sizeof(double));
  double* probs = (double*)malloc(sizeof(double) * (size_t)V);
  int rc = oracle_logprob_gather(b->logits, b->ld, b->target, total, V, cur);
  if (rc) goto done;
  int64_t stale = 0;
  oracle_behaviour(b->stage, b->cur_stage, b->buffered_lp, cur, cfg->is_enabled, cfg->behav_mode,
                   total, behav, &stale);

  const double inv_t = 1.0 / (double)total; /* grpo.hpp:135 */
  if (out->dlogits) memset(out->dlogits, 0, sizeof(double) * (size_t)total * (size_t)V);
  double objective = 0.0;
  int64_t n_clipped = 0;
  for (int64_t i = 0; i < b->n_traj; ++i) {
    const double adv = b->adv[i];
    const int64_t t0 = b->tok_off[i], t1 = b->tok_off[i + 1];
    for (int64_t t = t0; t < t1; ++t) { /* grpo.hpp:147-163 */
      if (!isfinite(cur[t]) || !isfinite(behav[t])) {
        rc = fail(ORACLE_E_CONTRACT, "token_ratio requires finite log-probs");
        goto done;
      }
      double ratio = exp(cur[t] - behav[t]);
      double clamped = ratio;
      if (clamped < 1.0 - cfg->clip_low) clamped = 1.0 - cfg->clip_low;
      if (clamped > 1.0 + cfg->clip_high) clamped = 1.0 + cfg->clip_high;
      double unclipped = ratio * adv;
      double clipped = clamped * adv;
      int bind = 0;
      if (unclipped <= clipped) {
        objective += unclipped;
        w[t] = ratio * adv;
      } else {
        objective += clipped;
        bind = 1;
      }
      if (out->obj) out->obj[t] = bind ? clipped : unclipped;
      n_clipped += bind;
      if (out->clipped) out->clipped[t] = (uint8_t)bind;
      if (cfg->kl_coeff > 0.0) { /* grpo.hpp:158-162 */
        double d = b->ref_lp[t] - cur[t];
        objective -= cfg->kl_coeff * (exp(d) - d - 1.0);
        w[t] += cfg->kl_coeff * (exp(d) - 1.0);
        if (out->obj) out->obj[t] -= cfg->kl_coeff * (exp(d) - d - 1.0);
      }
    }
    /* policy.hpp:180-196 with scale = -inv_t (grpo.hpp:166-167) */
    if (out->dlogits) {
      for (int64_t t = t0; t < t1; ++t) {
        double wv = -inv_t * w[t];
        if (wv == 0.0) continue;
        softmax_row(b->logits + t * b->ld, V, probs);
        double* g = out->dlogits + t * (int64_t)V;
        for (int32_t k = 0; k < V; ++k) g[k] -= wv * probs[k];
        g[b->target[t]] += wv;
      }
    }
    if (cfg->entropy_coeff != 0.0) { /* grpo.hpp:168-181 */
      for (int64_t t = t0; t < t1; ++t) {
        softmax_row(b->logits + t * b->ld, V, probs);
        double h = 0.0;
        for (int32_t k = 0; k < V; ++k) h -= probs[k] * log(probs[k]);
        objective += cfg->entropy_coeff * h;
        if (out->obj) out->obj[t] += cfg->entropy_coeff * h;
        if (out->dlogits) {
          double* g = out->dlogits + t * (int64_t)V;
          for (int32_t k = 0; k < V; ++k) {
            double dh = -probs[k] * (log(probs[k]) + h);
            g[k] -= inv_t * cfg->entropy_coeff * dh;
          }
        }
      }
    }
  }
  out->objective = objective;
  out->loss = -objective * inv_t; /* grpo.hpp:183 */
  out->stale_tokens = stale;
  out->clipped_tokens = n_clipped;
  if (out->cur_lp) memcpy(out->cur_lp, cur, sizeof(double) * (size_t)total);
  if (out->behav) memcpy(out->behav, behav, sizeof(double) * (size_t)total);
  if (out->weight) memcpy(out->weight, w, sizeof(double) * (size_t)total);
done:
  free(cur);
  free(behav);
  free(w);
  free(probs);
  return rc;
}
