/*
 * copris_oracle.h — TEST INFRASTRUCTURE ONLY. Not part of the product.
 *
 * CPU fp64 restatement of the reference's IS-corrected GRPO loss path
 * (CoPRIS, arXiv 2511.05589; reference = /root/reference/proj/include/copris),
 * in the row-per-token layout the GPU path uses: logits[t * ld + k] is the
 * logit row of packed token t. Every function cites the reference lines it
 * restates op-for-op (same operation order, fp64, no FMA contraction), so its
 * results are bit-identical to the reference on log-probs and loss.
 *
 * Parity pinning: tests/test_oracle.py checks this file against
 *   (a) the reference's own known-answer tests (test_policy.cpp, test_grpo.cpp),
 *   (b) golden fixtures captured from the reference itself (tests/golden/,
 *       made by oracle/gen_golden.cpp compiled against the reference headers),
 *   (c) oracle/_ref/libcopris_ref.so (reference compiled from its own headers)
 *       on random inputs, when that library is present.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
 * this code, and only as the checker.
 */
#ifndef COPRIS_ORACLE_H
#define COPRIS_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes mirror the reference's exception types (common.hpp:9-22) */
enum { ORACLE_OK = 0, ORACLE_E_CONTRACT = 1, ORACLE_E_CONFIG = 2 };

/* message of the last error on this thread (reference's fixed what() string) */
const char* oracle_last_error(void);

/* policy.hpp:114-120,170 (token_distribution_into + sequence_logprobs):
 * out_lp[t] = log(softmax(row_t)[target[t]]). Token outside [0,V) ->
 * ORACLE_E_CONTRACT "token out of vocabulary" (policy.hpp:169). */
int oracle_logprob_gather(const double* logits, int64_t ld, const int32_t* target,
                          int64_t n_tok, int32_t vocab, double* out_lp);

/* trajectory.hpp:69-75 (concat_segments) + trainer.hpp:149 (IS off) expressed
 * per token: behav[t] = (is_enabled && stage[t] < cur_stage) ? buffered_lp[t]
 * : cur_lp[t] (behav_mode 0); behav_mode 1 takes buffered_lp for every token
 * when IS is on. Counts stale tokens as rollout.hpp:99-110 does. */
void oracle_behaviour(const uint32_t* stage, uint32_t cur_stage, const double* buffered_lp,
                      const double* cur_lp, int is_enabled, int behav_mode, int64_t n_tok,
                      double* out_behav, int64_t* out_stale);

/* grpo.hpp:51-65 (compute_advantages), applied group by group. Groups are
 * trajectory ranges [group_off[g], group_off[g+1]). G<2 -> ORACLE_E_CONFIG. */
int oracle_advantages(const double* rewards, const int64_t* group_off, int64_t n_groups,
                      double adv_epsilon, double* out_adv);

/* grpo.hpp:35-47 (terminal_reward) over packed trajectories. */
int oracle_terminal_rewards(const int32_t* tokens, const int64_t* tok_off, int64_t n_traj,
                            const uint8_t* terminated, const int32_t* answer_target,
                            int32_t eos_token, double* out_reward);

typedef struct {
  double clip_low, clip_high, kl_coeff, entropy_coeff;
  int is_enabled;
  int behav_mode; /* 0: current-stage tokens use the recomputed lp; 1: recorded */
} oracle_clip_cfg;

typedef struct {
  const double* logits;      /* [n_tok x ld] */
  int64_t ld;
  int32_t vocab;
  int64_t n_tok;
  int64_t n_traj;
  const int64_t* tok_off;    /* [n_traj+1] */
  const int32_t* target;     /* [n_tok]: the generated tokens */
  const uint32_t* stage;     /* [n_tok]: policy version of the token's segment */
  uint32_t cur_stage;        /* rollout_version of the batch */
  const double* buffered_lp; /* [n_tok]: concat_segments values */
  const double* ref_lp;      /* [n_tok] or NULL (only read when kl_coeff > 0) */
  const double* adv;         /* [n_traj] */
} oracle_batch;

typedef struct {
  double loss;
  double objective;  /* sum before the -1/T scaling */
  double* dlogits;   /* [n_tok x vocab] or NULL */
  double* cur_lp;    /* [n_tok] or NULL */
  double* behav;     /* [n_tok] or NULL */
  double* weight;    /* [n_tok] or NULL: w_t of grpo.hpp:150-162 */
  uint8_t* clipped;  /* [n_tok] or NULL: 1 where the clamp branch binds */
  double* obj;       /* [n_tok] or NULL: the token's objective terms (clip - KL + entropy) */
  int64_t stale_tokens;
  int64_t clipped_tokens;
} oracle_result;

/* grpo.hpp:117-185 (grpo_step_loss) with policy.hpp:180-196
 * (accumulate_weighted_logprob_grad) in row-per-token form. */
int oracle_is_loss(const oracle_batch* b, const oracle_clip_cfg* cfg, oracle_result* out);

#ifdef __cplusplus
}
#endif
#endif
