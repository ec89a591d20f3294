/*
 * copris_b200.h — C-ABI of the B200-native CoPRIS IS-corrected loss path.
 *
 * Drop-in boundary for the reference's loss entry points
 * (/root/reference/proj/include/copris). The reference is header-only C++ with
 * no FFI of its own; each entry point below names the reference function it
 * replaces. All pointers are caller-owned DEVICE buffers unless a parameter
 * says "host". `stream` is a cudaStream_t passed as void* (NULL = legacy
 * default stream). No call allocates on the hot path and no call falls back to
 * the CPU: every compute entry point launches sm_100a kernels or fails.
 *
 * Status: every call returns COPRIS_OK (0) or an error code; the message is in
 * copris_last_error() (thread-local). COPRIS_E_CONTRACT / COPRIS_E_CONFIG carry
 * the reference's exception type (ContractViolation / ConfigError,
 * common.hpp:9-18) and its fixed message. Conditions only the device can see
 * (token outside the vocabulary, non-finite log-prob) are latched in a device
 * error word and reported by copris_ctx_check().
 *
 * Packed batch layout: trajectories are concatenated in
 * batch order (groups in batch order, members ascending traj_id,
 * rollout.hpp:75-95); token t of the packed batch is row t of the logits.
 *   tok_off[n_traj+1]  int64   token offsets of trajectories
 *   group_off[P+1]     int64   trajectory offsets of prompt groups
 *   target[T]          int32   generated token ids
 *   stage[T]           uint32  policy version of the segment holding token t
 *   buffered_lp[T]     f32     concat_segments() values (trajectory.hpp:69-75)
 *   tok_traj[T]        int32   trajectory index of token t
 *   adv[n_traj]        f64     group-relative advantages
 */
#ifndef COPRIS_B200_H
#define COPRIS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define COPRIS_B200_ABI_VERSION 3

#if defined(__GNUC__)
#define COPRIS_API __attribute__((visibility("default")))
#else
#define COPRIS_API
#endif

enum copris_status {
  COPRIS_OK = 0,
  COPRIS_E_CONTRACT = 1, /* copris::ContractViolation */
  COPRIS_E_CONFIG = 2,   /* copris::ConfigError */
  COPRIS_E_CUDA = 3,     /* CUDA runtime / launch failure */
  COPRIS_E_INVALID = 4   /* malformed call (null pointer, bad dtype, ...) */
};

enum copris_dtype { COPRIS_BF16 = 0, COPRIS_F32 = 1 };

/* Source of the behaviour log-prob of CURRENT-stage tokens when IS is on.
 * RECOMPUTED (default): the recomputed current log-prob, which the reference's
 *   sampler records bit-identically (test_policy.cpp:157-172), so the ratio of
 *   every current-stage token is exactly 1 (acceptance C3).
 * RECORDED: buffered_lp for every token, i.e. concat_segments() verbatim. */
enum copris_behav_mode { COPRIS_BEHAV_RECOMPUTED = 0, COPRIS_BEHAV_RECORDED = 1 };

/* bits of the per-token flags byte */
enum { COPRIS_FLAG_STALE = 1, COPRIS_FLAG_CLIPPED = 2, COPRIS_FLAG_MASKED = 4 };

typedef struct copris_ctx copris_ctx;

COPRIS_API int copris_abi_version(void);
COPRIS_API const char* copris_last_error(void);

/* Context: device binding, SM count, device error word, row-claim counter and
 * reduction scratch. Re-entrant: one context per (thread, device) or shared
 * under the caller's lock; no global mutable state (SURVEY.md §8(b) Threading).
 * A context's launches must not overlap on different streams (the row-claim
 * counter and the reduction scratch are per context): issue them on one
 * stream, or use one context per stream. */
COPRIS_API int copris_ctx_create(int device, copris_ctx** out);
COPRIS_API int copris_ctx_destroy(copris_ctx* ctx);
/* Kernel selection and tunables of this context (not a reference entry point).
 * copris_ctx_create reads the COPRIS_* environment ONCE into the context;
 * launches never read the environment again. Change an option between
 * launches (not concurrently with a launch on the same context). Names:
 * fused_impl (0 auto, 1 stream, 2 tma, 3 pair, 4 solo), lookahead, slots, resident,
 * pair_lookahead, pair_st256, pair_bf16_stage, pair_pw8, pair_dynamic, lmhead_impl (0 pair, 1 single SM), lmhead_group, lmhead_tma_store,
 * gemm_wide, gemm_mc, gemm_splits, gemm_a_evict_first, dw_group, dw_policy,
 * dw_kchunk, trace. COPRIS_E_INVALID for an unknown name or out-of-range value. */
COPRIS_API int copris_ctx_set_option(copris_ctx* ctx, const char* name, int64_t value);
COPRIS_API int copris_ctx_get_option(const copris_ctx* ctx, const char* name, int64_t* value);
/* Synchronises `stream`, then reports and clears the device error word. */
COPRIS_API int copris_ctx_check(copris_ctx* ctx, void* stream);

/* ---- K1: streaming log-softmax + gather ------------------------------------
 * Replaces sequence_logprobs (policy.hpp:160-173) over packed rows:
 *   out_lp[t] = z[t][target[t]] - logsumexp(z[t]),  out_lse[t] = logsumexp(z[t]).
 * Rows are logits + r*ld for r in [0,n_tok); target/out indexed by r.
 * out_lse may be NULL. Token outside [0,vocab) -> device error
 * "token out of vocabulary" (policy.hpp:169). */
COPRIS_API int copris_logprob_gather(copris_ctx* ctx, const void* logits, int64_t ld, int32_t dtype,
                          const int32_t* target, int64_t n_tok, int32_t vocab, float* out_lp,
                          float* out_lse, void* stream);

/* ---- LM-head forward fused with the log-softmax statistics -----------------
 * SURVEY.md §8(f) rank 3 (producer of a8, trainer.hpp:146). On tcgen05 tensor
 * cores: logits[t][k] = bf16( sum_h hidden[t][h] * weight[k][h] ) (fp32
 * accumulate) for t < n_rows, k < vocab, written with row stride ld_logits,
 * plus partials[t][j] = {max, sum_{k in tile j, k != target[t]} exp(z - max)}
 * (float2, n_vt = copris_lmhead_num_vtiles(vocab) per row) of the ROUNDED
 * logits. hidden [n_rows x hidden_dim] and weight [vocab x hidden_dim]
 * (nn.Linear layout) are bf16 with 16-byte aligned row strides ld_hidden /
 * ld_weight (elements); ld_logits % 8 == 0.
 * copris_lse_merge then yields exactly what copris_logprob_gather computes
 * from the stored logits — (cur_lp, lse) — reading only the partials and the
 * target logit; the loss continues with copris_behaviour_concat +
 * copris_is_loss_bwd (one streaming pass). partials == NULL (target may then
 * be NULL): logits only, no statistics — for a step whose loss runs the
 * one-pass fused kernel (copris_is_loss_fused) on the logits; needs the
 * default CTA-pair kernel with TMA stores (vocab % 8 == 0), else
 * COPRIS_E_INVALID. */
COPRIS_API int32_t copris_lmhead_num_vtiles(int32_t vocab);
COPRIS_API int copris_lmhead_logits(copris_ctx* ctx, const void* hidden, int64_t ld_hidden,
                                    const void* weight, int64_t ld_weight, int64_t n_rows,
                                    int32_t hidden_dim, int32_t vocab, const int32_t* target,
                                    void* logits, int64_t ld_logits, float* partials,
                                    void* stream);
COPRIS_API int copris_lse_merge(copris_ctx* ctx, const float* partials, int32_t n_vt,
                                const void* logits, int64_t ld, const int32_t* target,
                                int64_t n_rows, int32_t vocab, float* out_lp, float* out_lse,
                                void* stream);

/* LM-head backward, hidden gradient, on the same CTA-pair tcgen05 kernel:
 *   dhidden[t][h] = bf16( sum_k dlogits[t][k] * weight_t[h][k] )   (fp32 accumulate)
 * for t < n_rows, h < hidden_dim; weight_t = weight^T [hidden_dim x vocab]
 * (K-major along the vocab, transposed once per optimizer step). The vocab
 * reduction is split over copris_lmhead_dhidden_splits(...) ranges into
 * `work` (splits * n_rows * hidden_dim fp32) and summed in a fixed order, so
 * reruns are bitwise identical. hidden_dim % 4 == 0; bf16 operands with
 * 16-byte aligned rows (ld_* in elements). */
COPRIS_API int32_t copris_lmhead_dhidden_splits(copris_ctx* ctx, int64_t n_rows, int32_t hidden_dim);
COPRIS_API int copris_lmhead_dhidden(copris_ctx* ctx, const void* dlogits, int64_t ld_dlogits,
                                     const void* weight_t, int64_t ld_weight_t, int64_t n_rows,
                                     int32_t hidden_dim, int32_t vocab, void* dhidden,
                                     int64_t ld_dhidden, float* work, void* stream);

/* LM-head backward, weight gradient, on the same CTA-pair tcgen05 kernel with
 * both operands MN-major (the token dimension is the reduction):
 *   dweight[k][h] += sum_t dlogits[t][k] * hidden[t][h]   (fp32 accumulate)
 * for k < vocab, h < hidden_dim, t < n_rows; dweight is fp32 [vocab x
 * hidden_dim] (ld_dweight % 4 == 0, 16-byte aligned). Each 256 x 256 tile of
 * dweight is accumulated by one CTA pair in token order, so reruns are bitwise
 * identical. Replaces the cuBLAS addmm of the reference-facing trainer step
 * (the table-gradient scatter of trainer.hpp:176 in the LLM setting). */
COPRIS_API int copris_lmhead_dweight(copris_ctx* ctx, const void* dlogits, int64_t ld_dlogits,
                                     const void* hidden, int64_t ld_hidden, int64_t n_rows,
                                     int32_t hidden_dim, int32_t vocab, float* dweight,
                                     int64_t ld_dweight, void* stream);

/* ---- K2: segmented cross-stage behaviour concat -----------------------------
 * copris_expand_segments: per-token stage ids from segment tables
 *   (segments in packed order; seg_off[n_seg+1] token offsets, seg_ver[n_seg]).
 * copris_behaviour_concat replaces concat_segments (trajectory.hpp:69-75) and
 *   the IS-off substitution (trainer.hpp:149):
 *   behav[t] = is_enabled ? (stage[t] < cur_stage || mode == RECORDED
 *                            ? buffered_lp[t] : cur_lp[t]) : cur_lp[t]
 *   Bit-exact (a select, no arithmetic). out_flags (optional) gets
 *   COPRIS_FLAG_STALE where stage[t] < cur_stage (rollout.hpp:105). */
COPRIS_API int copris_expand_segments(copris_ctx* ctx, const int64_t* seg_off, const uint32_t* seg_ver,
                           int64_t n_seg, uint32_t* out_stage, void* stream);
COPRIS_API int copris_behaviour_concat(copris_ctx* ctx, const uint32_t* stage, uint32_t cur_stage,
                            const float* buffered_lp, const float* cur_lp, int32_t is_enabled,
                            int32_t behav_mode, int64_t n_tok, float* out_behav,
                            uint8_t* out_flags, void* stream);

/* ---- K3a: rewards and group-normalised advantages ---------------------------
 * copris_terminal_rewards replaces terminal_reward (grpo.hpp:35-47);
 * copris_group_advantages replaces compute_advantages (grpo.hpp:51-65) for all
 *   groups at once: adv = (R - mean) / (population std + adv_epsilon), fp64.
 *   A group with fewer than 2 members -> COPRIS_E_CONFIG
 *   "advantage group size must be >= 2" (checked on the host from group_off,
 *   which is therefore a HOST array here).
 * copris_token_traj expands tok_off (device array) into the per-token
 *   trajectory index tok_traj[T]. */
COPRIS_API int copris_terminal_rewards(copris_ctx* ctx, const int32_t* tokens, const int64_t* tok_off,
                            int64_t n_traj, const uint8_t* terminated,
                            const int32_t* answer_target, int32_t eos_token, double* out_reward,
                            void* stream);
COPRIS_API int copris_group_advantages(copris_ctx* ctx, const double* rewards,
                            const int64_t* group_off_host, const int64_t* group_off,
                            int64_t n_groups, double adv_epsilon, double* out_adv, void* stream);
COPRIS_API int copris_token_traj(copris_ctx* ctx, const int64_t* tok_off, int64_t n_traj, int64_t n_tok,
                      int32_t* out_tok_traj, void* stream);

/* ---- K3: the IS-corrected clipped GRPO loss and its logit gradient ----------
 * One call processes a CHUNK of n_rows packed rows whose packed token indices
 * are [row_base, row_base + n_rows): logits/dlogits are chunk-local (row r at
 * ptr + r*ld), every per-token array is indexed by the packed index. Per token
 * (grpo.hpp:147-181, policy.hpp:180-196):
 *   r = exp(cur - behav); c = clamp(r, 1-clip_low, 1+clip_high)
 *   u = r*A, v = c*A; u <= v ? (obj = u, w = r*A) : (obj = v, w = 0, clipped)
 *   kl:      d = ref - cur; obj -= kl*(e^d - d - 1); w += kl*(e^d - 1)
 *   entropy: obj += c_H * H
 *   dlogits[k] = coef*(1[k=y] - p_k) [+ (c_H/T) p_k (log p_k + H)], coef = -w/T
 * with T = cfg.total_tokens (the GLOBAL token count, grpo.hpp:135). The loss
 * is -sum(obj)/T, reduced by copris_loss_reduce (+ an allreduce when sharded).
 */
typedef struct {
  const void* logits;        /* [n_rows x ld] chunk */
  int64_t ld;                /* elements between rows (>= vocab) */
  int32_t logits_dtype;      /* copris_dtype */
  int32_t vocab;
  int64_t n_rows;
  int64_t row_base;          /* packed index of chunk row 0 */
  const int32_t* target;     /* [T] */
  const uint32_t* stage;     /* [T] */
  const float* buffered_lp;  /* [T] */
  const float* ref_lp;       /* [T]; required iff kl_coeff > 0 */
  const int32_t* tok_traj;   /* [T] */
  const double* adv;         /* [n_traj] */
  uint32_t cur_stage;        /* rollout_version of the batch */
  uint32_t _pad;
  /* [T] optional token mask (NULL: every token counts). A token with mask 0 is
   * left out of the loss as if it were not in the batch: obj 0, dlogits row 0,
   * no error checks, flags = COPRIS_FLAG_MASKED only, not counted by
   * copris_loss_reduce; cur_lp/lse are still written. total_tokens is then the
   * global count of UNMASKED tokens (the masked token mean). */
  const uint8_t* loss_mask;
} copris_loss_batch;

typedef struct {
  double clip_low, clip_high, kl_coeff, entropy_coeff; /* ClipConfig, grpo.hpp:15-28 */
  int32_t is_enabled;        /* RunConfig::is_enabled, trainer.hpp:23 */
  int32_t behav_mode;        /* copris_behav_mode */
  int64_t total_tokens;      /* global T for the 1/T token-mean */
} copris_loss_cfg;

typedef struct {
  void* dlogits;             /* [n_rows x ld_dlogits] chunk, or NULL (no backward) */
  int64_t ld_dlogits;
  int32_t dlogits_dtype;     /* copris_dtype */
  int32_t _pad;
  float* cur_lp;             /* [T] required */
  float* lse;                /* [T] optional */
  float* behav;              /* [T] optional */
  double* obj;               /* [T] required: per-token objective */
  double* coef;              /* [T] optional: dlogits row scale -w/T */
  uint8_t* flags;            /* [T] required: COPRIS_FLAG_* */
  /* optional DEVICE f64[4]: after this chunk, reduce rows [0, row_base + n_rows)
   * exactly as copris_loss_reduce does (bitwise the same out4); small batches
   * (<= 8,192 tokens) are reduced by the loss launch itself (its last CTA), so
   * a one-chunk step is ONE kernel launch. Pass it with the last chunk only. */
  double* out4;
} copris_loss_out;

/* Fused single pass: log-softmax+gather, behaviour select, ratio/clip/KL/
 * entropy, and dlogits from ONE read of each logits row (rows held in shared
 * memory across a 2-CTA cluster at large vocab, TMA bulk loads). */
COPRIS_API int copris_is_loss_fused(copris_ctx* ctx, const copris_loss_batch* batch,
                         const copris_loss_cfg* cfg, const copris_loss_out* out, void* stream);

/* Unfused K3: consumes cur_lp/lse (K1) and behav (K2) and streams the logits
 * a second time to write dlogits. Same per-token arithmetic as the fused path;
 * out->cur_lp/lse/behav are ignored (the inputs are passed explicitly). */
COPRIS_API int copris_is_loss_bwd(copris_ctx* ctx, const copris_loss_batch* batch,
                       const copris_loss_cfg* cfg, const float* cur_lp, const float* lse,
                       const float* behav, const copris_loss_out* out, void* stream);

/* Deterministic fixed-order reduction of the per-token outputs:
 * out4[0] = sum obj (fp64), out4[1] = tokens (without COPRIS_FLAG_MASKED ones),
 * out4[2] = stale tokens (rollout.hpp:99-110), out4[3] = clipped tokens.
 * out4 is a DEVICE f64[4]. */
COPRIS_API int copris_loss_reduce(copris_ctx* ctx, const double* obj, const uint8_t* flags, int64_t n_tok,
                       double* out4, void* stream);

/* ---- Sharded batches: the one collective --------------------
 * Each rank runs the kernels on its whole prompt groups with the GLOBAL token
 * count, reduces its own out4, then SUM-allreduces the four fp64 scalars:
 *   copris_allreduce_scalars(comm, d_out4, stream); loss = -out4[0] / T_global.
 * `comm` is an ncclComm_t (the caller's own, or one made by the helpers below:
 * one process driving several GPUs -> copris_nccl_comm_init_all, one process
 * per GPU -> copris_nccl_unique_id on rank 0, broadcast the 128 bytes, then
 * copris_nccl_comm_init_rank on every rank). NCCL is loaded at run time
 * (libnccl.so.2, the copy already in the process if any); COPRIS_E_CUDA
 * carries NCCL's message. dlogits never leave the rank. */
COPRIS_API int copris_allreduce_scalars(void* comm, double* d_buf4, void* stream);
COPRIS_API int copris_nccl_comm_init_all(int32_t n_dev, const int32_t* devices, void** out_comms);
COPRIS_API int copris_nccl_unique_id(uint8_t out_id[128]);
COPRIS_API int copris_nccl_comm_init_rank(int32_t device, int32_t n_ranks, const uint8_t id[128],
                                          int32_t rank, void** out_comm);
COPRIS_API int copris_nccl_comm_destroy(void* comm);

/* ---- Host-buffer drop-in for grpo_step_loss (grpo.hpp:117-185) -------------
 * The reference call takes host data and returns a host gradient. This entry
 * takes HOST arrays (page-locked memory lets the copies overlap compute),
 * streams the logits through a pre-allocated device workspace in chunks of
 * `chunk_rows` rows — H2D of chunk c+1, the fused kernel on chunk c and D2H of
 * chunk c-1 run on three streams — and returns when the loss, the counts and
 * (optionally) the host dlogits are ready. Synchronous, like the reference.
 * cfg->total_tokens = 0 means "this batch's own token count"; a sharded caller
 * passes the global count and sums `objective`/`loss` across ranks. */
typedef struct copris_workspace copris_workspace;

COPRIS_API int copris_workspace_create(copris_ctx* ctx, int64_t chunk_rows, int32_t vocab,
                                       int32_t logits_dtype, int32_t dlogits_dtype,
                                       int64_t max_tokens, int64_t max_traj,
                                       copris_workspace** out);
COPRIS_API int copris_workspace_destroy(copris_workspace* ws);

typedef struct {
  const void* logits;          /* host [n_tok x ld] */
  int64_t ld;
  int32_t logits_dtype;
  int32_t vocab;
  int64_t n_tok;
  int64_t n_traj;
  const int64_t* tok_off;      /* host [n_traj+1] */
  const int32_t* target;       /* host [n_tok] */
  const uint32_t* stage;       /* host [n_tok] */
  const float* buffered_lp;    /* host [n_tok] */
  const float* ref_lp;         /* host [n_tok] or NULL */
  const double* adv;           /* host [n_traj], or NULL: computed from rewards */
  const double* rewards;       /* host [n_traj] (when adv == NULL) */
  const int64_t* group_off;    /* host [n_groups+1] (when adv == NULL) */
  int64_t n_groups;
  double adv_epsilon;
  uint32_t cur_stage;
  uint32_t _pad;
} copris_host_batch;

typedef struct {
  void* dlogits;               /* host [n_tok x ld_dlogits], or NULL */
  int64_t ld_dlogits;
  int32_t dlogits_dtype;
  int32_t _pad;
  float* cur_lp;               /* host [n_tok] or NULL */
  double loss;                 /* -objective / T */
  double objective;
  int64_t token_count, stale_tokens, clipped_tokens;
} copris_host_result;

COPRIS_API int copris_grpo_step_loss_host(copris_ctx* ctx, copris_workspace* ws,
                                          const copris_host_batch* batch,
                                          const copris_loss_cfg* cfg, copris_host_result* out);

/* ---- After the gradient: Adam and checkpoints ----
 * copris_adam_update replaces AdamOptimizer::update (grpo.hpp:205-227) on
 * DEVICE fp64 params/grad/moments of n elements: `step` is the update count
 * AFTER this update (t in the reference), bias corrections use the host's
 * pow() exactly as the reference does, and the per-element arithmetic is
 * unfused fp64 — bit-identical to the reference. The caller bumps the policy
 * version. copris_checkpoint_write/read implement the CPRSCKPT format of
 * io.hpp:397-438 byte for byte (HOST pointers; dims = {Q, H, V, answer_vocab}). */
typedef struct {
  double lr, beta1, beta2, eps, weight_decay; /* AdamConfig, grpo.hpp:187-201 */
} copris_adam_cfg;

COPRIS_API int copris_adam_update(copris_ctx* ctx, double* params, const double* grad, double* m,
                                  double* v, int64_t n, int64_t step, const copris_adam_cfg* cfg,
                                  void* stream);
/* The whole AdamOptimizer object (grpo.hpp:205-235) for a HOST-side parameter
 * table: the optimizer owns device copies of the moments (the reference's m_,
 * v_) and its step count t_; each copris_adam_host_update copies params and
 * grad in, runs copris_adam_update's kernel and copies params back, on the
 * optimizer's own stream, synchronously (the reference update is a blocking
 * call). `n` must equal the size given at creation, else COPRIS_E_CONTRACT
 * "gradient shape mismatch" (grpo.hpp:210). */
typedef struct copris_adam_host copris_adam_host;
COPRIS_API int copris_adam_host_create(copris_ctx* ctx, int64_t n, const copris_adam_cfg* cfg,
                                       copris_adam_host** out);
COPRIS_API int copris_adam_host_update(copris_adam_host* opt, double* params, const double* grad,
                                       int64_t n);
COPRIS_API int copris_adam_host_steps(const copris_adam_host* opt, int64_t* t);
COPRIS_API int copris_adam_host_destroy(copris_adam_host* opt);
COPRIS_API int copris_checkpoint_write(const char* path, const double* logits, const int32_t dims[4],
                                       uint64_t version, uint64_t seed);
/* Reads the header first: call with logits == NULL to get dims/version/seed,
 * then again with a buffer of Q*H*V doubles. */
COPRIS_API int copris_checkpoint_read(const char* path, double* logits, int32_t dims[4],
                                      uint64_t* version, uint64_t* seed);

/* ---- Host rollout buffer / scheduler (rollout.hpp:125-386) -----------------
 * The concurrency-controlled scheduler stays host-side bookkeeping
 * (include/copris_b200/rollout.hpp, bit-exact decisions); these entry points
 * expose it to non-C++ callers. `ids` outputs are caller buffers of `cap`
 * entries; `*n` receives the count (COPRIS_E_INVALID if cap is too small). */
typedef struct copris_engine copris_engine;

enum copris_sched_mode { COPRIS_SYNCHRONOUS = 0, COPRIS_NAIVE_PARTIAL = 1, COPRIS_COPRIS = 2 };
enum copris_engine_list {
  COPRIS_LIST_IN_FLIGHT = 0, COPRIS_LIST_RESUME_QUEUE = 1, COPRIS_LIST_BUFFERED = 2,
  COPRIS_LIST_CONSUMED = 3, COPRIS_LIST_EVICTED = 4
};

typedef struct {
  int32_t mode;                /* copris_sched_mode */
  int32_t concurrency, batch_prompts, rollouts_per_prompt, max_response_len, max_staleness;
  int32_t num_classes, horizon, vocab, answer_vocab;
  uint64_t seed;               /* question classes come from stream (seed, "prompt") */
} copris_engine_cfg;

/* A formed training batch in the packed layout (caller-owned host buffers,
 * sized from copris_engine_early_terminate's sizes[] = {groups, trajectories,
 * tokens, segments}). */
typedef struct {
  uint64_t rollout_version;    /* out */
  int64_t* group_off;          /* [groups+1] */
  uint64_t* group_ids;         /* [groups] */
  int32_t* group_class;        /* [groups] */
  uint64_t* traj_ids;          /* [traj] */
  int64_t* tok_off;            /* [traj+1] */
  int32_t* tokens;             /* [tokens] */
  int64_t* seg_off;            /* [segments+1] */
  uint32_t* seg_ver;           /* [segments] */
  float* buffered_lp;          /* [tokens] concat_segments */
  uint32_t* stage;             /* [tokens] */
  uint8_t* terminated;         /* [traj] */
  int32_t* answer_target;      /* [traj] */
} copris_packed_host;

COPRIS_API int copris_engine_create(const copris_engine_cfg* cfg, copris_engine** out);
COPRIS_API int copris_engine_destroy(copris_engine* e);
COPRIS_API int copris_engine_begin_stage(copris_engine* e, uint64_t version, uint64_t* ids,
                                         int64_t cap, int64_t* n);
COPRIS_API int copris_engine_refill_active(copris_engine* e, uint64_t* ids, int64_t cap, int64_t* n);
COPRIS_API int copris_engine_append_token(copris_engine* e, uint64_t id, int32_t token, double logprob,
                                          int32_t* terminated);
COPRIS_API int copris_engine_complete(copris_engine* e, uint64_t id, int32_t* batch_ready);
COPRIS_API int copris_engine_early_terminate(copris_engine* e, int64_t sizes[4]);
COPRIS_API int copris_engine_batch_copy(const copris_engine* e, copris_packed_host* out);
COPRIS_API int copris_engine_list(const copris_engine* e, int32_t which, uint64_t* ids, int64_t cap,
                                  int64_t* n);
/* out[7] = {in_flight, buffered partials, buffered completes, total admitted,
 *           stage version, batch ready, stage tokens in buffer} */
COPRIS_API int copris_engine_stats(const copris_engine* e, int64_t out[7]);

/* Introspection (not a reference entry point): cluster size, grid and kernel
 * name of the last copris_is_loss_* launch on this context. */
COPRIS_API int copris_ctx_last_launch(const copris_ctx* ctx, int* cluster, int* grid, int* num_sms,
                           const char** kernel_name);

/* Introspection: 1 when the last copris_is_loss_fused launch on this context
 * also reduced into copris_loss_out.out4 (no separate reduction launch). */
COPRIS_API int copris_ctx_last_fused_reduce(const copris_ctx* ctx);

/* Diagnostics (not a reference entry point): per-CTA phase-cycle counters of
 * the fused kernels, recorded when the context's `trace` option is on
 * (COPRIS_TRACE in the environment at creation); 10 int64 per CTA (pass B, barrier A, scalar phase,
 * barrier B, pass C, rows). Reading resets them. */
COPRIS_API int copris_ctx_trace_read(copris_ctx* ctx, long long* host, int n);

#ifdef __cplusplus
}
#endif
#endif /* COPRIS_B200_H */
