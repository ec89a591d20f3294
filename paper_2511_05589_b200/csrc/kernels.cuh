// kernels.cuh — device-side parameter blocks and host launchers for the
// sm_100a kernels of the IS-corrected loss path. Launchers return a
// cudaError_t; argument validation and error mapping live in capi.cu.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace copris_b200 {

// Allow `bytes` of dynamic shared memory for `func` on the current device. The
// attribute is per function and device — shared by every context and thread of
// the process — so it is raised once, to the device's opt-in maximum, and never
// lowered: concurrent launches of the same kernel with different sizes on other
// threads cannot see a smaller limit (re-entrancy).
cudaError_t allow_dyn_smem(const void* func, int bytes);

// Bits of the device error word (copris_ctx_check maps them to the
// reference's exception messages).
enum : uint32_t {
  ERR_TOKEN_OOV = 1u,        // policy.hpp:169 "token out of vocabulary"
  ERR_NONFINITE_LP = 2u,     // grpo.hpp:69-70 "token_ratio requires finite log-probs"
  ERR_NONFINITE_ADV = 4u,    // grpo.hpp:128 "advantage must be finite"
  ERR_NOT_TERMINATED = 8u,   // grpo.hpp:36 "terminal_reward requires a terminated trajectory"
  ERR_EMPTY_TERMINATED = 16u,  // grpo.hpp:38 "terminated trajectory cannot be empty"
};

// Everything one loss launch needs, by value (kernel parameter space).
struct LossParams {
  // batch
  const void* logits;
  int64_t ld;
  int32_t vocab;
  int32_t cur_stage;
  int64_t n_rows;
  int64_t row_base;
  const int32_t* target;
  const uint32_t* stage;
  const float* buffered_lp;
  const float* ref_lp;
  const int32_t* tok_traj;
  const double* adv;
  const uint8_t* loss_mask;  // optional: 0 = token left out of the loss
  // unfused-K3 inputs (nullptr in the fused kernel)
  const float* in_cur_lp;
  const float* in_lse;
  const float* in_behav;
  // cfg (grpo.hpp:15-28, 135)
  double clamp_lo;   // 1 - clip_low
  double clamp_hi;   // 1 + clip_high
  double kl_coeff;
  double entropy_coeff;
  double inv_t;      // 1 / T_global
  int32_t is_enabled;
  int32_t behav_mode;
  // out
  void* dlogits;
  int64_t ld_d;
  float* cur_lp;
  float* lse;
  float* behav;
  double* obj;
  double* coef;
  uint8_t* flags;
  uint32_t* err;
  long long* trace;  // optional per-CTA phase-cycle accumulators (COPRIS_TRACE)
  unsigned long long* row_ctr;  // dynamic row claims: 0 at launch; the last CTA rearms it (reduce.cuh)
  int32_t gather_only;  // K1 mode: only (cur_lp, lse) per row — no metadata, no objective
  // optional fused reduction: the launch also reduces rows [0, red_n) of
  // obj/flags into out4 (the last CTA to finish does it; kernels that do not
  // support it leave out4 to a separate reduce launch, see launch_fused)
  double* out4;
  void* red_scratch;
  int64_t red_n;
};

// Phase accumulators written by the fused kernels when LossParams::trace is
// set: [cta * kTraceSlots + k], k = pass B, wait A, scalar, wait B, pass C, rows,
// ring waits (2), lifetime ns, lifetime cycles (the pair family: slots 6/7 =
// start globaltimer ns and SM id instead of the ring waits).
constexpr int kTraceSlots = 10;
constexpr int kTraceCtas = 2048;

enum class DType : int { BF16 = 0, F32 = 1 };

// Kernel selection and tunables of one context. Filled once from the COPRIS_*
// environment at copris_ctx_create (tuning_from_env) and changed only through
// copris_ctx_set_option; launchers read this copy and never the environment,
// so a setenv on one thread cannot change another context's kernels mid-run
// (re-entrancy).
struct Tuning {
  int fused_impl = 0;     // 0 auto, 1 stream (TMA ring + L2 re-read), 2 tma (row in smem), 3 pair, 4 solo
  int lookahead = 2;      // stream kernel: ring segments of row r+1 before pass 2 of row r
  int slots = 0;          // stream kernel ring slots (0 = as many 32 KB slots as fit 192 KB)
  int resident = 1;       // stream kernel: pass 2 from resident segments when 3 rows fit
  int pair_lookahead = 3; // pair kernel: slots of row r+1 through pass 1 before pass 2 of row r
  int pair_st256 = 0;     // pair kernel, bf16 dlogits: 32-byte stores (lane-pair swap) in pass 2
  int pair_bf16_stage = 1; // pair kernel, bf16 dlogits: bf16 (not f16) exponentials in TMEM, bf16x2 pass 2
  int pair_pw8 = 1;       // pair kernel: 8-warp CTAs, two per SM, when the half row fits (V <= 114,688)
  int pair_dynamic = 1;   // pair kernels: rows after the first claimed from the context's counter
  int lmhead_impl = 0;    // 0 CTA pair (cta_group::2), 1 single SM
  int lmhead_group = 16;  // LM-head raster group (token pairs per vocab sweep)
  int lmhead_tma_store = 1;
  int gemm_wide = 1;      // dhidden GEMM: 256 x 512 tiles per pair
  int gemm_mc = 0;        // dhidden GEMM: 4-CTA clusters with W^T multicast
  int gemm_splits = 0;    // 0 = automatic split-K count
  int gemm_a_evict_first = 0;
  int dw_group = 1;
  int dw_policy = 2;
  int64_t dw_kchunk = 8192;
  int trace = 0;          // per-CTA phase tracing (COPRIS_TRACE)
};

Tuning tuning_from_env();
// Sets one option by name; returns false for an unknown name or bad value.
bool tuning_set(Tuning& t, const char* name, int64_t value);
bool tuning_get(const Tuning& t, const char* name, int64_t* value);

struct LaunchInfo {
  int num_sms;
  int cluster;       // CTAs per row chosen by the dispatcher (fused TMA path)
  int grid;          // CTAs launched
  const char* kernel;
  int reduced;       // 1: the loss launch itself reduced into out4 (no second launch)
};

// Fused single-pass loss. Chooses the TMA/cluster kernel when rows are 16-byte
// aligned, otherwise the generic kernel.
cudaError_t launch_fused(const LossParams& p, DType in, DType out, int num_sms,
                         const Tuning& tu, cudaStream_t stream, LaunchInfo* info);
// Unfused K3 (second logits pass from lse).
cudaError_t launch_bwd(const LossParams& p, DType in, DType out, int num_sms,
                       cudaStream_t stream, LaunchInfo* info);
// K1.
cudaError_t launch_logprob_gather(const void* logits, int64_t ld, DType in, const int32_t* target,
                                  int64_t n_tok, int32_t vocab, float* out_lp, float* out_lse,
                                  uint32_t* err, unsigned long long* row_ctr, void* red_scratch,
                                  int num_sms, const Tuning& tu, cudaStream_t stream);
// K2.
cudaError_t launch_expand_segments(const int64_t* seg_off, const uint32_t* seg_ver, int64_t n_seg,
                                   uint32_t* out_stage, cudaStream_t stream);
cudaError_t launch_behaviour(const uint32_t* stage, uint32_t cur_stage, const float* blp,
                             const float* cur_lp, int is_enabled, int behav_mode, int64_t n_tok,
                             float* out_behav, uint8_t* out_flags, cudaStream_t stream);
// K3a and helpers.
cudaError_t launch_terminal_rewards(const int32_t* tokens, const int64_t* tok_off, int64_t n_traj,
                                    const uint8_t* terminated, const int32_t* answer_target,
                                    int32_t eos, double* out, uint32_t* err, cudaStream_t stream);
cudaError_t launch_group_advantages(const double* rewards, const int64_t* group_off,
                                    int64_t n_groups, double eps, double* out_adv,
                                    cudaStream_t stream);
cudaError_t launch_token_traj(const int64_t* tok_off, int64_t n_traj, int32_t* out,
                              cudaStream_t stream);
cudaError_t launch_adam(double* p, const double* g, double* m, double* v, int64_t n, double lr,
                        double b1, double b2, double eps, double wd, double bc1, double bc2,
                        int num_sms, cudaStream_t stream);
// Deterministic reduction; scratch holds >= reduce_scratch_bytes() bytes.
size_t reduce_scratch_bytes();
cudaError_t launch_reduce(const double* obj, const uint8_t* flags, int64_t n_tok, double* out4,
                          void* scratch, int num_sms, cudaStream_t stream);

}  // namespace copris_b200
