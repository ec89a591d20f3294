// ref_harness.cpp — TEST INFRASTRUCTURE ONLY.
//
// A C-ABI shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/copris, compiled read-only by oracle/Makefile
// into oracle/_ref/libcopris_ref.so). It lets the tests and bench.py's
// reference arm run the reference's own hot path — sequence_logprobs
// (policy.hpp:160-173), concat_segments (trajectory.hpp:69-75),
// compute_advantages (grpo.hpp:51-65) and grpo_step_loss (grpo.hpp:117-185) —
// on a packed row-per-token batch:
//
//   PolicyShape{num_classes = n_traj, horizon = Lmax, vocab = V}
//   row (class i, position t) := logits row of packed token tok_off[i] + t
//
// so every token owns exactly one table row and the table gradient row (i, t)
// is the token's dlogits row. Nothing here re-implements reference math.
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "copris/grpo.hpp"
#include "copris/io.hpp"
#include "copris/policy.hpp"
#include "copris/trajectory.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const copris::ContractViolation& e) {
    g_err = e.what();
    return 1;
  } catch (const copris::ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

struct Packed {
  copris::PolicyParams params;
  std::vector<copris::Trajectory> trajs;
};

// Builds the one-row-per-token table and the stage-tagged trajectories.
Packed build(const double* logits, int64_t ld, int32_t vocab, int64_t n_traj,
             const int64_t* tok_off, const int32_t* target, const uint32_t* stage,
             const double* buffered_lp) {
  int64_t lmax = 1;
  for (int64_t i = 0; i < n_traj; ++i) lmax = std::max<int64_t>(lmax, tok_off[i + 1] - tok_off[i]);
  copris::PolicyShape shape;
  shape.num_classes = static_cast<int>(std::max<int64_t>(1, n_traj));
  shape.horizon = static_cast<int>(lmax);
  shape.vocab = vocab;
  shape.answer_vocab = 1;
  Packed p{copris::PolicyParams(shape), {}};
  p.trajs.resize(n_traj);
  for (int64_t i = 0; i < n_traj; ++i) {
    copris::Trajectory& t = p.trajs[i];
    t.traj_id = static_cast<uint64_t>(i);
    t.question = copris::Question::from_class(static_cast<int>(i), shape);
    for (int64_t j = tok_off[i]; j < tok_off[i + 1]; ++j) {
      int pos = static_cast<int>(j - tok_off[i]);
      auto row = p.params.row_mut(static_cast<int>(i), pos);
      for (int32_t k = 0; k < vocab; ++k) row[k] = logits[j * ld + k];
      t.tokens.tokens.push_back(target[j]);
      uint64_t ver = stage ? stage[j] : 0;
      if (t.segments.empty() || t.segments.back().policy_version != ver)
        t.segments.push_back(copris::LogProbSegment{ver, {}});
      t.segments.back().logprobs.push_back(buffered_lp ? buffered_lp[j] : 0.0);
    }
    t.tokens.terminated = true;
  }
  return p;
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

int ref_logprob_gather(const double* logits, int64_t ld, const int32_t* target, int64_t n_tok,
                       int32_t vocab, double* out_lp) {
  return guarded([&] {
    int64_t off[2] = {0, n_tok};
    Packed p = build(logits, ld, vocab, 1, off, target, nullptr, nullptr);
    auto lp = copris::sequence_logprobs(p.params, p.trajs[0].question, p.trajs[0].tokens);
    std::memcpy(out_lp, lp.data(), sizeof(double) * lp.size());
  });
}

int ref_advantages(const double* rewards, const int64_t* group_off, int64_t n_groups,
                   double adv_epsilon, double* out_adv) {
  return guarded([&] {
    for (int64_t g = 0; g < n_groups; ++g) {
      std::span<const double> r(rewards + group_off[g],
                                static_cast<size_t>(group_off[g + 1] - group_off[g]));
      auto adv = copris::compute_advantages(r, adv_epsilon);
      std::memcpy(out_adv + group_off[g], adv.data(), sizeof(double) * adv.size());
    }
  });
}

int ref_terminal_rewards(const int32_t* tokens, const int64_t* tok_off, int64_t n_traj,
                         const uint8_t* terminated, const int32_t* answer_target,
                         int32_t eos_token, double* out_reward) {
  return guarded([&] {
    for (int64_t i = 0; i < n_traj; ++i) {
      copris::Trajectory t;
      t.tokens.tokens.assign(tokens + tok_off[i], tokens + tok_off[i + 1]);
      t.tokens.terminated = terminated[i] != 0;
      copris::Question q{0, answer_target[i]};
      out_reward[i] = copris::terminal_reward(t, q, eos_token);
    }
  });
}

// The reference's loss path over a packed batch. When current_from_recompute
// is set, the log-probs of current-stage tokens (stage == cur_stage) are taken
// from sequence_logprobs, which is what the reference's sampler records for
// them (bitwise: test_policy.cpp:157-172). `seconds` receives the time spent
// inside the reference functions (table construction excluded).
int ref_is_loss(const double* logits, int64_t ld, int32_t vocab, int64_t n_traj,
                const int64_t* tok_off, const int32_t* target, const uint32_t* stage,
                uint32_t cur_stage, const double* buffered_lp, const double* ref_logits,
                const double* adv, double clip_low, double clip_high, double kl_coeff,
                double entropy_coeff, int is_enabled, int current_from_recompute,
                double* out_loss, double* out_dlogits, double* out_cur_lp, double* out_stored_lp,
                double* seconds) {
  return guarded([&] {
    const int64_t n_tok = tok_off[n_traj];
    std::vector<double> blp(buffered_lp, buffered_lp + n_tok);
    Packed p = build(logits, ld, vocab, n_traj, tok_off, target, stage, blp.data());
    Packed ref;
    if (kl_coeff > 0.0) ref = build(ref_logits, ld, vocab, n_traj, tok_off, target, stage, blp.data());
    copris::ClipConfig cfg;
    cfg.clip_low = clip_low;
    cfg.clip_high = clip_high;
    cfg.kl_coeff = kl_coeff;
    cfg.entropy_coeff = entropy_coeff;

    double t0 = now_s();
    std::vector<copris::GrpoItem> items;
    items.reserve(n_traj);
    for (int64_t i = 0; i < n_traj; ++i) {
      copris::Trajectory& tr = p.trajs[i];
      copris::GrpoItem item;
      item.traj = &tr;
      item.advantage = adv[i];
      item.current_lp = copris::sequence_logprobs(p.params, tr.question, tr.tokens);
      if (current_from_recompute) {
        size_t t = 0;
        for (auto& seg : tr.segments)
          for (double& lp : seg.logprobs) {
            if (seg.policy_version == cur_stage) lp = item.current_lp[t];
            ++t;
          }
      }
      item.stored_lp = is_enabled ? copris::concat_segments(tr) : item.current_lp;
      if (kl_coeff > 0.0)
        item.ref_lp = copris::sequence_logprobs(ref.params, tr.question, tr.tokens);
      items.push_back(std::move(item));
    }
    copris::GrpoStepResult res = copris::grpo_step_loss(p.params, items, cfg);
    double t1 = now_s();
    if (seconds) *seconds = t1 - t0;

    *out_loss = res.loss;
    for (int64_t i = 0; i < n_traj; ++i) {
      for (int64_t j = tok_off[i]; j < tok_off[i + 1]; ++j) {
        int pos = static_cast<int>(j - tok_off[i]);
        if (out_dlogits)
          std::memcpy(out_dlogits + j * vocab,
                      res.grad.data() + p.params.shape.row_offset(static_cast<int>(i), pos),
                      sizeof(double) * vocab);
        if (out_cur_lp) out_cur_lp[j] = items[i].current_lp[pos];
        if (out_stored_lp) out_stored_lp[j] = items[i].stored_lp[pos];
      }
    }
  });
}

// AdamOptimizer (grpo.hpp:203-233): `k` updates with grads[k][n] on a table of
// n = Q*H*V parameters.
int ref_adam(const int32_t dims[4], double* params, const double* grads, int k, double lr,
             double b1, double b2, double eps, double wd) {
  return guarded([&] {
    copris::PolicyParams p(copris::PolicyShape{dims[0], dims[1], dims[2], dims[3]});
    const size_t n = p.logits.size();
    std::memcpy(p.logits.data(), params, n * sizeof(double));
    copris::AdamOptimizer opt(copris::AdamConfig{lr, b1, b2, eps, wd});
    for (int i = 0; i < k; ++i)
      opt.update(p, std::span<const double>(grads + static_cast<size_t>(i) * n, n));
    std::memcpy(params, p.logits.data(), n * sizeof(double));
  });
}

// io.hpp:397-438
int ref_write_checkpoint(const char* path, const int32_t dims[4], const double* logits,
                         uint64_t version, uint64_t seed) {
  return guarded([&] {
    copris::PolicyParams p(copris::PolicyShape{dims[0], dims[1], dims[2], dims[3]});
    std::memcpy(p.logits.data(), logits, p.logits.size() * sizeof(double));
    p.version = version;
    copris::write_checkpoint(path, p, seed);
  });
}

int ref_read_checkpoint(const char* path, int32_t dims[4], double* logits, uint64_t* version,
                        uint64_t* seed) {
  return guarded([&] {
    copris::PolicyParams p = copris::read_checkpoint(path, seed);
    dims[0] = p.shape.num_classes;
    dims[1] = p.shape.horizon;
    dims[2] = p.shape.vocab;
    dims[3] = p.shape.answer_vocab;
    if (logits) std::memcpy(logits, p.logits.data(), p.logits.size() * sizeof(double));
    *version = p.version;
  });
}

}  // extern "C"
