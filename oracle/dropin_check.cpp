// dropin_check.cpp — TEST INFRASTRUCTURE (built into oracle/_ref/, needs the
// reference headers at build time; runs on the GPU box).
//
// Runs the UNMODIFIED reference Trainer and, at its observation seam
// (Trainer::set_inspector, trainer.hpp:117-118,174) — i.e. with exactly the
// arguments trainer.hpp:176 passes to grpo_step_loss — computes the step both
// with the reference's grpo_step_loss and with copris_b200::DropIn (the GPU
// path behind the C-ABI). Prints one JSON line per captured step and exits
// nonzero if the loss or the table gradient differ beyond 1e-5 (relative).
#include <cmath>
#include <cstdio>
#include <span>
#include <vector>

#include "copris/trainer.hpp"
#include "copris_b200/grpo_dropin.hpp"

using namespace copris;

namespace {

RunConfig desk_config() {  // io.hpp:445-457
  RunConfig cfg;
  cfg.mode = SchedulingMode::Copris;
  cfg.engine = EngineConfig{16, 4, 4, 8, 0};
  cfg.policy = PolicyShape{4, 8, 6, 4};
  cfg.cluster = ClusterConfig{4, 1.0, 0.05, 64, 8};
  cfg.length_model = LengthModel{LengthMode::PolicyDriven, 0.0, 0.0};
  cfg.seed = 1;
  cfg.eval_every = 0;
  return cfg;
}

}  // namespace

int main() {
  copris_b200::DropIn gpu(0);
  struct Case {
    const char* name;
    RunConfig cfg;
    int steps;
  };
  std::vector<Case> cases;
  cases.push_back({"desk", desk_config(), 6});
  {
    RunConfig c = desk_config();
    c.engine.batch_prompts = 16;
    c.engine.concurrency = 48;
    cases.push_back({"b16_c48", c, 12});
    c.is_enabled = false;
    cases.push_back({"b16_c48_is_off", c, 6});
    c.is_enabled = true;
    c.clip.kl_coeff = 0.1;
    c.clip.entropy_coeff = 0.01;
    cases.push_back({"b16_c48_kl_entropy", c, 6});
  }
  {  // wider vocabulary and horizon, heavy buffering (4-5 stages per trajectory)
    RunConfig c = desk_config();
    c.engine.batch_prompts = 16;
    c.engine.concurrency = 128;
    c.engine.max_response_len = 16;
    c.policy = PolicyShape{4, 16, 64, 4};
    c.cluster.memory_capacity = 4096;
    cases.push_back({"v64_h16_c128", c, 8});
  }
  int bad = 0;
  for (auto& cs : cases) {
    Trainer trainer(cs.cfg);
    int step = 0;
    trainer.set_inspector([&](const TrainBatch& batch, const std::vector<GrpoItem>& items) {
      const PolicyParams& params = trainer.params();
      GrpoStepResult ref = grpo_step_loss(params, items, cs.cfg.clip);
      GrpoStepResult got = gpu.grpo_step_loss<GrpoStepResult, ContractViolation, ConfigError>(
          params, std::span<const GrpoItem>(items), cs.cfg.clip);
      double gmax = 0.0, gerr = 0.0;
      for (size_t i = 0; i < ref.grad.size(); ++i) {
        gmax = std::max(gmax, std::abs(ref.grad[i]));
        gerr = std::max(gerr, std::abs(ref.grad[i] - got.grad[i]));
      }
      const double lerr = std::abs(ref.loss - got.loss);
      const bool ok = got.token_count == ref.token_count && lerr <= 1e-5 * std::max(1e-3, std::abs(ref.loss)) &&
                      gerr <= 1e-5 * gmax;
      bad += !ok;
      std::printf(
          "{\"case\":\"%s\",\"step\":%d,\"tokens\":%zu,\"rollout_version\":%llu,\"loss_ref\":%.17g,"
          "\"loss_gpu\":%.17g,\"loss_abs_err\":%.3g,\"grad_max\":%.6g,\"grad_abs_err\":%.3g,\"ok\":%s}\n",
          cs.name, step, ref.token_count, (unsigned long long)batch.rollout_version, ref.loss, got.loss,
          lerr, gmax, gerr, ok ? "true" : "false");
    });
    for (step = 0; step < cs.steps; ++step) trainer.train_step();
  }
  return bad ? 1 : 0;
}
