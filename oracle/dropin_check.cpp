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
#include <cstring>
#include <mutex>
#include <span>
#include <thread>
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

struct Case {
  const char* name;
  RunConfig cfg;
  int steps;
};

struct StepOut {
  double loss_gpu;
  bool ok;
};

// One case: the reference Trainer with its own DropIn context; prints one JSON
// line per captured step (under `io`) and returns the GPU losses in step order.
std::vector<StepOut> run_case(const Case& cs, const char* mode, std::mutex& io) {
  copris_b200::DropIn gpu(0);
  std::vector<StepOut> outs;
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
    outs.push_back({got.loss, ok});
    std::lock_guard<std::mutex> lock(io);
    std::printf(
        "{\"mode\":\"%s\",\"case\":\"%s\",\"step\":%d,\"tokens\":%zu,\"rollout_version\":%llu,"
        "\"loss_ref\":%.17g,\"loss_gpu\":%.17g,\"loss_abs_err\":%.3g,\"grad_max\":%.6g,"
        "\"grad_abs_err\":%.3g,\"ok\":%s}\n",
        mode, cs.name, step, ref.token_count, (unsigned long long)batch.rollout_version, ref.loss,
        got.loss, lerr, gmax, gerr, ok ? "true" : "false");
  });
  for (step = 0; step < cs.steps; ++step) trainer.train_step();
  return outs;
}

}  // namespace

// usage: dropin_check [--threads]   (--threads: after the sequential pass, every
// case again on its own std::thread with its own context, as the reference CLI
// runs one Trainer per thread (copris_cli.cpp:98-115); the GPU losses must be
// bitwise the sequential ones)
int main(int argc, char** argv) {
  const bool threaded = argc > 1 && std::strcmp(argv[1], "--threads") == 0;
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
  std::mutex io;
  int bad = 0;
  std::vector<std::vector<StepOut>> seq;
  for (auto& cs : cases) {
    seq.push_back(run_case(cs, "sequential", io));
    for (auto& o : seq.back()) bad += !o.ok;
  }
  if (threaded) {
    std::vector<std::vector<StepOut>> par(cases.size());
    std::vector<std::thread> ts;
    for (size_t i = 0; i < cases.size(); ++i)
      ts.emplace_back([&, i] { par[i] = run_case(cases[i], "threaded", io); });
    for (auto& t : ts) t.join();
    for (size_t i = 0; i < cases.size(); ++i) {
      bool same = par[i].size() == seq[i].size();
      for (size_t k = 0; same && k < par[i].size(); ++k)
        same = std::memcmp(&par[i][k].loss_gpu, &seq[i][k].loss_gpu, sizeof(double)) == 0 &&
               par[i][k].ok;
      bad += !same;
      std::printf("{\"mode\":\"threaded_vs_sequential\",\"case\":\"%s\",\"steps\":%zu,\"ok\":%s}\n",
                  cases[i].name, par[i].size(), same ? "true" : "false");
    }
  }
  return bad ? 1 : 0;
}
