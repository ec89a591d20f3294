// gen_golden.cpp — TEST INFRASTRUCTURE ONLY.
//
// Runs the UNMODIFIED reference Trainer (trainer.hpp:120-181) at desk scale
// (BASELINE config #1) and captures, through its observation seam
// Trainer::set_inspector (trainer.hpp:117-118,174), the exact inputs the
// reference hands to grpo_step_loss plus what grpo_step_loss returns for them.
// Output: one JSON document per case on stdout-selected paths, written to
// tests/golden/ by tests/golden/make_golden.sh. Doubles are printed with 17
// significant digits so they round-trip exactly.
#include <cstdio>
#include <string>
#include <vector>

#include "copris/trainer.hpp"

using namespace copris;

namespace {

// io.hpp:445-457 desk_default_config(), restated so this generator does not
// need nlohmann/json.
RunConfig desk_config() {
  RunConfig cfg;
  cfg.mode = SchedulingMode::Copris;
  cfg.is_enabled = true;
  cfg.engine = EngineConfig{16, 4, 4, 8, 0};
  cfg.policy = PolicyShape{4, 8, 6, 4};
  cfg.cluster = ClusterConfig{4, 1.0, 0.05, 64, 8};
  cfg.length_model = LengthModel{LengthMode::PolicyDriven, 0.0, 0.0};
  cfg.total_steps = 200;
  cfg.seed = 1;
  cfg.eval_every = 0;
  return cfg;
}

struct Out {
  FILE* f;
  bool first = true;
  void sep() {
    if (!first) std::fputc(',', f);
    first = false;
  }
};

void put_d(FILE* f, double v) { std::fprintf(f, "%.17g", v); }

void put_vec(FILE* f, const std::vector<double>& v) {
  std::fputc('[', f);
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) std::fputc(',', f);
    put_d(f, v[i]);
  }
  std::fputc(']', f);
}

void put_ivec(FILE* f, const std::vector<int>& v) {
  std::fputc('[', f);
  for (size_t i = 0; i < v.size(); ++i) std::fprintf(f, i ? ",%d" : "%d", v[i]);
  std::fputc(']', f);
}

struct Case {
  std::string name;
  RunConfig cfg;
  int steps;
  std::vector<int> capture;
};

void run_case(const Case& c, const std::string& dir) {
  std::string path = dir + "/trainer_" + c.name + ".json";
  FILE* f = std::fopen(path.c_str(), "w");
  if (!f) throw std::runtime_error("cannot open " + path);
  Trainer trainer(c.cfg);
  PolicyParams reference = trainer.params();  // version-0 snapshot (trainer.hpp:100)
  const PolicyShape& sh = c.cfg.policy;
  std::fprintf(f, "{\"case\":\"%s\",\"seed\":%llu,", c.name.c_str(),
               (unsigned long long)c.cfg.seed);
  std::fprintf(f,
               "\"policy\":{\"num_classes\":%d,\"horizon\":%d,\"vocab\":%d,\"answer_vocab\":%d},",
               sh.num_classes, sh.horizon, sh.vocab, sh.answer_vocab);
  std::fprintf(f, "\"engine\":{\"concurrency\":%d,\"batch_prompts\":%d,\"rollouts_per_prompt\":%d},",
               c.cfg.engine.concurrency, c.cfg.engine.batch_prompts,
               c.cfg.engine.rollouts_per_prompt);
  std::fprintf(f, "\"clip\":{\"clip_low\":");
  put_d(f, c.cfg.clip.clip_low);
  std::fprintf(f, ",\"clip_high\":");
  put_d(f, c.cfg.clip.clip_high);
  std::fprintf(f, ",\"kl_coeff\":");
  put_d(f, c.cfg.clip.kl_coeff);
  std::fprintf(f, ",\"entropy_coeff\":");
  put_d(f, c.cfg.clip.entropy_coeff);
  std::fprintf(f, ",\"adv_epsilon\":");
  put_d(f, c.cfg.clip.adv_epsilon);
  std::fprintf(f, "},\"is_enabled\":%s,", c.cfg.is_enabled ? "true" : "false");
  std::fprintf(f, "\"reference_params\":");
  put_vec(f, reference.logits);
  std::fprintf(f, ",\"steps\":[");
  Out steps{f};
  int step = 0;
  trainer.set_inspector([&](const TrainBatch& batch, const std::vector<GrpoItem>& items) {
    bool want = false;
    for (int s : c.capture) want |= (s == step);
    if (!want) return;
    steps.sep();
    const PolicyParams& params = trainer.params();
    GrpoStepResult res = grpo_step_loss(params, items, c.cfg.clip);
    std::fprintf(f, "{\"step\":%d,\"rollout_version\":%llu,\"params_version\":%llu,", step,
                 (unsigned long long)batch.rollout_version, (unsigned long long)params.version);
    std::fprintf(f, "\"offpolicy_fraction\":");
    put_d(f, offpolicy_token_fraction(batch, batch.rollout_version));
    std::fprintf(f, ",\"params\":");
    put_vec(f, params.logits);
    std::fprintf(f, ",\"groups\":[");
    size_t idx = 0;
    for (size_t gi = 0; gi < batch.groups.size(); ++gi) {
      const auto& g = batch.groups[gi];
      if (gi) std::fputc(',', f);
      std::fprintf(f, "{\"group_id\":%llu,\"class_id\":%d,\"target_token\":%d,\"members\":[",
                   (unsigned long long)g.group_id, g.question.class_id, g.question.target_token);
      for (size_t mi = 0; mi < g.members.size(); ++mi, ++idx) {
        const Trajectory& t = g.members[mi];
        const GrpoItem& it = items[idx];
        if (mi) std::fputc(',', f);
        std::fprintf(f, "{\"traj_id\":%llu,\"terminated\":%s,\"tokens\":",
                     (unsigned long long)t.traj_id, t.tokens.terminated ? "true" : "false");
        put_ivec(f, t.tokens.tokens);
        std::fprintf(f, ",\"segments\":[");
        for (size_t si = 0; si < t.segments.size(); ++si) {
          if (si) std::fputc(',', f);
          std::fprintf(f, "{\"version\":%llu,\"logprobs\":",
                       (unsigned long long)t.segments[si].policy_version);
          put_vec(f, t.segments[si].logprobs);
          std::fputc('}', f);
        }
        std::fprintf(f, "],\"advantage\":");
        put_d(f, it.advantage);
        std::fprintf(f, ",\"reward\":");
        put_d(f, terminal_reward(t, g.question, sh.eos_token()));
        std::fprintf(f, ",\"current_lp\":");
        put_vec(f, it.current_lp);
        std::fprintf(f, ",\"stored_lp\":");
        put_vec(f, it.stored_lp);
        std::fprintf(f, ",\"ref_lp\":");
        put_vec(f, it.ref_lp);
        std::fputc('}', f);
      }
      std::fprintf(f, "]}");
    }
    std::fprintf(f, "],\"loss\":");
    put_d(f, res.loss);
    std::fprintf(f, ",\"token_count\":%zu,\"grad\":", res.token_count);
    put_vec(f, res.grad);
    std::fputc('}', f);
  });
  for (step = 0; step < c.steps; ++step) trainer.train_step();
  std::fprintf(f, "]}\n");
  std::fclose(f);
  std::printf("wrote %s\n", path.c_str());
}

}  // namespace

int main(int argc, char** argv) {
  std::string dir = argc > 1 ? argv[1] : ".";
  std::vector<Case> cases;
  {
    Case c{"desk", desk_config(), 6, {0, 1, 2, 3, 4, 5}};
    cases.push_back(c);
  }
  {  // BASELINE config #1: 16 prompts x 4 responses, buffered multi-stage
    RunConfig cfg = desk_config();
    cfg.engine.batch_prompts = 16;
    cfg.engine.concurrency = 48;
    cases.push_back({"b16_c48", cfg, 20, {5, 12, 19}});
    cfg.engine.concurrency = 128;
    cases.push_back({"b16_c128", cfg, 20, {10, 19}});
  }
  {
    RunConfig cfg = desk_config();
    cfg.engine.batch_prompts = 16;
    cfg.engine.concurrency = 48;
    cfg.is_enabled = false;
    cases.push_back({"b16_c48_is_off", cfg, 8, {7}});
  }
  {
    RunConfig cfg = desk_config();
    cfg.engine.batch_prompts = 16;
    cfg.engine.concurrency = 48;
    cfg.clip.kl_coeff = 0.1;
    cfg.clip.entropy_coeff = 0.01;
    cases.push_back({"b16_c48_kl_entropy", cfg, 8, {3, 7}});
  }
  {  // long-tail lengths, more stages per trajectory
    RunConfig cfg = desk_config();
    cfg.engine.batch_prompts = 16;
    cfg.engine.concurrency = 128;
    cfg.engine.max_response_len = 64;
    cfg.policy.horizon = 64;
    cfg.cluster.memory_capacity = 4096;
    cfg.length_model = LengthModel{LengthMode::Lognormal, 3.0, 1.0};
    cases.push_back({"lognormal_h64_c128", cfg, 12, {11}});
  }
  for (const auto& c : cases) run_case(c, dir);
  return 0;
}
