// engine_check.cpp — TEST INFRASTRUCTURE (built into oracle/_ref/ from the
// reference headers; runs on CPU).
//
// Drives the UNMODIFIED reference RolloutEngine (rollout.hpp:125-386) and
// copris_b200::RolloutEngine (include/copris_b200/rollout.hpp) with the same
// event stream — stage starts, token appends under random interleavings,
// completions, refills, early terminations, staleness eviction, misuse that
// must throw — and compares every decision and query after every event.
// It also records the reference's stream as JSON lines (argv[1]) so the
// C-ABI engine can be replayed against it without the reference present.
// Exit code 0 iff every decision matched.
#include <cstdio>
#include <string>
#include <vector>

#include "copris/rollout.hpp"
#include "copris_b200/rollout.hpp"

namespace ref = copris;
namespace mine = copris_b200;

namespace {

int g_fail = 0;
long g_checks = 0;
FILE* g_rec = nullptr;

void fail(const std::string& what) {
  if (g_fail < 20) std::fprintf(stderr, "MISMATCH: %s\n", what.c_str());
  ++g_fail;
}

template <class A, class B>
void same(const A& a, const B& b, const std::string& what) {
  ++g_checks;
  if (!(a == b)) fail(what);
}

std::string ids_json(const std::vector<uint64_t>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
  return s + "]";
}

void compare_traj(const ref::Trajectory& a, const mine::Trajectory& b, const std::string& w) {
  same(a.traj_id, b.traj_id, w + " id");
  same(a.group_id, b.group_id, w + " group");
  same(a.question.class_id, b.question.class_id, w + " class");
  same(a.tokens.tokens, b.tokens, w + " tokens");
  same(a.tokens.terminated, b.terminated, w + " terminated");
  same(static_cast<int>(a.status), static_cast<int>(b.status), w + " status");
  same(a.created_version, b.created_version, w + " created_version");
  same(a.segments.size(), b.segments.size(), w + " segments");
  for (size_t i = 0; i < a.segments.size() && i < b.segments.size(); ++i) {
    same(a.segments[i].policy_version, b.segments[i].policy_version, w + " seg version");
    same(a.segments[i].logprobs, b.segments[i].logprobs, w + " seg logprobs");
  }
}

void compare_state(const ref::RolloutEngine& a, const mine::RolloutEngine& b, const std::string& w) {
  std::vector<uint64_t> ai(a.in_flight_ids().begin(), a.in_flight_ids().end());
  std::vector<uint64_t> bi(b.in_flight_ids().begin(), b.in_flight_ids().end());
  same(ai, bi, w + " in_flight_ids");
  same(a.buffered_ids(), b.buffered_ids(), w + " buffered_ids");
  same(a.buffered_partial_count(), b.buffered_partial_count(), w + " partial count");
  same(a.buffered_complete_count(), b.buffered_complete_count(), w + " complete count");
  same(a.total_admitted(), b.total_admitted(), w + " total_admitted");
  same(a.consumed_ids(), b.consumed_ids(), w + " consumed");
  same(a.evicted_ids(), b.evicted_ids(), w + " evicted");
  same(a.stage_version(), b.stage_version(), w + " stage_version");
  same(a.batch_ready(), b.batch_ready(), w + " batch_ready");
  same(a.stage_tokens_in_buffer(a.stage_version()), b.stage_tokens_in_buffer(b.stage_version()),
       w + " stage tokens in buffer");
  for (uint64_t id : a.buffered_ids()) compare_traj(a.trajectory(id), b.trajectory(id), w + " traj");
}

template <class F, class G>
void same_throw(F fa, G fb, const std::string& w) {
  std::string ea = "none", eb = "none";
  try { fa(); } catch (const ref::ContractViolation& e) { ea = std::string("C:") + e.what(); }
  catch (const ref::ConfigError& e) { ea = std::string("F:") + e.what(); }
  try { fb(); } catch (const mine::ContractViolation& e) { eb = std::string("C:") + e.what(); }
  catch (const mine::ConfigError& e) { eb = std::string("F:") + e.what(); }
  same(ea, eb, w + " exception (" + ea + " vs " + eb + ")");
}

struct Scenario {
  const char* name;
  ref::SchedulingMode mode;
  int concurrency, batch_prompts, rollouts, horizon, staleness, vocab, stages;
  double eos_prob;
  uint64_t seed;
};

void run(const Scenario& sc) {
  ref::EngineConfig rc{sc.concurrency, sc.batch_prompts, sc.rollouts, sc.horizon, sc.staleness};
  mine::EngineConfig mc{sc.concurrency, sc.batch_prompts, sc.rollouts, sc.horizon, sc.staleness};
  ref::PolicyShape rs{4, sc.horizon, sc.vocab, 4};
  mine::PolicyShape ms{4, sc.horizon, sc.vocab, 4};
  ref::RolloutEngine a(rc, sc.mode, rs, ref::RngStream(sc.seed, "prompt"));
  mine::RolloutEngine b(mc, static_cast<mine::SchedulingMode>(sc.mode), ms,
                        mine::NamedStream(sc.seed, "prompt"));
  ref::RngStream drive(sc.seed, "driver");
  if (g_rec)
    std::fprintf(g_rec,
                 "{\"op\":\"create\",\"scenario\":\"%s\",\"mode\":%d,\"concurrency\":%d,\"batch_prompts\":%d,"
                 "\"rollouts\":%d,\"horizon\":%d,\"staleness\":%d,\"vocab\":%d,\"seed\":%llu}\n",
                 sc.name, static_cast<int>(sc.mode), sc.concurrency, sc.batch_prompts, sc.rollouts,
                 sc.horizon, sc.staleness, sc.vocab, (unsigned long long)sc.seed);
  const std::string w0 = sc.name;
  for (int stage = 0; stage < sc.stages; ++stage) {
    const uint64_t v = static_cast<uint64_t>(stage);
    auto ra = a.begin_stage(v);
    auto rb = b.begin_stage(v);
    same(ra, rb, w0 + " begin_stage admitted");
    if (g_rec) std::fprintf(g_rec, "{\"op\":\"begin_stage\",\"version\":%llu,\"admitted\":%s}\n",
                            (unsigned long long)v, ids_json(ra).c_str());
    compare_state(a, b, w0 + " after begin_stage");
    // misuse: a second begin_stage while trajectories are in flight
    same_throw([&] { a.begin_stage(v); }, [&] { b.begin_stage(v); }, w0 + " begin_stage twice");
    bool halted = false;
    int guard = 0;
    while (!halted && ++guard < 100000) {
      std::vector<uint64_t> act(a.in_flight_ids().begin(), a.in_flight_ids().end());
      if (act.empty()) break;
      const uint64_t id = act[drive.uniform_int(act.size())];
      const int pos = static_cast<int>(a.trajectory(id).tokens.size());
      int tok = static_cast<int>(drive.uniform_int(sc.vocab - 1));
      if (drive.uniform() < sc.eos_prob) tok = sc.vocab - 1;
      const double lp = -drive.uniform(0.0, 5.0);
      a.append_token(id, tok, lp);
      b.append_token(id, tok, lp);
      if (g_rec) std::fprintf(g_rec, "{\"op\":\"append\",\"id\":%llu,\"token\":%d,\"logprob\":%.17g}\n",
                              (unsigned long long)id, tok, lp);
      (void)pos;
      if (a.trajectory(id).tokens.terminated) {
        same_throw([&] { a.append_token(id, 0, -1.0); }, [&] { b.append_token(id, 0, -1.0); },
                   w0 + " append after termination");
        const bool fa = a.complete_trajectory(id);
        const bool fb = b.complete_trajectory(id);
        same(fa, fb, w0 + " complete -> batch_ready");
        if (g_rec) std::fprintf(g_rec, "{\"op\":\"complete\",\"id\":%llu,\"ready\":%s}\n",
                                (unsigned long long)id, fa ? "true" : "false");
        same_throw([&] { a.complete_trajectory(id); }, [&] { b.complete_trajectory(id); },
                   w0 + " double completion");
        if (fa) {
          ref::TrainBatch ba = a.early_terminate();
          mine::TrainBatch bb = b.early_terminate();
          same(ba.rollout_version, bb.rollout_version, w0 + " batch version");
          same(ba.groups.size(), bb.groups.size(), w0 + " batch groups");
          std::string gj = "[";
          for (size_t gi = 0; gi < ba.groups.size() && gi < bb.groups.size(); ++gi) {
            same(ba.groups[gi].group_id, bb.groups[gi].group_id, w0 + " batch group id");
            same(ba.groups[gi].question.class_id, bb.groups[gi].question.class_id, w0 + " group class");
            same(ba.groups[gi].members.size(), bb.groups[gi].members.size(), w0 + " group size");
            std::vector<uint64_t> mids;
            for (size_t mi = 0; mi < ba.groups[gi].members.size() && mi < bb.groups[gi].members.size(); ++mi) {
              compare_traj(ba.groups[gi].members[mi], bb.groups[gi].members[mi], w0 + " batch member");
              mids.push_back(ba.groups[gi].members[mi].traj_id);
            }
            gj += (gi ? "," : "") + std::string("{\"group\":") + std::to_string(ba.groups[gi].group_id) +
                  ",\"class\":" + std::to_string(ba.groups[gi].question.class_id) + ",\"members\":" +
                  ids_json(mids) + "}";
          }
          gj += "]";
          same(ref::offpolicy_token_fraction(ba, ba.rollout_version),
               mine::offpolicy_token_fraction(bb, bb.rollout_version), w0 + " offpolicy fraction");
          std::vector<uint64_t> resume(b.resume_queue().begin(), b.resume_queue().end());
          if (g_rec)
            std::fprintf(g_rec, "{\"op\":\"early_terminate\",\"version\":%llu,\"groups\":%s,\"resume\":%s}\n",
                         (unsigned long long)ba.rollout_version, gj.c_str(), ids_json(resume).c_str());
          halted = true;
        } else {
          auto fa2 = a.refill_active();
          auto fb2 = b.refill_active();
          same(fa2, fb2, w0 + " refill admitted");
          if (g_rec) std::fprintf(g_rec, "{\"op\":\"refill\",\"admitted\":%s}\n", ids_json(fa2).c_str());
        }
      }
      compare_state(a, b, w0 + " after event");
    }
    if (!halted) fail(w0 + " stage did not halt");
    same_throw([&] { a.early_terminate(); }, [&] { b.early_terminate(); }, w0 + " early_terminate twice");
  }
  if (g_rec) std::fprintf(g_rec, "{\"op\":\"end\",\"evicted\":%s,\"consumed\":%zu}\n",
                          ids_json(a.evicted_ids()).c_str(), a.consumed_ids().size());
}

}  // namespace

int main(int argc, char** argv) {
  if (argc > 1) g_rec = std::fopen(argv[1], "w");
  using M = ref::SchedulingMode;
  const Scenario scenarios[] = {
      {"copris_desk", M::Copris, 16, 4, 4, 8, 0, 6, 12, 0.25, 1},
      {"copris_b16_c48", M::Copris, 48, 16, 4, 8, 0, 6, 10, 0.2, 2},
      {"copris_c128_staleness1", M::Copris, 128, 16, 4, 8, 1, 6, 10, 0.15, 3},
      {"copris_c64_staleness2_h16", M::Copris, 64, 8, 8, 16, 2, 32, 10, 0.1, 4},
      {"naive_partial", M::NaivePartial, 24, 4, 4, 8, 0, 6, 10, 0.25, 5},
      {"naive_partial_staleness1", M::NaivePartial, 40, 4, 8, 12, 1, 16, 10, 0.15, 6},
      {"synchronous", M::Synchronous, 16, 4, 4, 8, 0, 6, 10, 0.25, 7},
      {"copris_g2", M::Copris, 20, 5, 2, 6, 0, 8, 12, 0.3, 8},
  };
  for (const auto& sc : scenarios) run(sc);
  // constructor validation errors
  same_throw([] { ref::RolloutEngine x(ref::EngineConfig{8, 4, 4, 8, 0}, M::NaivePartial, ref::PolicyShape{},
                                       ref::RngStream(1, "prompt")); },
             [] { mine::RolloutEngine x(mine::EngineConfig{8, 4, 4, 8, 0}, mine::SchedulingMode::NaivePartial,
                                        mine::PolicyShape{}, mine::NamedStream(1, "prompt")); },
             "naive dispatch validation");
  same_throw([] { ref::RolloutEngine x(ref::EngineConfig{0, 4, 4, 8, 0}, M::Copris, ref::PolicyShape{},
                                       ref::RngStream(1, "prompt")); },
             [] { mine::RolloutEngine x(mine::EngineConfig{0, 4, 4, 8, 0}, mine::SchedulingMode::Copris,
                                        mine::PolicyShape{}, mine::NamedStream(1, "prompt")); },
             "concurrency validation");
  if (g_rec) std::fclose(g_rec);
  std::printf("{\"checks\":%ld,\"mismatches\":%d}\n", g_checks, g_fail);
  return g_fail ? 1 : 0;
}
