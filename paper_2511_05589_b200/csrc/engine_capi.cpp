// engine_capi.cpp — C-ABI over the host rollout scheduler
// (include/copris_b200/rollout.hpp). Host-only bookkeeping: no device work.
#include <algorithm>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "../../include/copris_b200.h"
#include "../../include/copris_b200/rollout.hpp"
#include "internal.hpp"

using namespace copris_b200;

struct copris_engine {
  RolloutEngine engine;
  PackedBatch last;
  bool have_batch = false;
  int64_t admit_bound = 0;  // max ids one begin_stage / refill_active can admit
};

namespace {

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const ContractViolation& e) {
    return fail(COPRIS_E_CONTRACT, e.what());
  } catch (const ConfigError& e) {
    return fail(COPRIS_E_CONFIG, e.what());
  } catch (const std::exception& e) {
    return fail(COPRIS_E_INVALID, e.what());
  }
}

int put_ids(const std::vector<uint64_t>& v, uint64_t* ids, int64_t cap, int64_t* n) {
  if (n) *n = static_cast<int64_t>(v.size());
  if (static_cast<int64_t>(v.size()) > cap || (!ids && !v.empty()))
    return fail(COPRIS_E_INVALID, "id buffer capacity too small");
  if (!v.empty()) std::memcpy(ids, v.data(), v.size() * sizeof(uint64_t));
  return COPRIS_OK;
}

}  // namespace

extern "C" {

int copris_engine_create(const copris_engine_cfg* c, copris_engine** out) {
  if (!c || !out) return fail(COPRIS_E_INVALID, "null argument");
  *out = nullptr;
  if (c->mode < 0 || c->mode > 2) return fail(COPRIS_E_CONFIG, "unknown scheduling mode");
  return guarded([&] {
    EngineConfig ec{c->concurrency, c->batch_prompts, c->rollouts_per_prompt, c->max_response_len,
                    c->max_staleness};
    PolicyShape ps{c->num_classes, c->horizon, c->vocab, c->answer_vocab};
    // fill_to(target) admits at most `target` trajectories, target being the
    // concurrency (copris / naive) or B*N (synchronous), rollout.hpp:181-191
    const int64_t bound = std::max<int64_t>(c->concurrency,
                                            static_cast<int64_t>(c->batch_prompts) * c->rollouts_per_prompt);
    *out = new copris_engine{RolloutEngine(ec, static_cast<SchedulingMode>(c->mode), ps,
                                           NamedStream(c->seed, "prompt")),
                             {}, false, bound};
    return COPRIS_OK;
  });
}

int copris_engine_destroy(copris_engine* e) {
  delete e;
  return COPRIS_OK;
}

// The id buffer is checked against the admission bound BEFORE the engine
// admits anything: a too-small buffer leaves the engine state untouched.
static int check_cap(const copris_engine* e, const uint64_t* ids, int64_t cap) {
  if (!ids || cap < e->admit_bound)
    return fail(COPRIS_E_INVALID, "id buffer capacity too small (need max(concurrency, B*N))");
  return COPRIS_OK;
}

int copris_engine_begin_stage(copris_engine* e, uint64_t version, uint64_t* ids, int64_t cap,
                              int64_t* n) {
  if (!e) return fail(COPRIS_E_INVALID, "null engine");
  if (int rc = check_cap(e, ids, cap)) return rc;
  return guarded([&] { return put_ids(e->engine.begin_stage(version), ids, cap, n); });
}

int copris_engine_refill_active(copris_engine* e, uint64_t* ids, int64_t cap, int64_t* n) {
  if (!e) return fail(COPRIS_E_INVALID, "null engine");
  if (int rc = check_cap(e, ids, cap)) return rc;
  return guarded([&] { return put_ids(e->engine.refill_active(), ids, cap, n); });
}

int copris_engine_append_token(copris_engine* e, uint64_t id, int32_t token, double logprob,
                               int32_t* terminated) {
  if (!e) return fail(COPRIS_E_INVALID, "null engine");
  return guarded([&] {
    e->engine.append_token(id, token, logprob);
    if (terminated) *terminated = e->engine.trajectory(id).terminated ? 1 : 0;
    return COPRIS_OK;
  });
}

int copris_engine_complete(copris_engine* e, uint64_t id, int32_t* batch_ready) {
  if (!e) return fail(COPRIS_E_INVALID, "null engine");
  return guarded([&] {
    const bool r = e->engine.complete_trajectory(id);
    if (batch_ready) *batch_ready = r ? 1 : 0;
    return COPRIS_OK;
  });
}

int copris_engine_early_terminate(copris_engine* e, int64_t sizes[4]) {
  if (!e) return fail(COPRIS_E_INVALID, "null engine");
  return guarded([&] {
    e->last = pack(e->engine.early_terminate());
    e->have_batch = true;
    if (sizes) {
      sizes[0] = e->last.n_groups();
      sizes[1] = e->last.n_traj();
      sizes[2] = e->last.n_tok();
      sizes[3] = static_cast<int64_t>(e->last.seg_ver.size());
    }
    return COPRIS_OK;
  });
}

int copris_engine_batch_copy(const copris_engine* e, copris_packed_host* o) {
  if (!e || !o) return fail(COPRIS_E_INVALID, "null argument");
  if (!e->have_batch) return fail(COPRIS_E_CONTRACT, "no batch formed yet");
  const PackedBatch& p = e->last;
  auto cp = [](auto* dst, const auto& src) {
    if (dst && !src.empty()) std::memcpy(dst, src.data(), src.size() * sizeof(src[0]));
  };
  o->rollout_version = p.rollout_version;
  cp(o->group_off, p.group_off);
  cp(o->group_ids, p.group_ids);
  cp(o->group_class, p.group_class);
  cp(o->traj_ids, p.traj_ids);
  cp(o->tok_off, p.tok_off);
  cp(o->tokens, p.target);
  cp(o->seg_off, p.seg_off);
  cp(o->seg_ver, p.seg_ver);
  cp(o->buffered_lp, p.buffered_lp);
  cp(o->stage, p.stage);
  cp(o->terminated, p.terminated);
  cp(o->answer_target, p.answer_target);
  return COPRIS_OK;
}

int copris_engine_list(const copris_engine* e, int32_t which, uint64_t* ids, int64_t cap, int64_t* n) {
  if (!e) return fail(COPRIS_E_INVALID, "null engine");
  const RolloutEngine& g = e->engine;
  switch (which) {
    case COPRIS_LIST_IN_FLIGHT:
      return put_ids(std::vector<uint64_t>(g.in_flight_ids().begin(), g.in_flight_ids().end()), ids, cap, n);
    case COPRIS_LIST_RESUME_QUEUE:
      return put_ids(std::vector<uint64_t>(g.resume_queue().begin(), g.resume_queue().end()), ids, cap, n);
    case COPRIS_LIST_BUFFERED:
      return put_ids(g.buffered_ids(), ids, cap, n);
    case COPRIS_LIST_CONSUMED:
      return put_ids(g.consumed_ids(), ids, cap, n);
    case COPRIS_LIST_EVICTED:
      return put_ids(g.evicted_ids(), ids, cap, n);
    default:
      return fail(COPRIS_E_INVALID, "unknown list");
  }
}

int copris_engine_stats(const copris_engine* e, int64_t out[7]) {
  if (!e || !out) return fail(COPRIS_E_INVALID, "null argument");
  const RolloutEngine& g = e->engine;
  out[0] = static_cast<int64_t>(g.in_flight_count());
  out[1] = static_cast<int64_t>(g.buffered_partial_count());
  out[2] = static_cast<int64_t>(g.buffered_complete_count());
  out[3] = static_cast<int64_t>(g.total_admitted());
  out[4] = static_cast<int64_t>(g.stage_version());
  out[5] = g.batch_ready() ? 1 : 0;
  out[6] = static_cast<int64_t>(g.stage_tokens_in_buffer(g.stage_version()));
  return COPRIS_OK;
}

}  // extern "C"
