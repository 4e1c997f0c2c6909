// ssdlab_b200.hpp — header-only C++ shim over the C-ABI (ssd_b200.h) that
// re-exports the reference's speculator / verifier / speculation-cache
// interfaces (ssd-lab, proj/include/ssdlab/{specdec,cache,sim,categorical,
// errors}.hpp) with the model parameter widened to a B200-resident
// transformer pair (SURVEY.md §8b "Model parameter").
//
// Mapping (reference -> this shim):
//   ssdlab::Error and subclasses (errors.hpp:9-61)  -> ssdlab_b200::Error ... (same names, thrown from ssd_status)
//   dist::SamplingScheme (categorical.hpp:43-60)    -> ssdlab_b200::SamplingScheme
//   cache::FanOutPlan (cache.hpp:18-25)             -> ssdlab_b200::FanOutPlan
//   cache::geometric_fanout / uniform_fanout        -> same names (cache.hpp:57-64)
//   rng::Stream (rng.hpp:29-48)                     -> ssdlab_b200::Stream (same next_u64 / next_uniform)
//   specdec::draft (specdec.hpp:59-61)              -> Engine::draft(ctx, K, scheme, Stream&)
//   specdec::verify (specdec.hpp:81-83)             -> Engine::verify(ctx, spec, Stream&, VerifyOptions)
//   cache::build_cache (cache.hpp:149-154)          -> Engine::build_cache(ctx, spec, plan, scheme, next_K, Stream&)
//   SpeculationCache::lookup (cache.hpp:123-126)    -> SpeculationCache::lookup (non-owning pointer or nullptr)
//   sim::run_ar / run_sd                            -> Engine::run_ar / run_sd
//   sim::run_ssd / run_ssd_batch                    -> Engine::run_ssd_sequential
//   sim::run_protocol_harness (+ Transcript)        -> Engine::run_ssd (+ transcript_jsonl)
//   lm::SyntheticLM::logits_at (lm.cpp:82-84)       -> Engine::logits
//   (device side)                       -> Engine::prespec_begin / cache_lookup / cache_keys / cache_entry
//
// Differences the caller must know: distributions stay on the device — a
// Speculation carries its tokens and the fp32 draft LOGIT rows [K][V] they
// were drawn from (its dists = the scheme applied to those rows; empty rows
// = the uniform dists of the FastRandom backup). Seed-taking overloads
// (draft / build_cache / verify_rows with a uint64 seed) start a fresh
// Stream(seed).
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ssd_b200.h"

namespace ssdlab_b200 {

// ------------------------------------------------------------ errors.hpp:9-61
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
#define SSDLAB_B200_ERR(name) \
  struct name : Error {       \
    using Error::Error;       \
  };
SSDLAB_B200_ERR(AllZeroError)
SSDLAB_B200_ERR(DegenerateResidualError)
SSDLAB_B200_ERR(TooLargeError)
SSDLAB_B200_ERR(BudgetTooSmallError)
SSDLAB_B200_ERR(DivergentError)
SSDLAB_B200_ERR(InsufficientDataError)
SSDLAB_B200_ERR(UnreachableError)
SSDLAB_B200_ERR(NoCrossoverError)
SSDLAB_B200_ERR(ProtocolViolationError)
SSDLAB_B200_ERR(ConfigError)
SSDLAB_B200_ERR(CudaError)
#undef SSDLAB_B200_ERR

// Re-throw an ssd_status as the reference exception class it stands for.
inline void check(ssd_status s) {
  if (s == SSD_OK) return;
  const std::string m = ssd_last_error();
  switch (s) {
    case SSD_ALL_ZERO: throw AllZeroError(m);
    case SSD_DEGENERATE_RESIDUAL: throw DegenerateResidualError(m);
    case SSD_TOO_LARGE: throw TooLargeError(m);
    case SSD_BUDGET_TOO_SMALL: throw BudgetTooSmallError(m);
    case SSD_DIVERGENT: throw DivergentError(m);
    case SSD_INSUFFICIENT_DATA: throw InsufficientDataError(m);
    case SSD_UNREACHABLE: throw UnreachableError(m);
    case SSD_NO_CROSSOVER: throw NoCrossoverError(m);
    case SSD_PROTOCOL_VIOLATION: throw ProtocolViolationError(m);
    case SSD_CONFIG: throw ConfigError(m);
    case SSD_CUDA: throw CudaError(m);
    default: throw Error(m);
  }
}

// ------------------------------------------------------- categorical.hpp:43-60
struct SamplingScheme {
  enum class Kind { Standard, Saguaro } kind = Kind::Standard;
  double temperature = 1.0;  // 0 = greedy (the tau -> 0 limit)
  int fan_out = 0;
  double downweight = 1.0;
  static SamplingScheme standard(double t = 1.0) { return {Kind::Standard, t, 0, 1.0}; }
  static SamplingScheme greedy() { return {Kind::Standard, 0.0, 0, 1.0}; }
  static SamplingScheme saguaro(int f, double c, double t = 1.0) { return {Kind::Saguaro, t, f, c}; }
  ssd_scheme c() const { return ssd_scheme{kind == Kind::Saguaro ? 1 : 0, fan_out, temperature, downweight}; }
};

enum class Origin { Primary = 0, Backup = 1 };       // specdec.hpp:14-20
enum class BackupKind { SamePrimaryJIT = 0, FastRandom = 1 };  // sim.hpp:17-20

// ----------------------------------------------------------- cache.hpp:18-68
struct FanOutPlan {
  std::vector<int> fan_out;
  Origin role = Origin::Primary;
  int budget = 0;
  int lookahead() const { return int(fan_out.size()) - 1; }
  int total() const {
    int t = 0;
    for (int f : fan_out) t += f;
    return t;
  }
  ssd_plan c() const {
    if (fan_out.empty() || fan_out.size() > SSD_MAX_LOOKAHEAD + 1) throw TooLargeError("plan: lookahead out of range");
    ssd_plan p{};
    p.lookahead = lookahead();
    p.role = int(role);
    p.budget = budget ? budget : total();
    for (size_t k = 0; k < fan_out.size(); ++k) p.fan_out[k] = fan_out[k];
    return p;
  }
  static FanOutPlan from_c(const ssd_plan& p) {
    FanOutPlan f;
    f.fan_out.assign(p.fan_out, p.fan_out + p.lookahead + 1);
    f.role = Origin(p.role);
    f.budget = p.budget;
    return f;
  }
};

inline FanOutPlan geometric_fanout(double acceptance, double exponent, int lookahead, int budget,
                                   Origin role = Origin::Primary) {
  ssd_plan p{};
  check(ssd_geometric_fanout(acceptance, exponent, lookahead, budget, int(role), &p));
  return FanOutPlan::from_c(p);
}
inline FanOutPlan uniform_fanout(int lookahead, int budget, Origin role = Origin::Primary) {
  ssd_plan p{};
  check(ssd_uniform_fanout(lookahead, budget, int(role), &p));
  return FanOutPlan::from_c(p);
}

// ------------------------------------------------- hitmodel.hpp:39-53, perf.hpp:54-72
struct PowerLawFit {
  double exponent = 0.0, log_amplitude = 0.0, r_squared = 1.0;
};
inline PowerLawFit fit_powerlaw(std::span<const std::pair<double, double>> samples) {
  std::vector<double> f, m;
  for (const auto& [a, b] : samples) { f.push_back(a); m.push_back(b); }
  PowerLawFit out;
  check(ssd_fit_powerlaw(f.data(), m.data(), int(f.size()), &out.exponent, &out.log_amplitude, &out.r_squared));
  return out;
}
inline double speedup_batch(double hit_rate, double hit_tokens, double miss_tokens, double primary_time,
                            double backup_time, double batch) {
  double out = 0.0;
  check(ssd_speedup_batch(hit_rate, hit_tokens, miss_tokens, primary_time, backup_time, batch, &out));
  return out;
}
inline double critical_batch(double hit_rate, double hit_tokens, double miss_tokens, double primary_time) {
  double out = 0.0;
  check(ssd_critical_batch(hit_rate, hit_tokens, miss_tokens, primary_time, &out));
  return out;
}

// ---------------------------------------------------------------- rng.hpp:29-48
class Stream {
 public:
  explicit Stream(std::uint64_t seed) { ssd_rng_stream_seed(&s_, seed); }
  std::uint64_t next_u64() { return ssd_rng_stream_next_u64(&s_); }
  double next_uniform() { return ssd_rng_stream_next_uniform(&s_); }
  ssd_rng_stream* c() { return &s_; }

 private:
  ssd_rng_stream s_{};
};
inline std::uint64_t derive_seed(std::uint64_t root, std::uint64_t index) { return ssd_derive_seed(root, index); }

// ---------------------------------------------------------- specdec.hpp:22-52
struct Speculation {
  std::vector<int> tokens;
  std::vector<float> rows;  // [K][V] fp32 draft logits (empty unless requested)
  Origin origin = Origin::Primary;
};
struct VerificationOutcome {
  int accepted = 0;
  int bonus = 0;
  bool operator==(const VerificationOutcome& o) const { return accepted == o.accepted && bonus == o.bonus; }
  bool operator<(const VerificationOutcome& o) const {
    return accepted != o.accepted ? accepted < o.accepted : bonus < o.bonus;
  }
};
struct RoundResult {  // specdec.hpp:44-52
  VerificationOutcome outcome;
  std::vector<int> emitted;
};
struct VerifyOptions {  // specdec.hpp:63-79
  SamplingScheme target_scheme = SamplingScheme::standard();
  double accept_scale = 1.0;
};

// cache.hpp:114-135: immutable after build; lookup returns a non-owning
// pointer valid while the cache lives.
class SpeculationCache {
 public:
  const Speculation* lookup(const VerificationOutcome& key) const {
    auto it = entries_.find(key);
    return it == entries_.end() ? nullptr : &it->second;
  }
  size_t size() const { return entries_.size(); }
  const std::map<VerificationOutcome, Speculation>& entries() const { return entries_; }
  Origin role = Origin::Primary;

 private:
  friend class Engine;
  std::map<VerificationOutcome, Speculation> entries_;
};

// --------------------------------------------------------------- sim.hpp:28-104
struct SimConfig {
  int lookahead = 4;
  SamplingScheme scheme = SamplingScheme::standard();
  SamplingScheme target_scheme = SamplingScheme::standard();
  FanOutPlan primary_plan, backup_plan;
  BackupKind backup = BackupKind::FastRandom;
  double primary_time = 0.3, backup_time = 0.0;
  long rounds = 1000;
  std::uint64_t seed = 0;
  double accept_scale = 1.0;
  int batch_size = 1;  // sim.hpp:40 (run_ssd only: whole-batch stall semantics)
  ssd_sim_config c() const {
    ssd_sim_config s{};
    s.lookahead = lookahead;
    s.scheme = scheme.c();
    s.target_scheme = target_scheme.c();
    s.primary_plan = primary_plan.c();
    s.backup_plan = backup_plan.c();
    s.backup_kind = int(backup);
    s.primary_time = primary_time;
    s.backup_time = backup_time;
    s.rounds = rounds;
    s.seed = seed;
    s.accept_scale = accept_scale;
    return s;
  }
};

struct RunResult {
  ssd_run_stats stats{};
  std::vector<int> tokens;                     // sequence 0
  std::vector<std::vector<int>> streams;       // run_ssd: one per batch sequence
  std::vector<VerificationOutcome> outcomes;  // run_ssd only
  std::vector<int> hits;                      // run_ssd only (-1 on the last round)
  std::string transcript_jsonl;               // run_ssd(..., with_transcript): Transcript::to_jsonl (sim.cpp:489-500)
  double hit_rate() const {
    const long l = stats.primary_origin_lookups + stats.backup_origin_lookups;
    return l ? double(stats.primary_origin_hits + stats.backup_origin_hits) / double(l) : 0.0;
  }
};

// ------------------------------------------------------------------- engine
class Engine {
 public:
  Engine(const ssd_model_shape& target, const ssd_model_shape& draft, const ssd_pair_params& pair, int device = 0,
         int max_branches = 64, int max_lookahead = 8, int max_batch = 1) {
    ssd_engine* e = nullptr;
    if (max_batch > 1)
      check(ssd_engine_create_batch(&target, &draft, &pair, device, max_batch, max_branches, max_lookahead, &e));
    else
      check(ssd_engine_create(&target, &draft, &pair, device, max_branches, max_lookahead, &e));
    h_.reset(e);
    vocab_ = target.vocab;
  }
  int vocab() const { return vocab_; }
  ssd_engine* handle() const { return h_.get(); }

  // lm::SyntheticLM::logits_at (lm.cpp:82-84); which: 0 target, 1 draft
  std::vector<float> logits(int which, std::span<const int> ctx) const {
    std::vector<float> out(static_cast<size_t>(vocab_));
    check(ssd_logits(h_.get(), which, ctx.data(), int(ctx.size()), out.data()));
    return out;
  }

  // specdec::draft (specdec.cpp:8-25) with Stream(seed)
  Speculation draft(std::span<const int> ctx, int lookahead, const SamplingScheme& scheme, std::uint64_t seed,
                    bool with_rows = false, Origin origin = Origin::Primary) const {
    Speculation s;
    s.tokens.resize(size_t(lookahead));
    if (with_rows) s.rows.resize(size_t(lookahead) * size_t(vocab_));
    const ssd_scheme sc = scheme.c();
    check(ssd_draft(h_.get(), ctx.data(), int(ctx.size()), lookahead, &sc, seed, s.tokens.data(),
                    with_rows ? s.rows.data() : nullptr));
    s.origin = origin;
    return s;
  }

  // specdec::draft (specdec.hpp:59-61) drawing from the caller's Stream
  Speculation draft(std::span<const int> ctx, int lookahead, const SamplingScheme& scheme, Stream& rng,
                    Origin origin = Origin::Primary) const {
    Speculation s;
    s.tokens.resize(size_t(lookahead));
    s.rows.resize(size_t(lookahead) * size_t(vocab_));
    const ssd_scheme sc = scheme.c();
    check(ssd_draft_stream(h_.get(), ctx.data(), int(ctx.size()), lookahead, &sc, rng.c(), s.tokens.data(),
                           s.rows.data()));
    s.origin = origin;
    return s;
  }

  // specdec::verify (specdec.hpp:81-83): the target's verify forward over
  // ctx || spec plus the fused decision, coins and bonus from `rng`;
  // draft_scheme is the law spec.rows were drawn under
  RoundResult verify(std::span<const int> ctx, const Speculation& spec, Stream& rng,
                     const SamplingScheme& draft_scheme, const VerifyOptions& opt = {}) const {
    const int K = int(spec.tokens.size());
    if (!spec.rows.empty() && spec.rows.size() != size_t(K) * size_t(vocab_))
      throw Error("verify: speculation rows must be [K][V]");
    const ssd_scheme ds = draft_scheme.c(), ts = opt.target_scheme.c();
    RoundResult r;
    r.emitted.resize(size_t(K + 1));
    check(ssd_verify(h_.get(), ctx.data(), int(ctx.size()), spec.tokens.data(), K,
                     spec.rows.empty() ? nullptr : spec.rows.data(), &ds, &ts, opt.accept_scale, rng.c(),
                     &r.outcome.accepted, &r.outcome.bonus, r.emitted.data()));
    r.emitted.resize(size_t(r.outcome.accepted + 1));
    return r;
  }

  // cache::build_cache (cache.hpp:149-154): one next_u64 from `rng`, entries
  // of next_lookahead tokens with the draft rows they were drawn from
  SpeculationCache build_cache(std::span<const int> ctx, const Speculation& spec, const FanOutPlan& plan,
                               const SamplingScheme& scheme, int next_lookahead, Stream& rng) const {
    if (plan.role != spec.origin) throw Error("build_cache: plan role does not match speculation origin");
    const ssd_plan p = plan.c();
    const ssd_scheme sc = scheme.c();
    const int tot = std::max(1, plan.total());
    std::vector<int> keys(size_t(2 * tot)), toks(size_t(tot) * size_t(next_lookahead));
    std::vector<float> rows(size_t(tot) * size_t(next_lookahead) * size_t(vocab_));
    int count = 0;
    check(ssd_build_cache_stream(h_.get(), ctx.data(), int(ctx.size()), spec.tokens.data(), int(spec.tokens.size()),
                                 &p, &sc, next_lookahead, rng.c(), keys.data(), toks.data(), rows.data(), &count));
    SpeculationCache c;
    c.role = plan.role;
    const size_t per = size_t(next_lookahead) * size_t(vocab_);
    for (int i = 0; i < count; ++i) {
      Speculation e;
      e.tokens.assign(toks.begin() + i * next_lookahead, toks.begin() + (i + 1) * next_lookahead);
      e.rows.assign(rows.begin() + long(i * per), rows.begin() + long((i + 1) * per));
      e.origin = Origin::Primary;
      c.entries_.emplace(VerificationOutcome{keys[size_t(2 * i)], keys[size_t(2 * i + 1)]}, std::move(e));
    }
    return c;
  }

  // Asynchronous pre-speculation of DEVICE buffers ordered after
  // `cuda_stream`; lookups wait for it
  void prespec_begin(const int32_t* d_ctx, int n, const int32_t* d_spec, int lookahead, const FanOutPlan& plan,
                     const SamplingScheme& scheme, int next_lookahead, Stream& rng, void* cuda_stream = nullptr) {
    const ssd_plan p = plan.c();
    const ssd_scheme sc = scheme.c();
    check(ssd_prespec_begin(h_.get(), d_ctx, n, d_spec, lookahead, &p, &sc, next_lookahead, rng.c(), cuda_stream));
  }
  int cache_lookup(const VerificationOutcome& key) const {
    int slot = -1;
    check(ssd_cache_lookup(h_.get(), key.accepted, key.bonus, &slot));
    return slot;
  }
  std::vector<VerificationOutcome> cache_keys() const {
    int n = 0;
    check(ssd_cache_keys(h_.get(), nullptr, &n));
    std::vector<int> k(size_t(2 * std::max(n, 1)));
    check(ssd_cache_keys(h_.get(), k.data(), &n));
    std::vector<VerificationOutcome> out;
    for (int i = 0; i < n; ++i) out.push_back({k[size_t(2 * i)], k[size_t(2 * i + 1)]});
    return out;
  }
  Speculation cache_entry(int slot, int next_lookahead) const {
    Speculation e;
    e.tokens.resize(size_t(next_lookahead));
    e.rows.resize(size_t(next_lookahead) * size_t(vocab_));
    check(ssd_cache_entry(h_.get(), slot, e.tokens.data(), e.rows.data()));
    return e;
  }

  // specdec::verify decision (specdec.cpp:27-69) on target rows [K+1][V] and
  // the speculation's draft rows [K][V] (empty = uniform, the FastRandom backup)
  VerificationOutcome verify_rows(std::span<const float> target_rows, const Speculation& spec,
                                  const SamplingScheme& draft_scheme, const SamplingScheme& target_scheme,
                                  std::uint64_t seed, double accept_scale = 1.0) const {
    const int K = int(spec.tokens.size());
    if (target_rows.size() != size_t(K + 1) * size_t(vocab_)) throw Error("verify: target rows must be [K+1][V]");
    const ssd_scheme ds = draft_scheme.c(), ts = target_scheme.c();
    VerificationOutcome o;
    check(ssd_verify_rows(h_.get(), target_rows.data(), spec.rows.empty() ? nullptr : spec.rows.data(),
                          spec.tokens.data(), K, vocab_, &ds, &ts, accept_scale, seed, &o.accepted, &o.bonus));
    return o;
  }

  // cache::build_cache (cache.cpp:232-277); base_seed = the one draw the
  // reference takes from the caller's stream (cache.cpp:245)
  SpeculationCache build_cache(std::span<const int> ctx, const Speculation& spec, const FanOutPlan& plan,
                               const SamplingScheme& scheme, int next_lookahead, std::uint64_t base_seed) const {
    if (plan.role != spec.origin) throw Error("build_cache: plan role does not match speculation origin");
    const ssd_plan p = plan.c();
    const ssd_scheme sc = scheme.c();
    const int tot = std::max(1, plan.total());
    std::vector<int> keys(size_t(2 * tot)), toks(size_t(tot) * size_t(next_lookahead));
    int count = 0;
    check(ssd_build_cache(h_.get(), ctx.data(), int(ctx.size()), spec.tokens.data(), int(spec.tokens.size()), &p,
                          &sc, next_lookahead, base_seed, keys.data(), toks.data(), &count));
    SpeculationCache c;
    c.role = plan.role;
    for (int i = 0; i < count; ++i) {
      Speculation e;
      e.tokens.assign(toks.begin() + i * next_lookahead, toks.begin() + (i + 1) * next_lookahead);
      e.origin = Origin::Primary;
      c.entries_.emplace(VerificationOutcome{keys[size_t(2 * i)], keys[size_t(2 * i + 1)]}, std::move(e));
    }
    return c;
  }

  RunResult run_ar(std::span<const int> prompt, const SamplingScheme& target_scheme, long tokens,
                   std::uint64_t seed) const {
    RunResult r;
    r.tokens.resize(size_t(tokens));
    const ssd_scheme ts = target_scheme.c();
    check(ssd_run_ar(h_.get(), prompt.data(), int(prompt.size()), &ts, tokens, seed, r.tokens.data(), tokens,
                     &r.stats));
    return r;
  }

  RunResult run_sd(std::span<const int> prompt, const SimConfig& cfg) const {
    RunResult r;
    const long cap = cfg.rounds * (cfg.lookahead + 1);
    r.tokens.resize(size_t(cap));
    const ssd_sim_config c = cfg.c();
    int64_t n = 0;
    check(ssd_run_sd(h_.get(), prompt.data(), int(prompt.size()), &c, r.tokens.data(), cap, &n, &r.stats));
    r.tokens.resize(size_t(n));
    return r;
  }

  // sim::run_protocol_harness (sim.cpp:502-601), cfg.batch_size sequences;
  // with_transcript: the JSONL round transcript (sim.cpp:489-500)
  RunResult run_ssd(std::span<const int> prompt, const SimConfig& cfg, bool with_transcript = false) const {
    return run(prompt, cfg, SSD_SEMANTICS_HARNESS, with_transcript);
  }
  // sim::run_ssd / run_ssd_batch (sim.cpp:123-250)
  RunResult run_ssd_sequential(std::span<const int> prompt, const SimConfig& cfg) const {
    return run(prompt, cfg, SSD_SEMANTICS_SEQUENTIAL, false);
  }

 private:
  RunResult run(std::span<const int> prompt, const SimConfig& cfg, int semantics, bool with_transcript) const {
    RunResult r;
    const long cap = cfg.rounds * (cfg.lookahead + 1);
    const int b = cfg.batch_size;
    std::vector<int> all(size_t(cap) * size_t(b > 0 ? b : 1));
    std::vector<int64_t> lens(size_t(b > 0 ? b : 1));
    std::vector<int> oc(size_t(2 * cfg.rounds));
    r.hits.resize(size_t(cfg.rounds));
    const ssd_sim_config c = cfg.c();
    ssd_run_options opt{};
    opt.semantics = semantics;
    int64_t need = 0;
    std::vector<char> tbuf;
    if (with_transcript) {
      tbuf.resize(size_t(4096 + cfg.rounds * b * (96 + 16 * (cfg.lookahead + 4)) + 256 * cfg.rounds));
      opt.transcript = tbuf.data();
      opt.transcript_cap = int64_t(tbuf.size());
      opt.transcript_len = &need;
    }
    check(ssd_run_ssd_ex(h_.get(), prompt.data(), int(prompt.size()), &c, b, &opt, all.data(), cap, lens.data(),
                         oc.data(), r.hits.data(), &r.stats));
    if (with_transcript) {
      if (need >= int64_t(tbuf.size())) throw Error("transcript: buffer too small");
      r.transcript_jsonl.assign(tbuf.data(), size_t(need));
    }
    for (int j = 0; j < b; ++j)
      r.streams.emplace_back(all.begin() + long(j) * cap, all.begin() + long(j) * cap + lens[size_t(j)]);
    r.tokens = r.streams[0];
    for (long i = 0; i < cfg.rounds; ++i) r.outcomes.push_back({oc[size_t(2 * i)], oc[size_t(2 * i + 1)]});
    return r;
  }

  struct Del {
    void operator()(ssd_engine* e) const { ssd_engine_destroy(e); }
  };
  std::unique_ptr<ssd_engine, Del> h_;
  int vocab_ = 0;
};

}  // namespace ssdlab_b200
