// TEST INFRASTRUCTURE ONLY — extern "C" driver over the UNMODIFIED reference
// (ssd-lab) hot-path sources, compiled from /root/reference/proj/src by
// oracle/Makefile into oracle/_ref/libssdref.so. Same JSON request schema as
// oracle/oracle_capi.cpp, so one request runs through both and the outputs
// are compared bit-for-bit (tests/test_oracle_golden.py) and frozen as
// golden fixtures (tests/golden/, made by oracle/make_golden.py).
//
// This file is my own code; it only calls the reference's public API
// (ssdlab/{categorical,lm,specdec,cache,sim}.hpp).
#include <algorithm>
#include <cstring>
#include <memory>
#include <string>

#include <json.hpp>

#include "ssdlab/cache.hpp"
#include "ssdlab/categorical.hpp"
#include "ssdlab/errors.hpp"
#include "ssdlab/hitmodel.hpp"
#include "ssdlab/perf.hpp"
#include "ssdlab/lm.hpp"
#include "ssdlab/rng.hpp"
#include "ssdlab/sim.hpp"
#include "ssdlab/specdec.hpp"

using nlohmann::json;
using namespace ssdlab;

namespace {

dist::SamplingScheme scheme_of(const json& j) {
  if (j.is_null()) return dist::SamplingScheme::standard();
  const std::string kind = j.value("kind", std::string("standard"));
  const double tau = j.value("temperature", 1.0);
  if (kind == "saguaro") return dist::SamplingScheme::saguaro(j.value("fan_out", 0), j.value("downweight", 1.0), tau);
  return dist::SamplingScheme::standard(tau);
}

cache::FanOutPlan plan_of(const json& j, int K, specdec::Origin role) {
  if (j.contains("fan")) {
    cache::FanOutPlan p{j.at("fan").get<std::vector<int>>(), role, 0};
    p.budget = j.value("budget", p.total());
    return p;
  }
  if (j.contains("uniform")) return cache::uniform_fanout(K, j.at("uniform").get<int>(), role);
  const auto g = j.at("geometric");
  return cache::geometric_fanout(g.at(0).get<double>(), g.at(1).get<double>(), K, g.at(2).get<int>(), role);
}

struct Pair {
  std::shared_ptr<lm::SyntheticLM> target, draft;
  double eps = 0.0;
};

// Mirrors cli.cpp build_models (noise seed derive_seed(seed, 1)).
Pair models_of(const json& lmj) {
  Pair p;
  const auto seed = lmj.value("seed", std::uint64_t(0));
  if (lmj.contains("target_rows")) {  // hand-built tables (reference test fixtures)
    auto rows = [](const json& j) {
      std::vector<dist::Logits> r;
      for (const auto& x : j) r.push_back(dist::Logits{x.get<std::vector<double>>()});
      return r;
    };
    const json dr = lmj.value("draft_rows", lmj.at("target_rows"));
    const int order = lmj.at("order");
    p.target = std::make_shared<lm::SyntheticLM>(int(lmj.at("target_rows")[0].size()), order, seed, rows(lmj.at("target_rows")));
    p.draft = std::make_shared<lm::SyntheticLM>(int(dr[0].size()), order, seed, rows(dr));
    return p;
  }
  p.target = std::make_shared<lm::SyntheticLM>(lm::make_lm(lmj.at("vocab").get<int>(), lmj.at("order").get<int>(),
                                                           lmj.at("concentration").get<double>(), seed));
  const std::uint64_t noise = lmj.value("noise_seed", rng::derive_seed(seed, 1));
  if (lmj.contains("alpha_goal")) {
    auto pr = lm::calibrate_pair(*p.target, lmj.at("alpha_goal").get<double>(), noise);
    p.eps = pr.epsilon;
    p.draft = std::make_shared<lm::SyntheticLM>(std::move(pr.draft));
  } else {
    p.eps = lmj.at("epsilon").get<double>();
    p.draft = std::make_shared<lm::SyntheticLM>(lm::derive_draft(*p.target, p.eps, noise));
  }
  return p;
}

std::vector<std::vector<double>> rows_of(const lm::SyntheticLM& m) {
  std::vector<std::vector<double>> r;
  for (const auto& row : m.rows()) r.push_back(row.values);
  return r;
}

json stats_json(const sim::RunStats& s) {
  json o;
  o["rounds"] = s.rounds; o["batch"] = s.batch; o["tokens"] = s.tokens; o["vtime"] = s.virtual_time;
  o["p_lookups"] = s.primary_origin_lookups; o["p_hits"] = s.primary_origin_hits;
  o["b_lookups"] = s.backup_origin_lookups; o["b_hits"] = s.backup_origin_hits;
  o["hit_rounds"] = s.hit_rounds; o["miss_rounds"] = s.miss_rounds; o["initial_rounds"] = s.initial_rounds;
  o["hit_round_tokens"] = s.hit_round_tokens; o["miss_round_tokens"] = s.miss_round_tokens;
  o["accepted_sum"] = s.accepted_sum;
  o["streams"] = s.streams;
  json log = json::array();
  for (const auto& e : s.round_log) log.push_back({e.primary_origin ? 1 : 0, e.hit ? 1 : 0});
  o["log"] = log;
  return o;
}

json run(const json& req) {
  const std::string op = req.at("op");
  if (op == "fanout") {
    const int K = req.at("lookahead");
    json o;
    if (req.contains("uniform")) o["fan"] = cache::uniform_fanout(K, req.at("uniform")).fan_out;
    else {
      const auto g = req.at("geometric");
      o["fan"] = cache::geometric_fanout(g.at(0), g.at(1), K, g.at(2)).fan_out;
      o["continuous"] = cache::geometric_fanout_continuous(g.at(0), g.at(1), K, g.at(2).get<double>()).fan_out;
    }
    return o;
  }
  if (op == "fit_powerlaw") {
    std::vector<std::pair<double, double>> sm;
    for (const auto& e : req.at("samples")) sm.emplace_back(e.at(0).get<double>(), e.at(1).get<double>());
    const hitmodel::PowerLawFit f = hitmodel::fit_powerlaw(sm);
    return json{{"exponent", f.exponent}, {"log_amplitude", f.log_amplitude}, {"r_squared", f.r_squared}};
  }
  if (op == "perf") {
    const perf::TokenYields y{req.at("hit_tokens").get<double>(), req.at("miss_tokens").get<double>(), 1.0, 0.0};
    const perf::TimingParams t{req.at("primary_time").get<double>(), req.value("backup_time", 0.0)};
    const double p = req.at("hit_rate");
    json o;
    o["speedup_ssd"] = perf::speedup_ssd(p, y, t);
    if (req.contains("batch")) o["speedup_batch"] = perf::speedup_batch(p, y, t, req.at("batch").get<double>());
    if (req.value("critical", false)) o["critical_batch"] = perf::critical_batch(p, y, t);
    return o;
  }
  if (op == "top_indices") {
    return json{{"idx", dist::top_indices(dist::Logits{req.at("z").get<std::vector<double>>()}, req.at("count"))}};
  }
  if (op == "apply_scheme") {
    return json{{"p", dist::apply_scheme(dist::Logits{req.at("z").get<std::vector<double>>()}, scheme_of(req.at("scheme"))).probs}};
  }
  if (op == "residual") {
    return json{{"p", dist::residual(dist::Categorical{req.at("target").get<std::vector<double>>()},
                                     dist::Categorical{req.at("draft").get<std::vector<double>>()}).probs}};
  }
  if (op == "sample") {
    rng::Stream r(req.at("seed").get<std::uint64_t>());
    const dist::Categorical p{req.at("p").get<std::vector<double>>()};
    std::vector<int> out;
    for (int i = 0; i < req.value("n", 1); ++i) out.push_back(dist::sample(p, r));
    return json{{"draws", out}};
  }
  const Pair m = models_of(req.at("lm"));
  if (op == "models") return json{{"eps", m.eps}, {"target", rows_of(*m.target)}, {"draft", rows_of(*m.draft)}};
  if (op == "draft" || op == "verify" || op == "build_cache") {
    const auto s = scheme_of(req.value("scheme", json()));
    const int K = req.at("lookahead");
    const auto ctx = req.at("context").get<std::vector<int>>();
    specdec::Speculation spec;
    if (req.contains("spec")) {
      spec.tokens = req.at("spec").at("tokens").get<std::vector<int>>();
      for (const auto& d : req.at("spec").at("dists")) spec.draft_dists.push_back(dist::Categorical{d.get<std::vector<double>>()});
      spec.origin = req.value("origin", 0) ? specdec::Origin::Backup : specdec::Origin::Primary;
    } else {
      rng::Stream dr(req.at("draft_seed").get<std::uint64_t>());
      spec = specdec::draft(*m.draft, ctx, K, s, dr, req.value("origin", 0) ? specdec::Origin::Backup : specdec::Origin::Primary);
    }
    json o;
    o["spec"] = {{"tokens", spec.tokens}, {"origin", int(spec.origin)}};
    if (req.value("with_dists", false)) {
      std::vector<std::vector<double>> d;
      for (const auto& c : spec.draft_dists) d.push_back(c.probs);
      o["spec"]["dists"] = d;
    }
    if (op == "verify") {
      rng::Stream vr(req.at("seed").get<std::uint64_t>());
      specdec::VerifyOptions vo;
      vo.target_scheme = req.contains("target_scheme") ? scheme_of(req.at("target_scheme"))
                                                       : dist::SamplingScheme::standard(s.temperature);
      vo.accept_scale = req.value("accept_scale", 1.0);
      const auto r = specdec::verify(*m.target, ctx, spec, vr, vo);
      o["accepted"] = r.outcome.accepted; o["bonus"] = r.outcome.bonus; o["emitted"] = r.emitted;
    }
    if (op == "build_cache") {
      rng::Stream cr(req.at("seed").get<std::uint64_t>());
      const auto plan = plan_of(req.at("plan"), K, spec.origin);
      const auto c = cache::build_cache(*m.draft, ctx, spec, plan, s, req.value("next_lookahead", K), cr);
      json entries = json::array();
      for (const auto& [key, sp] : c.entries()) entries.push_back({key.accepted, key.bonus, sp.tokens});
      std::sort(entries.begin(), entries.end());
      o["entries"] = entries;
    }
    return o;
  }
  if (op == "simulate") {
    sim::SimConfig c;
    c.target = m.target;
    c.draft = m.draft;
    c.lookahead = req.at("lookahead");
    c.scheme = scheme_of(req.value("scheme", json()));
    c.target_scheme = req.contains("target_scheme") ? scheme_of(req.at("target_scheme"))
                                                    : dist::SamplingScheme::standard(c.scheme.temperature);
    if (req.contains("primary_plan")) c.primary_plan = plan_of(req.at("primary_plan"), c.lookahead, specdec::Origin::Primary);
    if (req.contains("backup_plan")) c.backup_plan = plan_of(req.at("backup_plan"), c.lookahead, specdec::Origin::Backup);
    const json t = req.value("timing", json::object());
    c.timing = {t.value("primary_time", 0.3), t.value("backup_time", 0.0)};
    c.backup_kind = req.value("backup", std::string("fast_random")) == "same_primary_jit" ? sim::BackupKind::SamePrimaryJIT
                                                                                      : sim::BackupKind::FastRandom;
    if (req.contains("synthetic_hit_rate")) {
      c.hit_mode = sim::HitMode::SyntheticIid;
      c.synthetic_hit_rate = req.at("synthetic_hit_rate");
    }
    c.batch_size = req.value("batch_size", 1);
    c.rounds = req.value("rounds", 1000L);
    c.seed = req.at("seed").get<std::uint64_t>();
    c.accept_scale = req.value("accept_scale", 1.0);
    c.keep_streams = req.value("keep_streams", true);
    const std::string mode = req.at("mode");
    json o;
    if (mode == "ar") o = stats_json(sim::run_ar(*m.target, c.target_scheme, c.rounds, c.seed));
    else if (mode == "sd") o = stats_json(sim::run_sd(c));
    else if (mode == "ssd") o = stats_json(c.batch_size > 1 ? sim::run_ssd_batch(c) : sim::run_ssd(c));
    else if (mode == "harness") {
      const auto h = sim::run_protocol_harness(c);
      o = stats_json(h.stats);
      json tr = json::array();
      for (const auto& msg : h.transcript.messages)
        tr.push_back({{"round", msg.round}, {"dir", msg.dir}, {"payload_summary", json::parse(msg.payload_summary)}, {"vclock", msg.vclock}});
      o["transcript"] = tr;
      json tm = json::array();
      for (const auto& x : h.timings) tm.push_back({x.verify_start, x.verify_end, x.cache_ready, x.all_hit});
      o["timings"] = tm;
    } else {
      throw ConfigError("config: mode must be ar, sd, ssd or harness");
    }
    o["eps"] = m.eps;
    o["primary_plan"] = c.primary_plan.fan_out;
    o["backup_plan"] = c.backup_plan.fan_out;
    return o;
  }
  throw ConfigError("unknown op " + op);
}

// errors.hpp:9-61 -> the C-ABI status numbering used across the repo.
int code_of(const std::exception& e) {
  if (dynamic_cast<const AllZeroError*>(&e)) return 2;
  if (dynamic_cast<const DegenerateResidualError*>(&e)) return 3;
  if (dynamic_cast<const TooLargeError*>(&e)) return 4;
  if (dynamic_cast<const BudgetTooSmallError*>(&e)) return 5;
  if (dynamic_cast<const DivergentError*>(&e)) return 6;
  if (dynamic_cast<const InsufficientDataError*>(&e)) return 7;
  if (dynamic_cast<const UnreachableError*>(&e)) return 8;
  if (dynamic_cast<const NoCrossoverError*>(&e)) return 9;
  if (dynamic_cast<const ProtocolViolationError*>(&e)) return 10;
  if (dynamic_cast<const ConfigError*>(&e)) return 11;
  return 1;
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

}  // namespace

extern "C" {
char* ref_call(const char* request) {
  try {
    return dup(run(json::parse(request)).dump());
  } catch (const std::exception& e) {
    return dup(json{{"error", e.what()}, {"code", code_of(e)}}.dump());
  }
}
void ref_free(char* p) { std::free(p); }
}
