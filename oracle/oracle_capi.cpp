// TEST INFRASTRUCTURE ONLY — extern "C" entry points into the CPU oracle,
// used by tests/ and bench.py (ctypes). JSON in, JSON out; the request
// schema is shared with oracle/ref_driver.cpp so the same request can be run
// through the restated oracle and through the compiled reference.
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>

#include <json.hpp>

#include "ssd_oracle.hpp"
#include "transformer_lm.hpp"

using nlohmann::json;
using namespace oracle;

namespace {

Scheme parse_scheme(const json& j) {
  Scheme s;
  if (j.is_null()) return s;
  const std::string kind = j.value("kind", std::string("standard"));
  s.saguaro = kind == "saguaro";
  s.temperature = j.value("temperature", 1.0);
  s.fan_out = j.value("fan_out", 0);
  s.downweight = j.value("downweight", 1.0);
  return s;
}

Plan parse_plan(const json& j, int K, Origin role) {
  if (j.contains("fan")) {
    Plan p{j.at("fan").get<std::vector<int>>(), role, 0};
    p.budget = j.value("budget", p.total());
    return p;
  }
  if (j.contains("uniform")) return uniform_plan(K, j.at("uniform").get<int>(), role);
  const auto g = j.at("geometric");  // [acceptance, exponent, budget]
  return geometric_plan(g.at(0).get<double>(), g.at(1).get<double>(), K, g.at(2).get<int>(), role);
}

json stats_json(const Stats& s) {
  json o;
  o["rounds"] = s.rounds; o["batch"] = s.batch; o["tokens"] = s.tokens; o["vtime"] = s.vtime;
  o["p_lookups"] = s.p_lookups; o["p_hits"] = s.p_hits; o["b_lookups"] = s.b_lookups; o["b_hits"] = s.b_hits;
  o["hit_rounds"] = s.hit_rounds; o["miss_rounds"] = s.miss_rounds; o["initial_rounds"] = s.initial_rounds;
  o["hit_round_tokens"] = s.hit_round_tokens; o["miss_round_tokens"] = s.miss_round_tokens;
  o["accepted_sum"] = s.accepted_sum;
  o["streams"] = s.streams;
  json log = json::array();
  for (const auto& e : s.log) log.push_back({e.primary_origin ? 1 : 0, e.hit ? 1 : 0});
  o["log"] = log;
  return o;
}

struct MarkovModels {
  std::unique_ptr<MarkovLM> target, draft;
  double eps = 0.0;
};

// reference cli.cpp:120-146 (build_models): noise seed = child_seed(seed, 1).
MarkovModels build_markov(const json& lm) {
  MarkovModels m;
  const auto seed = lm.value("seed", std::uint64_t(0));
  if (lm.contains("target_rows")) {  // hand-built tables (reference test fixtures)
    const auto tr = lm.at("target_rows").get<std::vector<Row>>();
    const auto dr = lm.value("draft_rows", tr);
    m.target = std::make_unique<MarkovLM>(int(tr[0].size()), lm.at("order").get<int>(), seed, tr);
    m.draft = std::make_unique<MarkovLM>(int(dr[0].size()), lm.at("order").get<int>(), seed, dr);
    return m;
  }
  m.target = std::make_unique<MarkovLM>(markov_make(lm.at("vocab").get<int>(), lm.at("order").get<int>(),
                                                    lm.at("concentration").get<double>(), seed));
  const std::uint64_t noise = lm.value("noise_seed", child_seed(seed, 1));
  if (lm.contains("alpha_goal")) {
    MarkovPair p = markov_calibrate(*m.target, lm.at("alpha_goal").get<double>(), noise);
    m.eps = p.eps;
    m.draft = std::make_unique<MarkovLM>(std::move(p.draft));
  } else {
    m.eps = lm.at("epsilon").get<double>();
    m.draft = std::make_unique<MarkovLM>(markov_mix_draft(*m.target, m.eps, noise));
  }
  return m;
}

// ---- transformer pairs, kept alive across calls (weights are expensive)
struct TfPair {
  std::unique_ptr<TransformerLM> target, draft;
};
std::mutex g_mu;
std::map<int, TfPair> g_pairs;
int g_next = 1;

TfShape parse_shape(const json& j) {
  TfShape s;
  s.vocab = j.at("vocab"); s.d = j.at("d"); s.layers = j.at("layers"); s.heads = j.at("heads");
  s.kv_heads = j.at("kv_heads"); s.head_dim = j.at("head_dim"); s.ffn = j.at("ffn");
  s.tied = j.value("tied", false); s.rope_theta = j.value("rope_theta", 500000.0);
  s.norm_eps = j.value("norm_eps", 1e-5f); s.max_ctx = j.value("max_ctx", 4096);
  return s;
}

PairParams parse_pair(const json& j) {
  PairParams p;
  p.seed = j.value("seed", p.seed);
  p.embed_scale = j.value("embed_scale", p.embed_scale);
  p.block_out_scale = j.value("block_out_scale", p.block_out_scale);
  p.shared_mlp_scale = j.value("shared_mlp_scale", p.shared_mlp_scale);
  p.target_private_embed = j.value("target_private_embed", p.target_private_embed);
  p.target_private_head = j.value("target_private_head", p.target_private_head);
  p.draft_gain_mix = j.value("draft_gain_mix", p.draft_gain_mix);
  p.logit_scale = j.value("logit_scale", p.logit_scale);
  return p;
}

struct Models {
  LanguageModel* target = nullptr;
  LanguageModel* draft = nullptr;
  MarkovModels markov;
  double eps = 0.0;
};

Models resolve(const json& req) {
  Models m;
  if (req.contains("tf_pair")) {
    std::lock_guard<std::mutex> g(g_mu);
    TfPair& p = g_pairs.at(req.at("tf_pair").get<int>());
    m.target = p.target.get();
    m.draft = p.draft.get();
    return m;
  }
  m.markov = build_markov(req.at("lm"));
  m.target = m.markov.target.get();
  m.draft = m.markov.draft.get();
  m.eps = m.markov.eps;
  return m;
}

SimCfg build_sim(const json& req, Models& m) {
  SimCfg c;
  c.target = m.target;
  c.draft = m.draft;
  c.K = req.at("lookahead");
  c.scheme = parse_scheme(req.value("scheme", json()));
  // reference cli.cpp:211-212: target scheme = standard(scheme.temperature)
  if (req.contains("target_scheme")) c.target_scheme = parse_scheme(req.at("target_scheme"));
  else c.target_scheme.temperature = c.scheme.temperature;
  if (req.contains("primary_plan")) c.primary_plan = parse_plan(req.at("primary_plan"), c.K, Origin::Primary);
  if (req.contains("backup_plan")) c.backup_plan = parse_plan(req.at("backup_plan"), c.K, Origin::Backup);
  const json t = req.value("timing", json::object());
  c.primary_time = t.value("primary_time", 0.3);
  c.backup_time_fast = t.value("backup_time", 0.0);
  c.backup = req.value("backup", std::string("fast_random")) == "same_primary_jit" ? Backup::SamePrimaryJIT : Backup::FastRandom;
  if (req.contains("synthetic_hit_rate")) { c.synthetic_iid = true; c.synthetic_hit_rate = req.at("synthetic_hit_rate"); }
  c.batch = req.value("batch_size", 1);
  c.rounds = req.value("rounds", 1000L);
  c.seed = req.at("seed").get<std::uint64_t>();
  c.accept_scale = req.value("accept_scale", 1.0);
  c.keep_streams = req.value("keep_streams", true);
  if (req.contains("prompt")) c.prompt = req.at("prompt").get<std::vector<int>>();
  return c;
}

json spec_json(const Spec& s, bool with_dists) {
  json o;
  o["tokens"] = s.tokens;
  o["origin"] = int(s.origin);
  if (with_dists) o["dists"] = s.dists;
  return o;
}

json run(const json& req) {
  const std::string op = req.at("op");
  if (op == "models") {
    MarkovModels m = build_markov(req.at("lm"));
    return json{{"eps", m.eps}, {"target", m.target->rows()}, {"draft", m.draft->rows()}};
  }
  if (op == "fanout") {
    const int K = req.at("lookahead");
    json o;
    if (req.contains("uniform")) o["fan"] = uniform_plan(K, req.at("uniform")).fan;
    else {
      const auto g = req.at("geometric");
      o["fan"] = geometric_plan(g.at(0), g.at(1), K, g.at(2)).fan;
      o["continuous"] = geometric_plan_continuous(g.at(0), g.at(1), K, g.at(2).get<double>());
    }
    return o;
  }
  if (op == "fit_powerlaw") {  // hitmodel.cpp:65-106
    std::vector<std::pair<double, double>> sm;
    for (const auto& e : req.at("samples")) sm.emplace_back(e.at(0).get<double>(), e.at(1).get<double>());
    const PowerLaw f = fit_powerlaw(sm);
    return json{{"exponent", f.exponent}, {"log_amplitude", f.log_amplitude}, {"r_squared", f.r_squared}};
  }
  if (op == "perf") {  // perf.cpp:19-73
    const Yields y{req.at("hit_tokens").get<double>(), req.at("miss_tokens").get<double>()};
    const double p = req.at("hit_rate"), tp = req.at("primary_time"), tb = req.value("backup_time", 0.0);
    json o;
    o["speedup_ssd"] = speedup_ssd(p, y, tp, tb);
    if (req.contains("batch")) o["speedup_batch"] = speedup_batch(p, y, tp, tb, req.at("batch").get<double>());
    if (req.value("critical", false)) o["critical_batch"] = critical_batch(p, y, tp);
    return o;
  }
  if (op == "top_indices") {
    const auto z = req.at("z").get<std::vector<double>>();
    return json{{"idx", rank_tokens(z, req.at("count"))}};
  }
  if (op == "apply_scheme") {
    const auto z = req.at("z").get<std::vector<double>>();
    return json{{"p", scheme_probs(z, parse_scheme(req.at("scheme")))}};
  }
  if (op == "residual") {
    return json{{"p", residual_probs(req.at("target").get<std::vector<double>>(), req.at("draft").get<std::vector<double>>())}};
  }
  if (op == "sample") {
    Rng r(req.at("seed").get<std::uint64_t>());
    const auto p = req.at("p").get<std::vector<double>>();
    std::vector<int> out;
    for (int i = 0; i < req.value("n", 1); ++i) out.push_back(draw(p, r));
    return json{{"draws", out}};
  }
  if (op == "verify_rows") {
    // specdec.cpp:27-69 on given logit rows: target row i is the target's
    // logits after ctx ++ s_1..s_i; draft rows give the recorded laws (absent
    // => the exact uniform law of the FastRandom backup, sim.cpp:35-48).
    struct RowsLM : LanguageModel {
      std::vector<Row> rows;
      int vocab() const override { return int(rows[0].size()); }
      std::span<const double> logits(std::span<const int> ctx) override { return rows.at(ctx.size() - 1); }
    } lm;
    lm.rows = req.at("target_rows").get<std::vector<Row>>();
    const auto toks = req.at("tokens").get<std::vector<int>>();
    const Scheme ds = parse_scheme(req.value("scheme", json()));
    Spec spec;
    spec.tokens = toks;
    if (req.contains("draft_rows")) {
      for (const auto& r : req.at("draft_rows")) spec.dists.push_back(scheme_probs(r.get<Row>(), ds));
    } else {
      spec.dists.assign(toks.size(), Row(lm.rows[0].size(), 1.0 / double(lm.rows[0].size())));
    }
    VerifyOpts vo;
    vo.target_scheme = parse_scheme(req.value("target_scheme", json()));
    vo.accept_scale = req.value("accept_scale", 1.0);
    Rng r(req.at("seed").get<std::uint64_t>());
    const std::vector<int> ctx{0};
    const Round out = verify_spec(lm, ctx, spec, r, vo);
    return json{{"accepted", out.key.k}, {"bonus", out.key.t}};
  }
  if (op == "keys_rows") {
    // cache.cpp:249-270 key selection on given rows.
    const auto rows = req.at("rows").get<std::vector<Row>>();
    const auto fan = req.at("fan").get<std::vector<int>>();
    const auto excl = req.at("excluded").get<std::vector<int>>();
    json keys = json::array();
    for (std::size_t k = 0; k < rows.size(); ++k) {
      std::vector<int> got;
      const int need = std::min(int(rows[k].size()), fan[k] + 1);
      for (int c : rank_tokens(rows[k], need)) {
        if (c == excl[k]) continue;
        if (int(got.size()) == fan[k]) break;
        got.push_back(c);
      }
      keys.push_back(got);
    }
    return json{{"keys", keys}};
  }
  Models m = resolve(req);
  if (op == "chain") {
    // One caller stream through draft -> verify -> build_cache, as a reference
    // caller threads its rng::Stream& (specdec.hpp:59-61, 81-83; cache.hpp:149-154);
    // "next_u64" = the stream's next draw afterwards (its position).
    const Scheme s = parse_scheme(req.value("scheme", json()));
    const int K = req.at("lookahead");
    const auto ctx = req.at("context").get<std::vector<int>>();
    Rng rng(req.at("seed").get<std::uint64_t>());
    const Spec spec = draft_tokens(*m.draft, ctx, K, s, rng, Origin::Primary);
    VerifyOpts vo;
    if (req.contains("target_scheme")) vo.target_scheme = parse_scheme(req.at("target_scheme"));
    else vo.target_scheme.temperature = s.temperature;
    vo.accept_scale = req.value("accept_scale", 1.0);
    const Round r = verify_spec(*m.target, ctx, spec, rng, vo);
    const Plan plan = parse_plan(req.at("plan"), K, Origin::Primary);
    const SpecCache c = prespeculate(*m.draft, ctx, spec, plan, s, req.value("next_lookahead", K), rng);
    json entries = json::array();
    for (const auto& e : c.entries) entries.push_back({e.key.k, e.key.t, e.spec.tokens});
    json o;
    o["spec"] = spec_json(spec, false);
    o["accepted"] = r.key.k;
    o["bonus"] = r.key.t;
    o["emitted"] = r.emitted;
    o["entries"] = entries;
    o["next_u64"] = rng.bits();
    return o;
  }
  if (op == "draft" || op == "verify" || op == "build_cache") {
    const Scheme s = parse_scheme(req.value("scheme", json()));
    const int K = req.at("lookahead");
    const auto ctx = req.at("context").get<std::vector<int>>();
    Spec spec;
    if (req.contains("spec")) {  // explicit speculation (tokens + recorded dists)
      spec.tokens = req.at("spec").at("tokens").get<std::vector<int>>();
      spec.dists = req.at("spec").at("dists").get<std::vector<Row>>();
      spec.origin = req.value("origin", 0) ? Origin::Backup : Origin::Primary;
    } else {
      Rng dr(req.at("draft_seed").get<std::uint64_t>());
      spec = draft_tokens(*m.draft, ctx, K, s, dr, req.value("origin", 0) ? Origin::Backup : Origin::Primary);
    }
    json o;
    o["spec"] = spec_json(spec, req.value("with_dists", false));
    if (op == "verify") {
      Rng vr(req.at("seed").get<std::uint64_t>());
      VerifyOpts vo;
      if (req.contains("target_scheme")) vo.target_scheme = parse_scheme(req.at("target_scheme"));
      else vo.target_scheme.temperature = s.temperature;
      vo.accept_scale = req.value("accept_scale", 1.0);
      const Round r = verify_spec(*m.target, ctx, spec, vr, vo);
      o["accepted"] = r.key.k; o["bonus"] = r.key.t; o["emitted"] = r.emitted;
    }
    if (op == "build_cache") {
      Rng cr(req.at("seed").get<std::uint64_t>());
      const Plan plan = parse_plan(req.at("plan"), K, spec.origin);
      const SpecCache c = prespeculate(*m.draft, ctx, spec, plan, s, req.value("next_lookahead", K), cr);
      json entries = json::array();
      for (const auto& e : c.entries) entries.push_back({e.key.k, e.key.t, e.spec.tokens});
      std::sort(entries.begin(), entries.end());
      o["entries"] = entries;
    }
    return o;
  }
  if (op == "simulate") {
    SimCfg c = build_sim(req, m);
    const std::string mode = req.at("mode");
    json o;
    if (mode == "ar") o = stats_json(sim_ar(*m.target, c.target_scheme, c.rounds, c.seed, c.prompt));
    else if (mode == "sd") o = stats_json(sim_sd(c));
    else if (mode == "ssd") o = stats_json(sim_ssd(c));
    else if (mode == "harness") {
      const HarnessOut h = sim_harness(c);
      o = stats_json(h.stats);
      json tr = json::array();
      for (const auto& msg : h.transcript)
        tr.push_back({{"round", msg.round}, {"dir", msg.dir}, {"payload_summary", json::parse(msg.summary)}, {"vclock", msg.vclock}});
      o["transcript"] = tr;
      json tm = json::array();
      for (const auto& t : h.timings) tm.push_back({t.verify_start, t.verify_end, t.cache_ready, t.all_hit});
      o["timings"] = tm;
      json oc = json::array();
      for (const auto& k : h.outcomes0) oc.push_back({k.k, k.t});
      o["outcomes0"] = oc;
      o["hits0"] = h.hits0;
      o["decode_seconds"] = h.decode_seconds;
    } else {
      throw ConfigError("config: mode must be ar, sd, ssd or harness");
    }
    o["eps"] = m.eps;
    o["primary_plan"] = c.primary_plan.fan;
    o["backup_plan"] = c.backup_plan.fan;
    return o;
  }
  throw ConfigError("unknown op " + op);
}

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

}  // namespace

extern "C" {

// Returns a malloc'd JSON string: either the result or {"error": msg, "code": c}.
char* oracle_call(const char* request) {
  try {
    return dup(run(json::parse(request)).dump());
  } catch (const oracle::Error& e) {
    return dup(json{{"error", e.what()}, {"code", e.code()}}.dump());
  } catch (const std::exception& e) {
    return dup(json{{"error", e.what()}, {"code", 1}}.dump());
  }
}

void oracle_free(char* p) { std::free(p); }

// Transformer pair: {"target": shape, "draft": shape, "pair": params, "threads": n, "accum": "f32"|"f64"}
int oracle_tf_create(const char* request) {
  try {
    const json j = json::parse(request);
    const TfShape ts = parse_shape(j.at("target")), ds = parse_shape(j.at("draft"));
    const PairParams pp = parse_pair(j.value("pair", json::object()));
    const int threads = j.value("threads", 0);
    TfPair p;
    p.target = std::make_unique<TransformerLM>(ts, ds, pp, Role::Target, threads);
    p.draft = std::make_unique<TransformerLM>(ds, ds, pp, Role::Draft, threads);
    if (j.value("accum", std::string("f32")) == "f64") {
      p.target->set_f64(true);
      p.draft->set_f64(true);
    }
    std::lock_guard<std::mutex> g(g_mu);
    g_pairs[g_next] = std::move(p);
    return g_next++;
  } catch (const std::exception&) {
    return -1;
  }
}

void oracle_tf_destroy(int h) {
  std::lock_guard<std::mutex> g(g_mu);
  g_pairs.erase(h);
}

// fp32 logits of model (0 target, 1 draft) after `ctx`; returns 0 on success.
int oracle_tf_logits(int h, int which, const int* ctx, int n, float* out) {
  try {
    TransformerLM* m;
    {
      std::lock_guard<std::mutex> g(g_mu);
      TfPair& p = g_pairs.at(h);
      m = which == 0 ? p.target.get() : p.draft.get();
    }
    m->logits(std::span<const int>(ctx, std::size_t(n)));
    std::memcpy(out, m->last_logits_f32().data(), m->last_logits_f32().size() * sizeof(float));
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

// Raw bf16 bits of weight elements, for generator parity: kind 0..6 layer
// tensors, 100 embed, 101 head. Returns 0 on success.
int oracle_tf_weight_bits(int h, int which, int layer, int kind, const long* rows, const long* cols, int n,
                          unsigned short* out) {
  try {
    std::lock_guard<std::mutex> g(g_mu);
    TfPair& p = g_pairs.at(h);
    TransformerLM* m = which == 0 ? p.target.get() : p.draft.get();
    for (int i = 0; i < n; ++i) {
      if (kind == 100) out[i] = m->embed_bits(std::size_t(rows[i]), std::size_t(cols[i]));
      else if (kind == 101) out[i] = m->head_bits(std::size_t(rows[i]), std::size_t(cols[i]));
      else out[i] = m->weight_bits(layer, TensorKind(kind), std::size_t(rows[i]), std::size_t(cols[i]));
    }
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

float oracle_tf_final_gain(int h, int which, int i) {
  std::lock_guard<std::mutex> g(g_mu);
  TfPair& p = g_pairs.at(h);
  return (which == 0 ? p.target : p.draft)->final_gain(std::size_t(i));
}

}  // extern "C"
