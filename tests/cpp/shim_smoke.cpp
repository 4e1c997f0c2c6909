// Drives the B200 engine through include/ssdlab_b200.hpp — the reference's
// ssdlab-style C++ interface — the way a reference-side caller would
// (sim.cpp's loops, test_cache.cpp's lookups). Prints one JSON line that
// tests/test_shim.py compares with the Python mirror of the same calls.
// Build: g++ -std=c++20 -I include tests/cpp/shim_smoke.cpp -L paper_2603_03251_b200 -lssd_b200
#include <cstdio>
#include <string>
#include <vector>

#include "ssdlab_b200.hpp"

using namespace ssdlab_b200;

static ssd_model_shape shape(int V, int d, int L, int H, int KVH, int hd, int F, int tied) {
  ssd_model_shape s{};
  s.vocab = V; s.d_model = d; s.n_layers = L; s.n_heads = H; s.n_kv_heads = KVH; s.head_dim = hd; s.ffn = F;
  s.tied = tied; s.max_ctx = 512; s.rope_theta = 500000.0; s.norm_eps = 1e-5f;
  return s;
}

static std::string ints(const std::vector<int>& v) {
  std::string s = "[";
  for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
  return s + "]";
}

int main(int argc, char** argv) {
  const bool compile_only = argc > 1 && std::string(argv[1]) == "--no-gpu";
  if (compile_only) {  // link check: plans are host-only
    FanOutPlan p = uniform_fanout(4, 20);
    std::printf("{\"uniform\": %s}\n", ints(p.fan_out).c_str());
    return p.total() == 20 ? 0 : 1;
  }
  const ssd_model_shape t = shape(32000, 512, 8, 8, 8, 64, 1536, 0), d = shape(32000, 256, 2, 4, 4, 64, 768, 1);
  const ssd_pair_params pair{20250809ull, 1.0f, 8.0f, 0.1f, 0.1f, 0.25f, 0.0f, 0.25f};
  Engine eng(t, d, pair, 0, 32, 4);
  std::vector<int> prompt;
  for (int i = 0; i < 8; ++i) prompt.push_back((i * 7919 + 13) % 32000);

  SimConfig cfg;
  cfg.lookahead = 4;
  cfg.scheme = SamplingScheme::greedy();
  cfg.target_scheme = SamplingScheme::greedy();
  cfg.primary_plan = FanOutPlan{{4, 4, 4, 4, 4}, Origin::Primary, 0};
  cfg.backup_plan = FanOutPlan{{4, 4, 4, 4, 4}, Origin::Backup, 0};
  cfg.primary_time = 0.4;
  cfg.rounds = 6;
  cfg.seed = 1;
  const RunResult r = eng.run_ssd(prompt, cfg);

  // emitted tokens are exactly the accepted prefix + bonus of each round
  size_t at = 0;
  bool consistent = true;
  for (const auto& o : r.outcomes) {
    at += size_t(o.accepted) + 1;
    if (at > r.tokens.size() || r.tokens[at - 1] != o.bonus) consistent = false;
  }
  consistent = consistent && at == r.tokens.size();

  // build_cache / lookup (cache.hpp:123-126): every key hits, a foreign key misses
  const Speculation spec = eng.draft(prompt, 4, SamplingScheme::greedy(), 7, false, Origin::Primary);
  const SpeculationCache cache = eng.build_cache(prompt, spec, cfg.primary_plan, SamplingScheme::greedy(), 4, 11);
  bool lookups = cache.size() == 20;
  for (const auto& [k, v] : cache.entries()) lookups = lookups && cache.lookup(k) == &v && v.tokens.size() == 4;
  lookups = lookups && cache.lookup(VerificationOutcome{0, spec.tokens[0]}) == nullptr;  // excluded s_1

  // errors map onto the reference classes (errors.hpp)
  bool too_large = false;
  try {
    SimConfig bad = cfg;
    bad.primary_plan = FanOutPlan{{40, 40, 40, 40, 40}, Origin::Primary, 0};
    eng.run_ssd(prompt, bad);
  } catch (const TooLargeError&) {
    too_large = true;
  }

  std::printf("{\"tokens\": %s, \"hit_rate\": %.6f, \"consistent\": %s, \"lookups\": %s, \"too_large\": %s, "
              "\"spec\": %s, \"cache_size\": %zu}\n",
              ints(r.tokens).c_str(), r.hit_rate(), consistent ? "true" : "false", lookups ? "true" : "false",
              too_large ? "true" : "false", ints(spec.tokens).c_str(), cache.size());
  return (consistent && lookups && too_large) ? 0 : 1;
}
