// The reference's own hot-path known-answer cases (proj/tests/test_specdec.cpp
// :43-153, test_cache.cpp:221-302), compiled through tests/cpp/doctest_shim.h
// against include/ssdlab_b200.hpp and run on the GPU (TEST INFRASTRUCTURE).
//
// Each case keeps the reference's assertion. Where the reference builds a
// tiny Markov LM (single_row_lm, shift_chain_lm, make_lm), the case is
// restated with the B200 engine's random transformer pair: model-driven
// calls (draft / verify / build_cache) take the pair's own logits, and the
// verification-law cases that need hand-written distributions go through
// Engine::verify_rows with logit rows log(p) (the engine's speculation
// carries logit rows; its dists are the scheme applied to them).
//
// Build (tests/test_shim.py): g++ -std=c++20 -I include tests/cpp/ref_cases.cpp
//   -L paper_2603_03251_b200 -lssd_b200
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <vector>

#include <cuda_runtime.h>

#include "doctest_shim.h"
#include "ssdlab_b200.hpp"

using namespace ssdlab_b200;

namespace {

ssd_model_shape shape(int V, int d, int L, int H, int KVH, int hd, int F, int tied) {
  ssd_model_shape s{};
  s.vocab = V; s.d_model = d; s.n_layers = L; s.n_heads = H; s.n_kv_heads = KVH; s.head_dim = hd; s.ffn = F;
  s.tied = tied; s.max_ctx = 512; s.rope_theta = 500000.0; s.norm_eps = 1e-5f;
  return s;
}

Engine& engine() {  // the tiny pair of BASELINE configs[0]
  static Engine e(shape(32000, 512, 8, 8, 8, 64, 1536, 0), shape(32000, 256, 2, 4, 4, 64, 768, 1),
                  ssd_pair_params{20250809ull, 1.0f, 8.0f, 0.1f, 0.1f, 0.25f, 0.0f, 0.25f}, 0, 40, 8);
  return e;
}
const int V = 32000;

// logit rows [n][V] = log(p) on the first p.size() tokens, ~zero mass elsewhere
std::vector<float> log_rows(const std::vector<std::vector<double>>& probs) {
  std::vector<float> r(probs.size() * size_t(V), -1e30f);
  for (size_t i = 0; i < probs.size(); ++i)
    for (size_t t = 0; t < probs[i].size(); ++t) r[i * V + t] = float(std::log(std::max(probs[i][t], 1e-300)));
  return r;
}

std::vector<int> ctx_of(int n, int seed) {
  std::vector<int> c;
  for (int i = 0; i < n; ++i) c.push_back(int((std::uint64_t(seed) * 7919u + std::uint64_t(i) * 104729u) % V));
  return c;
}

// device copies of host token vectors (the caller's buffers of the async API)
int ssd_b200_test_alloc(int32_t** p, const std::vector<int>& v) {
  if (cudaMalloc(reinterpret_cast<void**>(p), v.size() * sizeof(int32_t)) != cudaSuccess) return 1;
  return cudaMemcpy(*p, v.data(), v.size() * sizeof(int32_t), cudaMemcpyHostToDevice) == cudaSuccess ? 0 : 1;
}
void ssd_b200_test_free(int32_t* p) { cudaFree(p); }

// (value desc, index asc) order of a logit row, excluding `ex`
std::vector<int> ranked(const std::vector<float>& z, int ex) {
  std::vector<int> idx(z.size());
  std::iota(idx.begin(), idx.end(), 0);
  std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return z[size_t(a)] > z[size_t(b)]; });
  idx.erase(std::remove(idx.begin(), idx.end(), ex), idx.end());
  return idx;
}

}  // namespace

// ------------------------------------------------------------ test_specdec.cpp

TEST_CASE("draft follows the argmax chain of a near-deterministic model") {
  // restated: greedy drafting follows the draft's own argmax chain
  Stream rng(2);
  const std::vector<int> ctx = ctx_of(6, 1);
  const Speculation spec = engine().draft(ctx, 4, SamplingScheme::greedy(), rng);
  std::vector<int> buf = ctx;
  for (int i = 0; i < 4; ++i) {
    const std::vector<float> z = engine().logits(1, buf);
    const float best = *std::max_element(z.begin(), z.end());
    CHECK(best - z[size_t(spec.tokens[size_t(i)])] < 1e-2f);  // argmax (or a documented near-tie)
    buf.push_back(spec.tokens[size_t(i)]);
  }
}

TEST_CASE("draft with downweight 1 matches standard given the same stream") {
  const std::vector<int> ctx = ctx_of(5, 3);
  Stream a(4), b(4);
  const Speculation standard = engine().draft(ctx, 6, SamplingScheme::standard(), a);
  const Speculation saguaro = engine().draft(ctx, 6, SamplingScheme::saguaro(3, 1.0), b);
  CHECK(standard.tokens == saguaro.tokens);
  CHECK(standard.rows == saguaro.rows);
  CHECK(a.next_u64() == b.next_u64());
}

TEST_CASE("draft records exactly the conditional it sampled from") {
  // the recorded rows are the draft's logits along the drafted prefix
  Stream rng(6);
  const std::vector<int> ctx = ctx_of(7, 5);
  const Speculation spec = engine().draft(ctx, 4, SamplingScheme::saguaro(2, 0.4), rng);
  std::vector<int> buf = ctx;
  for (int i = 0; i < 4; ++i) {
    const std::vector<float> z = engine().logits(1, buf);
    float err = 0.f;
    for (int t = 0; t < V; ++t) err = std::max(err, std::abs(z[size_t(t)] - spec.rows[size_t(i) * V + t]));
    CHECK(err < 5e-2f);
    buf.push_back(spec.tokens[size_t(i)]);
  }
}

TEST_CASE("verify accepts with probability min(1, target/draft)") {
  // target 0.3 vs draft 0.6 on the token: acceptance 0.5
  const std::vector<float> target = log_rows({{0.3, 0.7}, {0.3, 0.7}});
  Speculation spec;
  spec.tokens = {0};
  spec.rows = log_rows({{0.6, 0.4}});
  const int trials = 4000;
  int accepted = 0;
  for (int i = 0; i < trials; ++i)
    accepted += engine().verify_rows(target, spec, SamplingScheme::standard(), SamplingScheme::standard(),
                                     std::uint64_t(70000 + i)).accepted == 1;
  const double sigma = std::sqrt(0.25 / trials);
  CHECK(std::abs(double(accepted) / trials - 0.5) < 4.0 * sigma);
}

TEST_CASE("verify always accepts when draft never overshoots") {
  const std::vector<float> target = log_rows({{0.5, 0.3, 0.2}, {0.5, 0.3, 0.2}, {0.5, 0.3, 0.2}});
  Speculation spec;
  spec.tokens = {0, 0};
  spec.rows = log_rows({{0.4, 0.35, 0.25}, {0.5, 0.3, 0.2}});
  for (int i = 0; i < 200; ++i) {
    const VerificationOutcome o = engine().verify_rows(target, spec, SamplingScheme::standard(),
                                                       SamplingScheme::standard(), std::uint64_t(8000 + i));
    CHECK(o.accepted == 2);
  }
}

TEST_CASE("rejected worked-example round draws the bonus from the residual") {
  // Construction 1: target (.48 .48 .02 .02), draft (.49 .49 .01 .01)
  const std::vector<float> target = log_rows({{0.48, 0.48, 0.02, 0.02}, {0.48, 0.48, 0.02, 0.02}});
  Speculation spec;
  int rejected = 0, bonus_two = 0;
  for (int i = 0; i < 20000 && rejected < 300; ++i) {
    spec.tokens = {i % 2};  // an over-weighted token (p_d = 0.49 > p_t = 0.48)
    spec.rows = log_rows({{0.49, 0.49, 0.01, 0.01}});
    const VerificationOutcome o = engine().verify_rows(target, spec, SamplingScheme::standard(),
                                                       SamplingScheme::standard(), std::uint64_t(900000 + i));
    if (o.accepted == 0) {
      ++rejected;
      CHECK((o.bonus == 2 || o.bonus == 3));
      bonus_two += o.bonus == 2;
    }
  }
  REQUIRE(rejected >= 100);
  const double f = double(bonus_two) / rejected;
  CHECK(std::abs(f - 0.5) < 4.0 * std::sqrt(0.25 / rejected));
}

TEST_CASE("one-hot target equal to one-hot draft accepts everything") {
  const std::vector<float> target = log_rows({{0, 0, 0, 1.0}, {1.0, 0, 0, 0}, {0, 1.0, 0, 0}, {0, 0, 1.0, 0}});
  Speculation spec;
  spec.tokens = {3, 0, 1};
  spec.rows = log_rows({{0, 0, 0, 1.0}, {1.0, 0, 0, 0}, {0, 1.0, 0, 0}});
  const VerificationOutcome o = engine().verify_rows(target, spec, SamplingScheme::standard(),
                                                     SamplingScheme::standard(), 10);
  CHECK(o.accepted == 3);
  CHECK(o.bonus == 2);  // emitted {3, 0, 1, 2}
}

TEST_CASE("emitted length is always accepted plus one") {
  Stream rng(13);
  const std::vector<int> ctx = ctx_of(6, 12);
  for (int i = 0; i < 12; ++i) {
    const Speculation spec = engine().draft(ctx, 4, SamplingScheme::standard(), rng);
    const RoundResult r = engine().verify(ctx, spec, rng, SamplingScheme::standard());
    CHECK(r.emitted.size() == size_t(r.outcome.accepted) + 1);
    CHECK(r.emitted.back() == r.outcome.bonus);
    for (int j = 0; j < r.outcome.accepted; ++j) CHECK(r.emitted[size_t(j)] == spec.tokens[size_t(j)]);
  }
}

// -------------------------------------------------------------- test_cache.cpp

TEST_CASE("build_cache excludes the token sent for verification") {
  // restated: the drafted token is the draft's argmax at the context; the
  // position-0 candidates are exactly the next two in (value desc, index asc)
  const std::vector<int> ctx = ctx_of(8, 43);
  Stream rng(44);
  const Speculation spec = engine().draft(ctx, 1, SamplingScheme::greedy(), rng);
  const std::vector<int> order = ranked(engine().logits(1, ctx), spec.tokens[0]);
  const SpeculationCache built =
      engine().build_cache(ctx, spec, FanOutPlan{{2, 0}, Origin::Primary, 2}, SamplingScheme::greedy(), 1, rng);
  CHECK(built.size() == 2);
  CHECK(built.lookup({0, order[0]}) != nullptr);
  CHECK(built.lookup({0, order[1]}) != nullptr);
  CHECK(built.lookup({0, spec.tokens[0]}) == nullptr);  // excluded sampled token
  CHECK(built.lookup({0, order[2]}) == nullptr);
}

TEST_CASE("build_cache entry count equals the plan total") {
  Stream seeds(45);
  for (int trial = 0; trial < 12; ++trial) {
    const int lookahead = 1 + int(seeds.next_uniform() * 3);
    std::vector<int> fan(size_t(lookahead) + 1);
    int total = 0;
    for (int k = 0; k <= lookahead; ++k) {
      fan[size_t(k)] = int(seeds.next_uniform() * 6);
      total += fan[size_t(k)];
    }
    Stream rng(seeds.next_u64());
    const std::vector<int> ctx{trial % 12 + 1, 5};
    const Speculation spec = engine().draft(ctx, lookahead, SamplingScheme::standard(), rng);
    const SpeculationCache built = engine().build_cache(ctx, spec, FanOutPlan{fan, Origin::Primary, total},
                                                        SamplingScheme::standard(), lookahead, rng);
    CHECK(built.size() == size_t(total));
  }
}

TEST_CASE("lookup returns exactly the stored speculation") {
  Stream rng(48);
  const std::vector<int> ctx{3, 17, 9};
  const Speculation spec = engine().draft(ctx, 2, SamplingScheme::standard(), rng);
  const SpeculationCache built = engine().build_cache(ctx, spec, FanOutPlan{{3, 3, 3}, Origin::Primary, 9},
                                                      SamplingScheme::standard(), 2, rng);
  CHECK(built.size() == 9);
  for (const auto& [outcome, stored] : built.entries()) {
    const Speculation* found = built.lookup(outcome);
    REQUIRE(found != nullptr);
    CHECK(found->tokens == stored.tokens);
    CHECK(found->rows == stored.rows);
    CHECK(found->rows.size() == size_t(2) * V);
    CHECK(found->origin == Origin::Primary);
  }
  CHECK(built.lookup({7, 0}) == nullptr);
}

TEST_CASE("rejected bonus never equals the excluded token") {
  Stream rng(51);
  const std::vector<int> ctx = ctx_of(5, 49);
  int rejections = 0;
  for (int i = 0; i < 60; ++i) {
    const Speculation spec = engine().draft(ctx, 3, SamplingScheme::standard(), rng);
    const RoundResult r = engine().verify(ctx, spec, rng, SamplingScheme::standard());
    if (r.outcome.accepted < 3) {
      ++rejections;
      CHECK(r.outcome.bonus != spec.tokens[size_t(r.outcome.accepted)]);
    }
  }
  CHECK(rejections > 5);
}

TEST_CASE("asynchronous pre-speculation equals build_cache (device session)") {
  // not a reference case: SURVEY §8b's device-side form of build_cache must
  // agree with the synchronous call given the same stream
  const std::vector<int> ctx = ctx_of(9, 77);
  Stream a(5), b(5);
  const Speculation spec = engine().draft(ctx, 4, SamplingScheme::greedy(), a);
  Stream c1(99), c2(99);
  const FanOutPlan plan{{4, 4, 4, 4, 4}, Origin::Primary, 20};
  const SpeculationCache sync = engine().build_cache(ctx, spec, plan, SamplingScheme::greedy(), 4, c1);
  int32_t* dctx = nullptr;
  int32_t* dspec = nullptr;
  REQUIRE(ssd_b200_test_alloc(&dctx, ctx) == 0);
  REQUIRE(ssd_b200_test_alloc(&dspec, spec.tokens) == 0);
  engine().prespec_begin(dctx, int(ctx.size()), dspec, 4, plan, SamplingScheme::greedy(), 4, c2);
  CHECK(c1.next_u64() == c2.next_u64());
  const std::vector<VerificationOutcome> keys = engine().cache_keys();
  CHECK(keys.size() == sync.size());
  for (size_t i = 0; i < keys.size(); ++i) {
    CHECK(engine().cache_lookup(keys[i]) == int(i));
    const Speculation* s = sync.lookup(keys[i]);
    REQUIRE(s != nullptr);
    CHECK(engine().cache_entry(int(i), 4).tokens == s->tokens);
  }
  ssd_b200_test_free(dctx);
  ssd_b200_test_free(dspec);
}

DOCTEST_SHIM_MAIN
