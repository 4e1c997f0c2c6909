// TEST INFRASTRUCTURE ONLY — CPU oracle for the Saguaro SSD hot path.
//
// This header declares a from-scratch restatement of the reference
// (ssd-lab, /root/reference/proj) speculator / verifier / speculation-cache
// logic. Nothing in the product (paper_2603_03251_b200/) links or calls it;
// only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs use it, as the checker and the CPU baseline.
//
// Differences from the reference, all deliberate:
//   * the model parameter is widened from the concrete lm::SyntheticLM to the
//     LanguageModel interface below (SURVEY §8b "Model parameter"), so the
//     same loops drive the Markov tables AND the CPU transformer oracle;
//   * temperature 0 is accepted and means greedy (the tau->0 limit: one-hot
//     at the top_indices(z,1) token, lowest index on ties).
//     The reference throws for temperature <= 0 (categorical.cpp:51,66-68).
//
// Parity: pinned bit-exact against the compiled reference (oracle/_ref) on
// its own Markov models — streams, counters, keys — see tests/golden/ and
// tests/test_oracle_golden.py.
#pragma once

#include <cstdint>
#include <memory>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace oracle {

// ---------------------------------------------------------------- errors
// One class per ssdlab::Error subclass (reference errors.hpp:9-61).
struct Error : std::runtime_error { using std::runtime_error::runtime_error; virtual int code() const { return 1; } };
#define ORACLE_ERR(name, c) \
  struct name : Error { using Error::Error; int code() const override { return c; } };
ORACLE_ERR(AllZeroError, 2)
ORACLE_ERR(DegenerateResidualError, 3)
ORACLE_ERR(TooLargeError, 4)
ORACLE_ERR(BudgetTooSmallError, 5)
ORACLE_ERR(DivergentError, 6)
ORACLE_ERR(InsufficientDataError, 7)
ORACLE_ERR(UnreachableError, 8)
ORACLE_ERR(NoCrossoverError, 9)
ORACLE_ERR(ProtocolViolationError, 10)
ORACLE_ERR(ConfigError, 11)
#undef ORACLE_ERR

// ---------------------------------------------------------------- rng
// reference rng.hpp:9-48: splitmix64 finaliser, seed split, mt19937_64 with
// 53-bit uniforms (one engine step per draw).
std::uint64_t mix64(std::uint64_t x);
std::uint64_t child_seed(std::uint64_t root, std::uint64_t index);

class Rng {
 public:
  explicit Rng(std::uint64_t seed) : mt_(seed) {}
  std::uint64_t bits() { return mt_(); }
  double unit() { return double(mt_() >> 11) * 0x1.0p-53; }
  std::mt19937_64& engine() { return mt_; }
 private:
  std::mt19937_64 mt_;
};

// ---------------------------------------------------------------- dist
using Row = std::vector<double>;

struct Scheme {               // reference categorical.hpp:43-60
  bool saguaro = false;
  double temperature = 1.0;   // 0 => greedy (oracle extension)
  int fan_out = 0;
  double downweight = 1.0;
};

std::vector<int> rank_tokens(std::span<const double> z, int count);  // top_indices
Row normalized(std::span<const double> w);                           // normalize
Row scheme_probs(std::span<const double> z, const Scheme& s);         // softmax/apply_scheme
Row residual_probs(std::span<const double> pt, std::span<const double> pd);
double accept_mass(std::span<const double> pt, std::span<const double> pd);  // acceptance_rate
int draw(std::span<const double> p, Rng& rng);                       // sample

// ---------------------------------------------------------------- model seam
// "Any LM that yields a logit row for a context".
class LanguageModel {
 public:
  virtual ~LanguageModel() = default;
  virtual int vocab() const = 0;
  // Logit row for the next token after `context`. The returned span stays
  // valid until the next call on this object.
  virtual std::span<const double> logits(std::span<const int> context) = 0;
  // Minimum context the model needs (Markov order); histories start with
  // this many zeros (reference sim.cpp:143, 233).
  virtual int history_pad() const { return 0; }
};

// ---------------------------------------------------------------- specdec
enum class Origin { Primary = 0, Backup = 1 };

struct Spec {                 // reference specdec.hpp:22-28
  std::vector<int> tokens;
  std::vector<Row> dists;
  Origin origin = Origin::Primary;
  int K() const { return int(tokens.size()); }
};

struct Outcome {              // (accepted, bonus): the cache key
  int k = 0;
  int t = 0;
  bool operator==(const Outcome& o) const { return k == o.k && t == o.t; }
};

struct Round {
  Outcome key;
  std::vector<int> emitted;
};

Spec draft_tokens(LanguageModel& lm, std::span<const int> ctx, int K, const Scheme& s,
                  Rng& rng, Origin origin = Origin::Primary);

struct VerifyOpts {
  Scheme target_scheme;       // default standard(1.0)
  double accept_scale = 1.0;  // negative-control fixture (specdec.hpp:63-69)
};

Round verify_spec(LanguageModel& target, std::span<const int> ctx, const Spec& spec,
                  Rng& rng, const VerifyOpts& o = {});

double expected_tokens(double alpha, int K);

// ---------------------------------------------------------------- cache
struct Plan {                 // reference cache.hpp:18-25
  std::vector<int> fan;
  Origin role = Origin::Primary;
  int budget = 0;
  int K() const { return int(fan.size()) - 1; }
  int total() const { int s = 0; for (int f : fan) s += f; return s; }
};

std::vector<double> geometric_plan_continuous(double a, double r, int K, double budget);
Plan geometric_plan(double a, double r, int K, int budget, Origin role = Origin::Primary);
Plan uniform_plan(int K, int budget, Origin role = Origin::Primary);
double plan_hit_rate(std::span<const int> fan, double a, double r);

// ---------------------------------------------------------------- perf
// reference perf.hpp:7-80 / perf.cpp:19-73: the latency model of the loop
// and the batch-size crossover of the two backup strategies.
struct Yields { double hit = 1.0, miss = 1.0; };
double speedup_ssd(double p, const Yields& y, double tp, double tb);
double speedup_batch(double p, const Yields& y, double tp, double tb, double batch);
double critical_batch(double p, const Yields& y, double tp);

// hitmodel.cpp:65-106: log-log least squares of miss = A F^-r.
struct PowerLaw { double exponent = 0.0, log_amplitude = 0.0, r_squared = 1.0; };
PowerLaw fit_powerlaw(const std::vector<std::pair<double, double>>& samples);

struct CacheEntry {
  Outcome key;
  Spec spec;
};

// Insertion order = entry ordinal (k ascending, candidate rank ascending);
// this is also the order of the derived entry streams (cache.cpp:245,264).
struct SpecCache {
  std::vector<CacheEntry> entries;
  Origin round_origin = Origin::Primary;
  const Spec* find(const Outcome& o) const {
    for (const auto& e : entries) if (e.key == o) return &e.spec;
    return nullptr;
  }
};

SpecCache prespeculate(LanguageModel& draft_lm, std::span<const int> ctx, const Spec& inflight,
                       const Plan& plan, const Scheme& s, int next_K, Rng& rng);

// ---------------------------------------------------------------- sim
enum class Backup { SamePrimaryJIT = 0, FastRandom = 1 };

struct SimCfg {               // reference sim.hpp:28-53
  LanguageModel* target = nullptr;
  LanguageModel* draft = nullptr;
  int K = 4;
  Scheme scheme;
  Scheme target_scheme;
  Plan primary_plan, backup_plan;
  double primary_time = 0.3, backup_time_fast = 0.0;
  Backup backup = Backup::FastRandom;
  bool synthetic_iid = false;
  double synthetic_hit_rate = 0.0;
  int batch = 1;
  long rounds = 1000;
  std::uint64_t seed = 0;
  double accept_scale = 1.0;
  bool keep_streams = true;
  // Initial history. Empty => history_pad() zeros, as the reference does
  // (sim.cpp:143); the transformer oracle needs a real prompt.
  std::vector<int> prompt;
  double backup_time() const { return backup == Backup::SamePrimaryJIT ? primary_time : backup_time_fast; }
};

struct LookupEvent { bool primary_origin; bool hit; };

struct Stats {                // reference sim.hpp:55-104
  long rounds = 0;
  int batch = 1;
  long tokens = 0;
  double vtime = 0.0;
  long p_lookups = 0, p_hits = 0, b_lookups = 0, b_hits = 0;
  long hit_rounds = 0, miss_rounds = 0, initial_rounds = 0;
  long hit_round_tokens = 0, miss_round_tokens = 0;
  double accepted_sum = 0.0;
  std::vector<std::vector<int>> streams;
  std::vector<LookupEvent> log;
};

Stats sim_ar(LanguageModel& target, const Scheme& ts, long tokens, std::uint64_t seed,
             const std::vector<int>& prompt = {});
Stats sim_sd(const SimCfg& c);
Stats sim_ssd(const SimCfg& c);   // run_ssd_batch semantics (batch >= 1)

struct Message { long round; std::string dir; std::string summary; double vclock; };
struct Timing { double verify_start, verify_end, cache_ready; bool all_hit; };
struct HarnessOut {
  std::vector<Message> transcript;
  Stats stats;
  std::vector<Timing> timings;
  // Per-round (k, t*) and hit bits of sequence 0, for GPU parity.
  std::vector<Outcome> outcomes0;
  std::vector<int> hits0;
  double decode_seconds = 0.0;  // wall time of the rounds (bench CPU baseline)
};
HarnessOut sim_harness(const SimCfg& c);

Spec uniform_spec(int V, int K, Rng& rng);   // sim.cpp:35-48 (FastRandom)

// ---------------------------------------------------------------- Markov LM
// Restatement of lm::SyntheticLM (lm.hpp / lm.cpp).
class MarkovLM : public LanguageModel {
 public:
  MarkovLM(int V, int order, std::uint64_t seed, std::vector<Row> rows);
  int vocab() const override { return V_; }
  int order() const { return m_; }
  int history_pad() const override { return m_; }
  std::uint64_t seed() const { return seed_; }
  const std::vector<Row>& rows() const { return rows_; }
  std::size_t row_of(std::span<const int> ctx) const;
  std::span<const double> logits(std::span<const int> ctx) override;
 private:
  int V_, m_;
  std::uint64_t seed_;
  std::vector<Row> rows_;
};

MarkovLM markov_make(int V, int order, double concentration, std::uint64_t seed);
MarkovLM markov_mix_draft(const MarkovLM& target, double eps, std::uint64_t noise_seed);
double markov_mean_acceptance(const MarkovLM& t, const MarkovLM& d, const Scheme& ts,
                              const Scheme& ds);
struct MarkovPair { MarkovLM draft; double eps; };
MarkovPair markov_calibrate(const MarkovLM& target, double alpha_goal, std::uint64_t seed);

}  // namespace oracle
