// TEST INFRASTRUCTURE ONLY — see ssd_oracle.hpp.
//
// CPU restatement of the reference's hot-path algorithms. Every function
// names the reference file:line it follows (paths relative to
// /root/reference/proj). Floating-point operation order is kept identical to
// the reference wherever it affects bits (sums in index order, exp of the
// shifted scaled logit, division by the running total), because the
// restatement is pinned bit-exact against the compiled reference.
#include "ssd_oracle.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <numeric>

namespace oracle {

// ============================================================== rng
// rng.hpp:9-14
std::uint64_t mix64(std::uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
// rng.hpp:24-26
std::uint64_t child_seed(std::uint64_t root, std::uint64_t index) {
  return mix64(root + (index + 1) * 0x9E3779B97F4A7C15ull);
}

// ============================================================== dist
// categorical.cpp:35-48 — indices of the `count` largest values, ties to the
// lowest index. A stable sort on the index-ordered list with a strict
// "greater" comparator yields exactly the (value desc, index asc) order.
std::vector<int> rank_tokens(std::span<const double> z, int count) {
  const int n = int(z.size());
  if (count < 0 || count > n) throw Error("top_indices: count out of range");
  std::vector<int> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  if (count < n / 4) {
    std::partial_sort(idx.begin(), idx.begin() + count, idx.end(), [&](int a, int b) {
      return z[a] != z[b] ? z[a] > z[b] : a < b;
    });
  } else {
    std::stable_sort(idx.begin(), idx.end(), [&](int a, int b) { return z[a] > z[b]; });
  }
  idx.resize(count);
  return idx;
}

// categorical.cpp:18-33
Row normalized(std::span<const double> w) {
  double s = 0.0;
  for (double x : w) {
    if (!(x >= 0.0) || !std::isfinite(x)) throw Error("normalize: weights must be finite and nonnegative");
    s += x;
  }
  if (s <= 0.0) throw AllZeroError("normalize: all weights are zero");
  Row out(w.size());
  for (std::size_t i = 0; i < w.size(); ++i) out[i] = w[i] / s;
  return out;
}

namespace {
Row one_hot(std::size_t n, int at) {
  Row r(n, 0.0);
  r[std::size_t(at)] = 1.0;
  return r;
}
}  // namespace

// categorical.cpp:50-92 (softmax and apply_scheme share the exp pass: the
// weight of token i is exp(z_i / tau - max_j z_j / tau)).
Row scheme_probs(std::span<const double> z, const Scheme& s) {
  if (z.empty()) throw Error("softmax: empty logits");
  if (s.saguaro) {
    if (s.fan_out < 1 || s.fan_out > int(z.size())) throw Error("apply_scheme: fan_out out of range");
    if (!(s.downweight >= 0.0) || !(s.downweight <= 1.0)) throw Error("apply_scheme: downweight must be in [0, 1]");
  }
  if (s.temperature == 0.0) {
    // Greedy: the tau -> 0 limit. Down-weighting by C > 0 cannot move the
    // argmax; C == 0 removes the top-F set, leaving rank F.
    for (double v : z) if (!std::isfinite(v)) throw Error("apply_scheme: logits must be finite");
    const int pick_rank = (s.saguaro && s.downweight == 0.0) ? s.fan_out : 0;
    if (pick_rank >= int(z.size())) throw AllZeroError("normalize: all weights are zero");
    return one_hot(z.size(), rank_tokens(z, pick_rank + 1)[std::size_t(pick_rank)]);
  }
  if (!(s.temperature > 0.0)) throw Error("apply_scheme: temperature must be > 0");
  double hi = -HUGE_VAL;
  for (double v : z) {
    if (!std::isfinite(v)) throw Error("softmax: logits must be finite");
    hi = std::max(hi, v / s.temperature);
  }
  Row w(z.size());
  for (std::size_t i = 0; i < z.size(); ++i) w[i] = std::exp(z[i] / s.temperature - hi);
  if (s.saguaro) {
    for (int t : rank_tokens(z, s.fan_out)) w[std::size_t(t)] *= s.downweight;
  }
  return normalized(w);
}

// categorical.cpp:94-110
Row residual_probs(std::span<const double> pt, std::span<const double> pd) {
  if (pt.size() != pd.size()) throw Error("residual: length mismatch");
  Row r(pt.size());
  double mass = 0.0;
  for (std::size_t i = 0; i < r.size(); ++i) {
    r[i] = std::max(pt[i] - pd[i], 0.0);
    mass += r[i];
  }
  if (mass <= 0.0) throw DegenerateResidualError("residual: zero positive mass (draft equals target)");
  for (double& v : r) v /= mass;
  return r;
}

// categorical.cpp:112-127
double accept_mass(std::span<const double> pt, std::span<const double> pd) {
  if (pt.size() != pd.size()) throw Error("acceptance_rate: length mismatch");
  double lo = 0.0, l1 = 0.0;
  for (std::size_t i = 0; i < pt.size(); ++i) {
    lo += std::min(pt[i], pd[i]);
    l1 += std::abs(pt[i] - pd[i]);
  }
  if (std::abs(lo - (1.0 - 0.5 * l1)) > 1e-12) throw Error("acceptance_rate: min-sum and L1 routes disagree");
  return lo;
}

// categorical.cpp:129-143 — inverse CDF with one uniform.
int draw(std::span<const double> p, Rng& rng) {
  const double u = rng.unit();
  double cdf = 0.0;
  int last = -1;
  for (int i = 0; i < int(p.size()); ++i) {
    if (p[i] > 0.0) last = i;
    cdf += p[i];
    if (u < cdf) return i;
  }
  if (last < 0) throw AllZeroError("sample: zero-mass distribution");
  return last;
}

// ============================================================== specdec
// specdec.cpp:8-25 — K autoregressive draws, recording each post-scheme law.
Spec draft_tokens(LanguageModel& lm, std::span<const int> ctx, int K, const Scheme& s,
                  Rng& rng, Origin origin) {
  if (K < 1) throw Error("draft: lookahead must be >= 1");
  Spec out;
  out.origin = origin;
  std::vector<int> seq(ctx.begin(), ctx.end());
  for (int i = 0; i < K; ++i) {
    Row p = scheme_probs(lm.logits(seq), s);
    const int tok = draw(p, rng);
    out.tokens.push_back(tok);
    out.dists.push_back(std::move(p));
    seq.push_back(tok);
  }
  return out;
}

// specdec.cpp:27-69 — sequential accept tests, residual bonus on the first
// rejection, target bonus at K+1 when everything is accepted.
Round verify_spec(LanguageModel& target, std::span<const int> ctx, const Spec& spec, Rng& rng,
                  const VerifyOpts& o) {
  const int K = spec.K();
  if (K < 1) throw Error("verify: empty speculation");
  if (spec.dists.size() != spec.tokens.size()) throw Error("verify: tokens and draft_dists length mismatch");
  std::vector<int> seq(ctx.begin(), ctx.end());
  Round r;
  for (int i = 0; i < K; ++i) {
    const Row pt = scheme_probs(target.logits(seq), o.target_scheme);
    const Row& pd = spec.dists[std::size_t(i)];
    const int x = spec.tokens[std::size_t(i)];
    const double q = pd[std::size_t(x)];
    if (!(q > 0.0)) throw Error("verify: drafted token has zero draft probability");
    double a = std::min(1.0, pt[std::size_t(x)] / q);
    a = std::min(1.0, a * o.accept_scale);
    if (rng.unit() < a) {
      seq.push_back(x);
      r.emitted.push_back(x);
      continue;
    }
    r.key.k = i;
    r.key.t = draw(residual_probs(pt, pd), rng);
    r.emitted.push_back(r.key.t);
    return r;
  }
  const Row pt = scheme_probs(target.logits(seq), o.target_scheme);
  r.key.k = K;
  r.key.t = draw(pt, rng);
  r.emitted = spec.tokens;
  r.emitted.push_back(r.key.t);
  return r;
}

// specdec.cpp:230-237
double expected_tokens(double alpha, int K) {
  if (K < 1) throw Error("expected_tokens: lookahead must be >= 1");
  if (!(alpha >= 0.0) || !(alpha <= 1.0)) throw Error("expected_tokens: alpha must be in [0, 1]");
  if (alpha == 1.0) return double(K + 1);
  return (1.0 - std::pow(alpha, K + 1)) / (1.0 - alpha);
}

// ============================================================== cache plans
// cache.cpp:150-169 — capped-geometric weights times power-law hit.
double plan_hit_rate(std::span<const int> fan, double a, double r) {
  const int K = int(fan.size()) - 1;
  if (K < 0) throw Error("conditional_hit_rate: empty plan");
  if (!(a >= 0.0) || !(a <= 1.0)) throw Error("conditional_hit_rate: acceptance must be in [0, 1]");
  auto hit_at = [&](int f) { return f >= 1 ? 1.0 - std::pow(double(f), -r) : 0.0; };
  double total = 0.0, w = 1.0;
  for (int k = 0; k < K; ++k) {
    total += w * (1.0 - a) * hit_at(fan[std::size_t(k)]);
    w *= a;
  }
  return total + w * hit_at(fan[std::size_t(K)]);
}

// cache.cpp:13-37
std::vector<double> geometric_plan_continuous(double a, double r, int K, double budget) {
  if (!(a > 0.0) || !(a < 1.0)) throw Error("geometric_fanout: acceptance must be in (0, 1)");
  if (!(r > 0.0)) throw Error("geometric_fanout: exponent must be > 0");
  if (K < 1) throw Error("geometric_fanout: lookahead must be >= 1");
  if (!(budget > 0.0)) throw Error("geometric_fanout: budget must be > 0");
  const double q = std::pow(a, 1.0 / (1.0 + r));
  const double cap = std::pow(a, K / (1.0 + r)) * std::pow(1.0 - a, -1.0 / (1.0 + r));
  const double geo = (1.0 - std::pow(q, K)) / (1.0 - q);
  const double f0 = budget / (cap + geo);
  std::vector<double> f(std::size_t(K) + 1);
  for (int k = 0; k < K; ++k) f[std::size_t(k)] = f0 * std::pow(q, k);
  f[std::size_t(K)] = f0 * cap;
  return f;
}

// cache.cpp:39-113 — largest-remainder rounding, min-1 floor, exchange polish.
Plan geometric_plan(double a, double r, int K, int budget, Origin role) {
  if (budget < K + 1) throw BudgetTooSmallError("geometric_fanout: budget must be at least lookahead + 1");
  const std::vector<double> cont = geometric_plan_continuous(a, r, K, budget);
  const std::size_t n = cont.size();
  std::vector<int> f(n);
  std::vector<double> frac(n);
  int used = 0;
  for (std::size_t k = 0; k < n; ++k) {
    f[k] = int(std::floor(cont[k]));
    frac[k] = cont[k] - f[k];
    used += f[k];
  }
  std::vector<std::size_t> by_frac(n);
  std::iota(by_frac.begin(), by_frac.end(), std::size_t(0));
  std::stable_sort(by_frac.begin(), by_frac.end(),
                   [&](std::size_t x, std::size_t y) { return frac[x] > frac[y]; });
  for (std::size_t i = 0; used < budget; ++i, ++used) f[by_frac[i % n]] += 1;
  for (std::size_t k = 0; k < n; ++k) {
    while (f[k] < 1) {
      std::size_t big = 0;
      for (std::size_t j = 1; j < n; ++j) if (f[j] > f[big]) big = j;
      if (f[big] <= 1) throw BudgetTooSmallError("geometric_fanout: cannot satisfy minimum");
      f[big] -= 1;
      f[k] += 1;
    }
  }
  for (;;) {
    double best = plan_hit_rate(f, a, r);
    std::size_t bf = 0, bt = 0;
    bool better = false;
    for (std::size_t from = 0; from < n; ++from) {
      if (f[from] <= 1) continue;
      for (std::size_t to = 0; to < n; ++to) {
        if (to == from) continue;
        f[from] -= 1; f[to] += 1;
        const double v = plan_hit_rate(f, a, r);
        f[from] += 1; f[to] -= 1;
        if (v > best + 1e-15) { best = v; bf = from; bt = to; better = true; }
      }
    }
    if (!better) break;
    f[bf] -= 1;
    f[bt] += 1;
  }
  return Plan{std::move(f), role, budget};
}

// cache.cpp:115-127
Plan uniform_plan(int K, int budget, Origin role) {
  if (K < 1) throw Error("uniform_fanout: lookahead must be >= 1");
  if (budget < K + 1) throw BudgetTooSmallError("uniform_fanout: budget must be at least lookahead + 1");
  const int n = K + 1;
  std::vector<int> f(std::size_t(n), budget / n);
  for (int k = 0; k < budget % n; ++k) f[std::size_t(k)] += 1;
  return Plan{std::move(f), role, budget};
}

// ============================================================== build_cache
// cache.cpp:232-277. Row k ranks the draft logits at ctx ++ s_1..s_k; for
// k < K the in-flight token s_{k+1} is skipped; each of the first F_k
// remaining candidates gets a fresh primary speculation drawn from stream
// child_seed(base, ordinal), base being ONE draw from the caller's stream.
SpecCache prespeculate(LanguageModel& lm, std::span<const int> ctx, const Spec& inflight,
                       const Plan& plan, const Scheme& s, int next_K, Rng& rng) {
  const int K = inflight.K();
  if (plan.K() != K) throw Error("build_cache: plan length does not match speculation");
  if (plan.role != inflight.origin) throw Error("build_cache: plan role does not match speculation origin");
  const std::uint64_t base = rng.bits();
  SpecCache cache;
  cache.round_origin = inflight.origin;
  std::vector<int> prefix(ctx.begin(), ctx.end());
  std::uint64_t ordinal = 0;
  for (int k = 0; k <= K; ++k) {
    const int want = plan.fan[std::size_t(k)];
    if (want > 0) {
      // Copy the row: the nested drafts below reuse the model's buffer.
      const std::span<const double> zs = lm.logits(prefix);
      const Row z(zs.begin(), zs.end());
      const int skip = k < K ? inflight.tokens[std::size_t(k)] : -1;
      // want + 1 ranked tokens always contain want candidates != skip.
      const int need = std::min(int(z.size()), want + 1);
      int got = 0;
      for (int cand : rank_tokens(z, need)) {
        if (cand == skip) continue;
        if (got == want) break;
        ++got;
        std::vector<int> cont = prefix;
        cont.push_back(cand);
        Rng entry(child_seed(base, ordinal++));
        cache.entries.push_back({Outcome{k, cand}, draft_tokens(lm, cont, next_K, s, entry, Origin::Primary)});
      }
    }
    if (k < K) prefix.push_back(inflight.tokens[std::size_t(k)]);
  }
  return cache;
}

// ============================================================== sim
// sim.cpp:35-48 — FastRandom backup: K draws from the exact uniform vector.
Spec uniform_spec(int V, int K, Rng& rng) {
  Spec s;
  s.origin = Origin::Backup;
  const Row u(std::size_t(V), 1.0 / V);
  for (int i = 0; i < K; ++i) {
    s.tokens.push_back(draw(u, rng));
    s.dists.push_back(u);
  }
  return s;
}

namespace {

std::span<const int> last_n(const std::vector<int>& h, int n) {
  return std::span<const int>(h).last(std::size_t(n));
}

// sim.cpp:17-33
void check_cfg(const SimCfg& c) {
  if (!c.target || !c.draft) throw Error("sim: target and draft models are required");
  if (c.target->vocab() != c.draft->vocab() || c.target->history_pad() != c.draft->history_pad())
    throw Error("sim: target and draft shapes differ");
  if (c.K < 1) throw Error("sim: lookahead must be >= 1");
  if (c.rounds < 1) throw Error("sim: rounds must be >= 1");
  if (c.batch < 1) throw Error("sim: batch_size must be >= 1");
  if (c.synthetic_iid && (!(c.synthetic_hit_rate >= 0.0) || !(c.synthetic_hit_rate <= 1.0)))
    throw Error("sim: synthetic_hit_rate must be in [0, 1]");
}

// Context handed to the models: the Markov tables only read their order;
// the transformer oracle reads the whole (unpadded) history.
std::span<const int> model_ctx(const std::vector<int>& h, LanguageModel& lm) {
  const int pad = lm.history_pad();
  if (pad > 0) return last_n(h, pad);
  return std::span<const int>(h);
}

enum class Src { Initial, Hit, Backup };

std::vector<int> start_history(const std::vector<int>& prompt, const LanguageModel& lm) {
  if (!prompt.empty()) return prompt;
  return std::vector<int>(std::size_t(lm.history_pad()), 0);
}

}  // namespace

// sim.cpp:64-86
Stats sim_ar(LanguageModel& target, const Scheme& ts, long tokens, std::uint64_t seed,
             const std::vector<int>& prompt) {
  if (tokens < 1) throw Error("run_ar: tokens must be >= 1");
  Rng rng(child_seed(seed, 0));
  std::vector<int> h = start_history(prompt, target);
  Stats st;
  st.rounds = tokens;
  st.streams.resize(1);
  for (long i = 0; i < tokens; ++i) {
    const int tok = draw(scheme_probs(target.logits(model_ctx(h, target)), ts), rng);
    h.push_back(tok);
    st.streams[0].push_back(tok);
  }
  st.tokens = tokens;
  st.vtime = double(tokens);
  return st;
}

// sim.cpp:88-121
Stats sim_sd(const SimCfg& c) {
  check_cfg(c);
  if (c.batch != 1) throw Error("run_sd: batch_size must be 1");
  Rng rng(child_seed(c.seed, 0));
  std::vector<int> h = start_history(c.prompt, *c.target);
  Stats st;
  st.rounds = c.rounds;
  st.streams.resize(1);
  const VerifyOpts vo{c.target_scheme, c.accept_scale};
  for (long r = 0; r < c.rounds; ++r) {
    const Spec s = draft_tokens(*c.draft, model_ctx(h, *c.draft), c.K, c.scheme, rng);
    const Round res = verify_spec(*c.target, model_ctx(h, *c.target), s, rng, vo);
    st.tokens += long(res.emitted.size());
    st.accepted_sum += res.key.k;
    h.insert(h.end(), res.emitted.begin(), res.emitted.end());
    if (c.keep_streams) st.streams[0].insert(st.streams[0].end(), res.emitted.begin(), res.emitted.end());
  }
  st.vtime = double(c.rounds) * (1.0 + c.primary_time);
  return st;
}

// sim.cpp:128-250 — the SSD round loop (sequential virtual-clock version).
Stats sim_ssd(const SimCfg& c) {
  check_cfg(c);
  const int B = c.batch, K = c.K;
  const VerifyOpts vo{c.target_scheme, c.accept_scale};
  struct Seq { Rng rng; std::vector<int> h; Spec spec; Src src; };
  std::vector<Seq> seqs;
  for (int j = 0; j < B; ++j) {
    Seq s{Rng(child_seed(c.seed, std::uint64_t(j))), start_history(c.prompt, *c.target), {}, Src::Initial};
    s.spec = draft_tokens(*c.draft, model_ctx(s.h, *c.draft), K, c.scheme, s.rng, Origin::Primary);
    seqs.push_back(std::move(s));
  }
  Stats st;
  st.rounds = c.rounds;
  st.batch = B;
  st.streams.resize(std::size_t(B));
  st.vtime = 1.0 + c.primary_time;
  bool prev_all_hit = true;
  for (long round = 1; round <= c.rounds; ++round) {
    if (round > 1) st.vtime += prev_all_hit ? std::max(1.0, c.primary_time) : 1.0 + c.backup_time();
    bool all_hit = true;
    for (int j = 0; j < B; ++j) {
      Seq& s = seqs[std::size_t(j)];
      const Round res = verify_spec(*c.target, model_ctx(s.h, *c.target), s.spec, s.rng, vo);
      const long n = long(res.emitted.size());
      st.tokens += n;
      st.accepted_sum += res.key.k;
      if (s.src == Src::Initial) ++st.initial_rounds;
      else if (s.src == Src::Hit) { ++st.hit_rounds; st.hit_round_tokens += n; }
      else { ++st.miss_rounds; st.miss_round_tokens += n; }

      if (round < c.rounds) {
        bool hit = false;
        Spec next;
        if (c.synthetic_iid) {
          hit = s.rng.unit() < c.synthetic_hit_rate;
        } else {
          const Plan& plan = s.spec.origin == Origin::Primary ? c.primary_plan : c.backup_plan;
          const SpecCache cache = prespeculate(*c.draft, model_ctx(s.h, *c.draft), s.spec, plan, c.scheme, K, s.rng);
          if (const Spec* f = cache.find(res.key)) { hit = true; next = *f; }
        }
        const bool from_primary = s.spec.origin == Origin::Primary;
        (from_primary ? st.p_lookups : st.b_lookups) += 1;
        (from_primary ? st.p_hits : st.b_hits) += hit ? 1 : 0;
        st.log.push_back({from_primary, hit});
        s.h.insert(s.h.end(), res.emitted.begin(), res.emitted.end());
        if (hit) {
          if (c.synthetic_iid) next = draft_tokens(*c.draft, model_ctx(s.h, *c.draft), K, c.scheme, s.rng, Origin::Primary);
          next.origin = Origin::Primary;
          s.spec = std::move(next);
          s.src = Src::Hit;
        } else {
          all_hit = false;
          s.spec = c.backup == Backup::SamePrimaryJIT
                       ? draft_tokens(*c.draft, model_ctx(s.h, *c.draft), K, c.scheme, s.rng, Origin::Backup)
                       : uniform_spec(c.target->vocab(), K, s.rng);
          s.src = Src::Backup;
        }
      } else {
        s.h.insert(s.h.end(), res.emitted.begin(), res.emitted.end());
      }
      if (c.keep_streams) {
        auto& out = st.streams[std::size_t(j)];
        out.insert(out.end(), res.emitted.begin(), res.emitted.end());
      }
    }
    prev_all_hit = all_hit;
  }
  return st;
}

// ============================================================== harness
// sim.cpp:258-601 — the two logical processes. The draft side owns the
// caches and its own streams child_seed(seed, j); the verifier side owns the
// target and streams child_seed(child_seed(seed, 0x5EED), j); they exchange
// exactly one message pair per round (draft first).
namespace {

std::string ints_json(const std::vector<int>& v) {
  std::string s = "[";
  for (std::size_t i = 0; i < v.size(); ++i) { if (i) s += ","; s += std::to_string(v[i]); }
  return s + "]";
}

struct ToVerifier { std::vector<int> hit; std::vector<Spec> specs; };
struct ToDraft { std::vector<Outcome> keys; std::vector<long> lens; };

class Wire {  // Channel (sim.cpp:271-317)
 public:
  explicit Wire(std::vector<Message>& log) : log_(log) {}
  void d2v(const ToVerifier& m, double clock) {
    if (n_d2v_ != n_v2d_) throw ProtocolViolationError("protocol: draft sent out of turn");
    ++n_d2v_;
    std::string toks = "[";
    for (std::size_t j = 0; j < m.specs.size(); ++j) { if (j) toks += ","; toks += ints_json(m.specs[j].tokens); }
    toks += "]";
    const std::size_t d0 = m.specs.empty() ? 0 : m.specs[0].dists.size();
    const std::size_t d1 = (m.specs.empty() || m.specs[0].dists.empty()) ? 0 : m.specs[0].dists[0].size();
    log_.push_back({n_d2v_, "d2v",
                    "{\"dists_shape\":[" + std::to_string(d0) + "," + std::to_string(d1) + "],\"hits\":" +
                        ints_json(m.hit) + ",\"tokens\":" + toks + "}",
                    clock});
  }
  void v2d(const ToDraft& m, double clock) {
    if (n_v2d_ + 1 != n_d2v_) throw ProtocolViolationError("protocol: verifier sent out of turn");
    ++n_v2d_;
    std::string oc = "[";
    for (std::size_t j = 0; j < m.keys.size(); ++j) {
      if (j) oc += ",";
      oc += "[" + std::to_string(m.keys[j].k) + "," + std::to_string(m.keys[j].t) + "]";
    }
    oc += "]";
    std::string lens = "[";
    for (std::size_t j = 0; j < m.lens.size(); ++j) { if (j) lens += ","; lens += std::to_string(m.lens[j]); }
    lens += "]";
    log_.push_back({n_v2d_, "v2d", "{\"outcomes\":" + oc + ",\"seq_lens\":" + lens + "}", clock});
  }
  long pairs() const { return n_v2d_; }
 private:
  std::vector<Message>& log_;
  long n_d2v_ = 0, n_v2d_ = 0;
};

}  // namespace

HarnessOut sim_harness(const SimCfg& c) {
  check_cfg(c);
  if (c.synthetic_iid) throw Error("run_protocol_harness: requires the real cache hit mode");
  const int B = c.batch, K = c.K;
  const VerifyOpts vo{c.target_scheme, c.accept_scale};
  HarnessOut out;
  Wire wire(out.transcript);

  // draft-side state (DraftProcess, sim.cpp:376-463)
  std::vector<Rng> d_rng;
  std::vector<std::vector<int>> d_hist;
  std::vector<Spec> d_spec(static_cast<std::size_t>(B));
  std::vector<Src> d_src(std::size_t(B), Src::Initial);
  std::vector<SpecCache> d_cache;
  // verifier-side state (VerifierProcess, sim.cpp:321-369)
  std::vector<Rng> v_rng;
  std::vector<std::vector<int>> v_hist;
  const std::uint64_t vseed = child_seed(c.seed, 0x5EED);
  for (int j = 0; j < B; ++j) {
    d_rng.emplace_back(child_seed(c.seed, std::uint64_t(j)));
    d_hist.push_back(start_history(c.prompt, *c.draft));
    v_rng.emplace_back(child_seed(vseed, std::uint64_t(j)));
    v_hist.push_back(start_history(c.prompt, *c.target));
  }
  Stats& st = out.stats;

  double clock = c.primary_time;
  ToVerifier inflight;
  for (int j = 0; j < B; ++j) {
    d_spec[std::size_t(j)] = draft_tokens(*c.draft, model_ctx(d_hist[std::size_t(j)], *c.draft), K, c.scheme,
                                         d_rng[std::size_t(j)], Origin::Primary);
    inflight.hit.push_back(0);
    inflight.specs.push_back(d_spec[std::size_t(j)]);
  }
  wire.d2v(inflight, clock);
  // wall time of the rounds alone (after prefill and the initial drafts):
  // the CPU baseline's decode rate (bench.py), not part of the algorithm
  const auto t_rounds = std::chrono::steady_clock::now();

  for (long round = 1; round <= c.rounds; ++round) {
    const double v0 = clock, v1 = clock + 1.0;
    // speculator: pre-speculate against the in-flight speculation
    d_cache.clear();
    for (int j = 0; j < B; ++j) {
      const Plan& plan = d_spec[std::size_t(j)].origin == Origin::Primary ? c.primary_plan : c.backup_plan;
      d_cache.push_back(prespeculate(*c.draft, model_ctx(d_hist[std::size_t(j)], *c.draft), d_spec[std::size_t(j)],
                                     plan, c.scheme, K, d_rng[std::size_t(j)]));
    }
    const double ready = v0 + c.primary_time;
    if (c.primary_time < 1.0 && ready >= v1) throw ProtocolViolationError("protocol: cache missed the overlap window");

    // verifier
    ToDraft back;
    for (int j = 0; j < B; ++j) {
      Spec s;
      s.tokens = inflight.specs[std::size_t(j)].tokens;
      s.dists = inflight.specs[std::size_t(j)].dists;
      const Round res = verify_spec(*c.target, model_ctx(v_hist[std::size_t(j)], *c.target), s, v_rng[std::size_t(j)], vo);
      auto& vh = v_hist[std::size_t(j)];
      vh.insert(vh.end(), res.emitted.begin(), res.emitted.end());
      st.tokens += long(res.emitted.size());
      st.accepted_sum += res.key.k;
      back.keys.push_back(res.key);
      back.lens.push_back(long(vh.size()) - long(start_history(c.prompt, *c.target).size()));
    }
    wire.v2d(back, v1);
    out.outcomes0.push_back(back.keys[0]);

    for (int j = 0; j < B; ++j) {
      const long n = back.keys[std::size_t(j)].k + 1;
      const Src src = d_src[std::size_t(j)];
      if (src == Src::Initial) ++st.initial_rounds;
      else if (src == Src::Hit) { ++st.hit_rounds; st.hit_round_tokens += n; }
      else { ++st.miss_rounds; st.miss_round_tokens += n; }
    }

    bool all_hit = false;
    if (round < c.rounds) {
      ToVerifier next;
      bool every = true;
      for (int j = 0; j < B; ++j) {
        const Outcome key = back.keys[std::size_t(j)];
        const Spec* found = d_cache[std::size_t(j)].find(key);
        const bool hit = found != nullptr;
        Spec& cur = d_spec[std::size_t(j)];
        const bool from_primary = cur.origin == Origin::Primary;
        st.log.push_back({from_primary, hit});
        (from_primary ? st.p_lookups : st.b_lookups) += 1;
        (from_primary ? st.p_hits : st.b_hits) += hit ? 1 : 0;
        auto& dh = d_hist[std::size_t(j)];
        dh.insert(dh.end(), cur.tokens.begin(), cur.tokens.begin() + key.k);
        dh.push_back(key.t);
        if (hit) {
          cur = *found;
          cur.origin = Origin::Primary;
          d_src[std::size_t(j)] = Src::Hit;
        } else {
          every = false;
          cur = c.backup == Backup::SamePrimaryJIT
                    ? draft_tokens(*c.draft, model_ctx(dh, *c.draft), K, c.scheme, d_rng[std::size_t(j)], Origin::Backup)
                    : uniform_spec(c.draft->vocab(), K, d_rng[std::size_t(j)]);
          d_src[std::size_t(j)] = Src::Backup;
        }
        if (j == 0) out.hits0.push_back(hit ? 1 : 0);
        next.hit.push_back(hit ? 1 : 0);
        next.specs.push_back(cur);
      }
      all_hit = every;
      const double respond = all_hit ? std::max(v1, ready) : v1 + c.backup_time();
      wire.d2v(next, respond);
      inflight = std::move(next);
      clock = respond;
    } else {
      clock = v1;
    }
    out.timings.push_back({v0, v1, ready, all_hit});
  }
  out.decode_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_rounds).count();
  if (wire.pairs() != c.rounds) throw ProtocolViolationError("protocol: message pair count mismatch");
  st.rounds = c.rounds;
  st.batch = B;
  st.vtime = clock;
  if (c.keep_streams) {
    const long skip = long(start_history(c.prompt, *c.target).size());
    for (auto& h : v_hist) st.streams.emplace_back(h.begin() + skip, h.end());
  }
  return out;
}

// ============================================================== perf
// perf.cpp:10-15
static void check_p(double p) {
  if (!(p >= 0.0) || !(p <= 1.0)) throw Error("perf: hit_rate must be in [0, 1]");
}

// perf.cpp:19-27: [p E_hit + (1-p) E_miss] / [p max(1, T_p) + (1-p)(1 + T_b)]
double speedup_ssd(double p, const Yields& y, double tp, double tb) {
  check_p(p);
  const double tokens = p * y.hit + (1.0 - p) * y.miss;
  const double latency = p * std::max(1.0, tp) + (1.0 - p) * (1.0 + tb);
  return tokens / latency;
}

// perf.cpp:44-55: whole-batch stall, the all-hit probability is p^b
double speedup_batch(double p, const Yields& y, double tp, double tb, double batch) {
  check_p(p);
  if (!(batch >= 1.0)) throw Error("speedup_batch: batch must be >= 1");
  const double tokens = p * y.hit + (1.0 - p) * y.miss;
  const double all = std::pow(p, batch);
  return tokens / (all * std::max(1.0, tp) + (1.0 - all) * (1.0 + tb));
}

// perf.cpp:57-73: b* = log(1 + 1/T_p - E_hit / (T_p E)) / log(p)
double critical_batch(double p, const Yields& y, double tp) {
  if (!(p > 0.0) || !(p < 1.0)) throw Error("critical_batch: hit_rate must be in (0, 1)");
  if (!(tp > 0.0)) throw Error("critical_batch: primary_time must be > 0");
  const double mean = p * y.hit + (1.0 - p) * y.miss;
  const double arg = 1.0 + 1.0 / tp - y.hit / (tp * mean);
  if (!(arg > 0.0) || arg > 1.0) throw NoCrossoverError("critical_batch: one backup strategy dominates at every batch size");
  return std::log(arg) / std::log(p);
}

// hitmodel.cpp:65-106
PowerLaw fit_powerlaw(const std::vector<std::pair<double, double>>& samples) {
  std::vector<double> xs;
  for (const auto& [f, m] : samples) {
    if (!(f >= 1.0)) throw Error("fit_powerlaw: fan-out values must be >= 1");
    if (!(m > 0.0) || !(m <= 1.0)) throw Error("fit_powerlaw: miss rates must be in (0, 1]");
    if (std::find(xs.begin(), xs.end(), f) == xs.end()) xs.push_back(f);
  }
  if (xs.size() < 2) throw InsufficientDataError("fit_powerlaw: need at least two distinct fan-out values");
  const double n = double(samples.size());
  double mx = 0.0, my = 0.0;
  for (const auto& [f, m] : samples) { mx += std::log(f); my += std::log(m); }
  mx /= n;
  my /= n;
  double sxx = 0.0, sxy = 0.0, syy = 0.0;
  for (const auto& [f, m] : samples) {
    const double dx = std::log(f) - mx, dy = std::log(m) - my;
    sxx += dx * dx;
    sxy += dx * dy;
    syy += dy * dy;
  }
  const double slope = sxy / sxx;
  PowerLaw out;
  out.exponent = -slope;
  out.log_amplitude = my - slope * mx;
  out.r_squared = syy > 0.0 ? 1.0 - (syy - slope * sxy) / syy : 1.0;
  return out;
}

// ============================================================== Markov LM
// lm.cpp:49-63
MarkovLM::MarkovLM(int V, int order, std::uint64_t seed, std::vector<Row> rows)
    : V_(V), m_(order), seed_(seed), rows_(std::move(rows)) {
  if (V_ < 2) throw Error("SyntheticLM: vocab_size must be >= 2");
  if (m_ < 0 || m_ > 2) throw Error("SyntheticLM: order must be 0..2");
  std::size_t want = 1;
  for (int i = 0; i < m_; ++i) want *= std::size_t(V_);
  if (rows_.size() != want) throw Error("SyntheticLM: table must cover all V^m contexts");
  for (const Row& r : rows_) {
    if (int(r.size()) != V_) throw Error("SyntheticLM: row length mismatch");
    for (double v : r) if (!std::isfinite(v)) throw Error("SyntheticLM: logits must be finite");
  }
}

// lm.cpp:65-80 — lexicographic index of the last m tokens.
std::size_t MarkovLM::row_of(std::span<const int> ctx) const {
  if (int(ctx.size()) < m_) throw Error("context_index: context shorter than model order");
  std::size_t r = 0;
  for (int i = int(ctx.size()) - m_; i < int(ctx.size()); ++i) {
    const int t = ctx[std::size_t(i)];
    if (t < 0 || t >= V_) throw Error("context_index: token out of range");
    r = r * std::size_t(V_) + std::size_t(t);
  }
  return r;
}

std::span<const double> MarkovLM::logits(std::span<const int> ctx) { return rows_[row_of(ctx)]; }

namespace {
// lm.cpp:22-29
Row log_weights(const Row& w) {
  double s = 0.0;
  for (double x : w) s += x;
  Row z(w.size());
  for (std::size_t i = 0; i < w.size(); ++i) z[i] = std::log(std::max(w[i] / s, 1e-300));
  return z;
}
// lm.cpp:31-45 — Dirichlet row: exponentials for concentration 1, else
// libstdc++'s gamma_distribution on the stream's engine.
Row dirichlet(int V, double conc, Rng& rng) {
  Row w(static_cast<std::size_t>(V));
  if (conc == 1.0) {
    for (double& x : w) x = -std::log(1.0 - rng.unit());
  } else {
    std::gamma_distribution<double> g(conc, 1.0);
    for (double& x : w) x = g(rng.engine());
  }
  for (double& x : w) x = std::max(x, 1e-300);
  return w;
}
}  // namespace

// lm.cpp:91-105
MarkovLM markov_make(int V, int order, double conc, std::uint64_t seed) {
  if (V < 2) throw Error("make_lm: vocab_size must be >= 2");
  if (!(conc > 0.0)) throw Error("make_lm: concentration must be > 0");
  std::size_t n = 1;
  for (int i = 0; i < order; ++i) n *= std::size_t(V);
  std::vector<Row> rows;
  rows.reserve(n);
  for (std::size_t c = 0; c < n; ++c) {
    Rng r(child_seed(seed, c));
    rows.push_back(log_weights(dirichlet(V, conc, r)));
  }
  return MarkovLM(V, order, seed, std::move(rows));
}

// lm.cpp:107-127
MarkovLM markov_mix_draft(const MarkovLM& t, double eps, std::uint64_t noise_seed) {
  if (!(eps >= 0.0) || !(eps <= 1.0)) throw Error("derive_draft: epsilon must be in [0, 1]");
  std::vector<Row> rows;
  rows.reserve(t.rows().size());
  Scheme standard;
  for (std::size_t c = 0; c < t.rows().size(); ++c) {
    const Row base = scheme_probs(t.rows()[c], standard);
    Rng r(child_seed(noise_seed, c));
    const Row noise = normalized(dirichlet(t.vocab(), 1.0, r));
    Row mix(base.size());
    for (std::size_t i = 0; i < mix.size(); ++i) mix[i] = (1.0 - eps) * base[i] + eps * noise[i];
    rows.push_back(log_weights(mix));
  }
  return MarkovLM(t.vocab(), t.order(), noise_seed, std::move(rows));
}

// lm.cpp:129-148
double markov_mean_acceptance(const MarkovLM& t, const MarkovLM& d, const Scheme& ts, const Scheme& ds) {
  if (t.vocab() != d.vocab() || t.order() != d.order()) throw Error("mean_acceptance: model shapes differ");
  double s = 0.0;
  for (std::size_t c = 0; c < t.rows().size(); ++c)
    s += accept_mass(scheme_probs(t.rows()[c], ts), scheme_probs(d.rows()[c], ds));
  return s / double(t.rows().size());
}

// lm.cpp:150-172 — 40-step bisection on the mixing weight.
MarkovPair markov_calibrate(const MarkovLM& t, double goal, std::uint64_t seed) {
  if (!(goal > 0.0) || !(goal < 1.0)) throw Error("calibrate_pair: alpha_goal must be in (0, 1)");
  const Scheme st;
  const double floor_alpha = markov_mean_acceptance(t, markov_mix_draft(t, 1.0, seed), st, st);
  if (goal < floor_alpha) throw UnreachableError("calibrate_pair: alpha_goal below attainable range");
  double lo = 0.0, hi = 1.0;
  for (int i = 0; i < 40; ++i) {
    const double mid = 0.5 * (lo + hi);
    if (markov_mean_acceptance(t, markov_mix_draft(t, mid, seed), st, st) > goal) lo = mid;
    else hi = mid;
  }
  const double eps = 0.5 * (lo + hi);
  return MarkovPair{markov_mix_draft(t, eps, seed), eps};
}

}  // namespace oracle
