// Host-side fan-out plans of the speculation cache (reference cache.hpp:18-68,
// cache.cpp:13-169): the per-position budget F_0..F_K that sizes the branch
// batch of pre-speculation. Host-only, evaluated once per configuration.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/ssd_b200.h"

namespace ssd {
extern thread_local std::string g_last_error;
}

namespace {

struct PlanError {
  ssd_status code;
  const char* msg;
};

// capped-geometric weight a^k (1-a) (a^K at the cap) times 1 - F^-r
double hit_rate(const std::vector<int>& f, double a, double r) {
  const int K = int(f.size()) - 1;
  double total = 0.0, w = 1.0;
  for (int k = 0; k < K; ++k) {
    total += w * (1.0 - a) * (f[size_t(k)] >= 1 ? 1.0 - std::pow(double(f[size_t(k)]), -r) : 0.0);
    w *= a;
  }
  return total + w * (f[size_t(K)] >= 1 ? 1.0 - std::pow(double(f[size_t(K)]), -r) : 0.0);
}

std::vector<double> continuous(double a, double r, int K, double budget) {
  if (!(a > 0.0) || !(a < 1.0)) throw PlanError{SSD_ERROR, "geometric_fanout: acceptance must be in (0, 1)"};
  if (!(r > 0.0)) throw PlanError{SSD_ERROR, "geometric_fanout: exponent must be > 0"};
  if (K < 1) throw PlanError{SSD_ERROR, "geometric_fanout: lookahead must be >= 1"};
  const double q = std::pow(a, 1.0 / (1.0 + r));
  const double cap = std::pow(a, K / (1.0 + r)) * std::pow(1.0 - a, -1.0 / (1.0 + r));
  const double f0 = budget / (cap + (1.0 - std::pow(q, K)) / (1.0 - q));
  std::vector<double> f(size_t(K) + 1);
  for (int k = 0; k < K; ++k) f[size_t(k)] = f0 * std::pow(q, k);
  f[size_t(K)] = f0 * cap;
  return f;
}

void to_plan(const std::vector<int>& f, int role, int budget, ssd_plan* out) {
  out->lookahead = int(f.size()) - 1;
  out->role = role;
  out->budget = budget;
  for (int k = 0; k <= SSD_MAX_LOOKAHEAD; ++k) out->fan_out[k] = k < int(f.size()) ? f[size_t(k)] : 0;
}

}  // namespace

extern "C" {

ssd_status ssd_geometric_fanout(double a, double r, int32_t K, int32_t budget, int32_t role, ssd_plan* out) {
  try {
    if (K > SSD_MAX_LOOKAHEAD) throw PlanError{SSD_TOO_LARGE, "geometric_fanout: lookahead too large"};
    if (budget < K + 1) throw PlanError{SSD_BUDGET_TOO_SMALL, "geometric_fanout: budget must be at least lookahead + 1"};
    const std::vector<double> c = continuous(a, r, K, double(budget));
    const size_t n = c.size();
    std::vector<int> f(n);
    std::vector<double> frac(n);
    int used = 0;
    for (size_t k = 0; k < n; ++k) {
      f[k] = int(std::floor(c[k]));
      frac[k] = c[k] - f[k];
      used += f[k];
    }
    std::vector<size_t> ord(n);
    std::iota(ord.begin(), ord.end(), size_t(0));
    std::stable_sort(ord.begin(), ord.end(), [&](size_t x, size_t y) { return frac[x] > frac[y]; });
    for (size_t i = 0; used < budget; ++i, ++used) f[ord[i % n]] += 1;
    for (size_t k = 0; k < n; ++k)
      while (f[k] < 1) {
        const size_t big = size_t(std::max_element(f.begin(), f.end()) - f.begin());
        if (f[big] <= 1) throw PlanError{SSD_BUDGET_TOO_SMALL, "geometric_fanout: cannot satisfy minimum"};
        f[big] -= 1;
        f[k] += 1;
      }
    for (;;) {  // exchange polish under the separable concave objective
      double best = hit_rate(f, a, r);
      size_t bf = 0, bt = 0;
      bool better = false;
      for (size_t from = 0; from < n; ++from) {
        if (f[from] <= 1) continue;
        for (size_t to = 0; to < n; ++to) {
          if (to == from) continue;
          --f[from]; ++f[to];
          const double v = hit_rate(f, a, r);
          ++f[from]; --f[to];
          if (v > best + 1e-15) { best = v; bf = from; bt = to; better = true; }
        }
      }
      if (!better) break;
      --f[bf];
      ++f[bt];
    }
    to_plan(f, role, budget, out);
    return SSD_OK;
  } catch (const PlanError& e) {
    ssd::g_last_error = e.msg;
    return e.code;
  }
}

ssd_status ssd_uniform_fanout(int32_t K, int32_t budget, int32_t role, ssd_plan* out) {
  if (K < 1) { ssd::g_last_error = "uniform_fanout: lookahead must be >= 1"; return SSD_ERROR; }
  if (K > SSD_MAX_LOOKAHEAD) { ssd::g_last_error = "uniform_fanout: lookahead too large"; return SSD_TOO_LARGE; }
  if (budget < K + 1) { ssd::g_last_error = "uniform_fanout: budget must be at least lookahead + 1"; return SSD_BUDGET_TOO_SMALL; }
  std::vector<int> f(size_t(K) + 1, budget / (K + 1));
  for (int k = 0; k < budget % (K + 1); ++k) f[size_t(k)] += 1;
  to_plan(f, role, budget, out);
  return SSD_OK;
}

double ssd_conditional_hit_rate(const ssd_plan* p, double a, double r) {
  std::vector<int> f(p->fan_out, p->fan_out + p->lookahead + 1);
  return hit_rate(f, a, r);
}

// hitmodel::fit_powerlaw (hitmodel.cpp:65-106): log-log least squares of the
// measured miss rate against the fan-out, miss = A F^-r; r is the exponent
// geometric_fanout takes (calibrated plans).
ssd_status ssd_fit_powerlaw(const double* fan_out, const double* miss, int32_t n, double* exponent,
                            double* log_amplitude, double* r_squared) {
  std::vector<double> xs;
  for (int i = 0; i < n; ++i) {
    if (!(fan_out[i] >= 1.0)) { ssd::g_last_error = "fit_powerlaw: fan-out values must be >= 1"; return SSD_ERROR; }
    if (!(miss[i] > 0.0) || !(miss[i] <= 1.0)) {
      ssd::g_last_error = "fit_powerlaw: miss rates must be in (0, 1]";
      return SSD_ERROR;
    }
    if (std::find(xs.begin(), xs.end(), fan_out[i]) == xs.end()) xs.push_back(fan_out[i]);
  }
  if (xs.size() < 2) {
    ssd::g_last_error = "fit_powerlaw: need at least two distinct fan-out values";
    return SSD_INSUFFICIENT_DATA;
  }
  double mx = 0.0, my = 0.0;
  for (int i = 0; i < n; ++i) { mx += std::log(fan_out[i]); my += std::log(miss[i]); }
  mx /= double(n);
  my /= double(n);
  double sxx = 0.0, sxy = 0.0, syy = 0.0;
  for (int i = 0; i < n; ++i) {
    const double dx = std::log(fan_out[i]) - mx, dy = std::log(miss[i]) - my;
    sxx += dx * dx;
    sxy += dx * dy;
    syy += dy * dy;
  }
  const double slope = sxy / sxx;
  *exponent = -slope;
  *log_amplitude = my - slope * mx;
  *r_squared = syy > 0.0 ? 1.0 - (syy - slope * sxy) / syy : 1.0;
  return SSD_OK;
}

// Latency model of the loop (perf.cpp:19-55) and the backup crossover b*
// (perf.cpp:57-73) that drives the Saguaro fallback policy at batch > 1:
// below b* re-using the primary as a JIT backup wins, at or above it the
// free FastRandom backup does (PAPER §5, whole-batch stalls).
ssd_status ssd_speedup_batch(double p, double hit_tokens, double miss_tokens, double primary_time, double backup_time,
                             double batch, double* out) {
  if (!(p >= 0.0) || !(p <= 1.0)) { ssd::g_last_error = "perf: hit_rate must be in [0, 1]"; return SSD_ERROR; }
  if (!(batch >= 1.0)) { ssd::g_last_error = "speedup_batch: batch must be >= 1"; return SSD_ERROR; }
  const double tokens = p * hit_tokens + (1.0 - p) * miss_tokens;
  const double all = std::pow(p, batch);
  *out = tokens / (all * std::max(1.0, primary_time) + (1.0 - all) * (1.0 + backup_time));
  return SSD_OK;
}

ssd_status ssd_critical_batch(double p, double hit_tokens, double miss_tokens, double primary_time, double* out) {
  if (!(p > 0.0) || !(p < 1.0)) { ssd::g_last_error = "critical_batch: hit_rate must be in (0, 1)"; return SSD_ERROR; }
  if (!(primary_time > 0.0)) { ssd::g_last_error = "critical_batch: primary_time must be > 0"; return SSD_ERROR; }
  const double mean = p * hit_tokens + (1.0 - p) * miss_tokens;
  const double arg = 1.0 + 1.0 / primary_time - hit_tokens / (primary_time * mean);
  if (!(arg > 0.0) || arg > 1.0) {
    ssd::g_last_error = "critical_batch: one backup strategy dominates at every batch size";
    return SSD_NO_CROSSOVER;
  }
  *out = std::log(arg) / std::log(p);
  return SSD_OK;
}

}  // extern "C"
