// TEST INFRASTRUCTURE ONLY — see transformer_lm.hpp.
#include "transformer_lm.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>

#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>

namespace oracle {

// ------------------------------------------------------------ thread pool
// Persistent workers for row-parallel GEMV (no OpenMP runtime in the image).
namespace {
class Pool {
 public:
  explicit Pool(int n) : n_(std::max(1, n)) {
    for (int i = 1; i < n_; ++i) workers_.emplace_back([this, i] { loop(i); });
  }
  ~Pool() {
    { std::lock_guard<std::mutex> g(mu_); stop_ = true; ++gen_; }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  int size() const { return n_; }
  // fn(begin, end) over [0, n) split in n_ contiguous chunks.
  void run(long n, const std::function<void(long, long)>& fn) {
    if (n_ == 1 || n < 2) { fn(0, n); return; }
    {
      std::lock_guard<std::mutex> g(mu_);
      fn_ = &fn; total_ = n; pending_ = n_ - 1; ++gen_;
    }
    cv_.notify_all();
    chunk(0, n, fn);
    std::unique_lock<std::mutex> g(mu_);
    done_.wait(g, [this] { return pending_ == 0; });
  }
 private:
  void chunk(int i, long n, const std::function<void(long, long)>& fn) {
    const long b = n * i / n_, e = n * (i + 1) / n_;
    if (b < e) fn(b, e);
  }
  void loop(int i) {
    long seen = 0;
    for (;;) {
      const std::function<void(long, long)>* fn;
      long n;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return gen_ != seen; });
        seen = gen_;
        if (stop_) return;
        fn = fn_; n = total_;
      }
      chunk(i, n, *fn);
      std::lock_guard<std::mutex> g(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  int n_;
  std::vector<std::thread> workers_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(long, long)>* fn_ = nullptr;
  long total_ = 0, gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
};

Pool& pool_for(int threads) {
  static std::mutex mu;
  static std::unique_ptr<Pool> p;
  std::lock_guard<std::mutex> g(mu);
  if (!p || p->size() != threads) p = std::make_unique<Pool>(threads);
  return *p;
}
}  // namespace

// ------------------------------------------------------------ generator
std::uint64_t tensor_key(std::uint64_t seed, std::uint32_t id) { return child_seed(seed, id); }

float unit_value(std::uint64_t key, std::uint64_t index) {
  const std::uint64_t h = child_seed(key, index);
  const std::int32_t top = std::int32_t(std::uint32_t(h >> 32));
  return float(top >> 8) * 0x1.0p-23f;  // exact: 24-bit integer times 2^-23
}

std::uint16_t to_bf16(float x) {
  std::uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return std::uint16_t((u >> 16) | 0x40);  // NaN
  u += 0x7fffu + ((u >> 16) & 1u);
  return std::uint16_t(u >> 16);
}

float from_bf16(std::uint16_t b) {
  const std::uint32_t u = std::uint32_t(b) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

static inline float bf16_round(float x) { return from_bf16(to_bf16(x)); }

std::uint32_t layer_tensor_id(Role r, int layer, TensorKind k) {
  return (std::uint32_t(r) << 24) | (std::uint32_t(layer) << 8) | std::uint32_t(k);
}

void rope_tables(const TfShape& s, std::vector<float>& cs, std::vector<float>& sn) {
  const int half = s.head_dim / 2;
  cs.assign(std::size_t(s.max_ctx) * half, 0.f);
  sn.assign(std::size_t(s.max_ctx) * half, 0.f);
  for (int p = 0; p < s.max_ctx; ++p)
    for (int i = 0; i < half; ++i) {
      const double inv = std::pow(s.rope_theta, -2.0 * i / double(s.head_dim));
      const double a = double(p) * inv;
      cs[std::size_t(p) * half + i] = float(std::cos(a));
      sn[std::size_t(p) * half + i] = float(std::sin(a));
    }
}

namespace {

float sign_of(std::uint64_t key, std::size_t i) { return unit_value(key, i) < 0.f ? -1.f : 1.f; }

// Input width of a layer tensor (its row length).
std::size_t in_dim(const TfShape& s, TensorKind k) {
  if (k == WO) return std::size_t(s.heads) * std::size_t(s.head_dim);
  if (k == WD) return std::size_t(s.ffn);
  return std::size_t(s.d);
}

}  // namespace

// Logical layer-tensor element, bf16 bits. The target's
// layer-0 MLP embeds the draft's layer-0 MLP in its [ffn_d x d_d] corner.
std::uint16_t layer_elem(const TfShape& self, const TfShape& draft, const PairParams& p, Role role, int l,
                         TensorKind k, std::size_t r, std::size_t c) {
  if (role == Role::Target && l == 0) {
    if ((k == WG || k == WU) && r < std::size_t(draft.ffn) && c < std::size_t(draft.d))
      return layer_elem(draft, draft, p, Role::Draft, 0, k, r, c);
    if (k == WD && r < std::size_t(draft.d) && c < std::size_t(draft.ffn))
      return layer_elem(draft, draft, p, Role::Draft, 0, k, r, c);
  }
  const std::size_t in = in_dim(self, k);
  float scale = 1.0f / std::sqrt(float(in));
  if (k == WO) scale = p.block_out_scale * scale;
  if (k == WD) scale = ((role == Role::Draft && l == 0) ? p.shared_mlp_scale : p.block_out_scale) * scale;
  return to_bf16(unit_value(tensor_key(p.seed, layer_tensor_id(role, l, k)), r * in + c) * scale);
}

// ------------------------------------------------------------ model
TransformerLM::TransformerLM(const TfShape& s, const TfShape& dr, const PairParams& p, Role role, int threads)
    : s_(s), threads_(threads > 0 ? threads : int(std::max(1u, std::thread::hardware_concurrency()))) {
  const int ds = dr.d;
  if (ds > s.d || dr.ffn > s.ffn) throw Error("TransformerLM: draft backbone exceeds the target");
  if (role == Role::Draft && (ds != s.d || !s.tied)) throw Error("TransformerLM: draft must be tied");
  Pool& pool = pool_for(threads_);
  const std::size_t V = std::size_t(s.vocab), d = std::size_t(s.d);
  const std::uint64_t kS = tensor_key(p.seed, kSharedEmbed);
  // embeddings / head
  embed_.resize(V * d);
  if (!s.tied) head_.resize(V * d);
  const std::uint64_t kPE = tensor_key(p.seed, kTargetPrivEmbed), kPH = tensor_key(p.seed, kTargetPrivHead);
  const std::size_t dp = d - std::size_t(ds);
  pool.run(long(V), [&](long vb, long ve) {
  for (std::size_t v = std::size_t(vb); v < std::size_t(ve); ++v)
    for (std::size_t i = 0; i < d; ++i) {
      if (i < std::size_t(ds)) {
        const std::uint16_t b = to_bf16(unit_value(kS, v * std::size_t(ds) + i) * p.embed_scale);
        embed_[v * d + i] = b;
        if (!s.tied) head_[v * d + i] = b;
      } else {
        const std::size_t j = v * dp + (i - std::size_t(ds));
        embed_[v * d + i] = to_bf16(unit_value(kPE, j) * p.target_private_embed);
        head_[v * d + i] = to_bf16(unit_value(kPH, j) * p.target_private_head);
      }
    }
  });
  // norm gains
  final_gain_.resize(d);
  ffn_gain0_.assign(d, 1.0f);
  const std::uint64_t kGS = tensor_key(p.seed, kGainShared), kGN = tensor_key(p.seed, kGainNoise),
                      kGT = tensor_key(p.seed, kGainTargetPriv);
  const float comp = std::sqrt(float(ds) / float(s.d));  // rms over d vs d_draft
  for (std::size_t i = 0; i < d; ++i) {
    if (role == Role::Draft) {
      final_gain_[i] = p.logit_scale * ((1.0f - p.draft_gain_mix) * sign_of(kGS, i) + p.draft_gain_mix * sign_of(kGN, i));
    } else {
      final_gain_[i] = p.logit_scale * (i < std::size_t(ds) ? sign_of(kGS, i) : sign_of(kGT, i - std::size_t(ds)));
      if (i < std::size_t(ds)) ffn_gain0_[i] = comp;
    }
  }
  // blocks
  const int qd = s.heads * s.head_dim, kvd = s.kv_heads * s.head_dim;
  layers_.resize(std::size_t(s.layers));
  for (int l = 0; l < s.layers; ++l) {
    Layer& L = layers_[std::size_t(l)];
    auto fill = [&](std::vector<std::uint16_t>& dst, TensorKind k, std::size_t rows) {
      const std::size_t cols = in_dim(s, k);
      dst.resize(rows * cols);
      pool.run(long(rows), [&](long rb, long re) {
        for (std::size_t r = std::size_t(rb); r < std::size_t(re); ++r)
          for (std::size_t c = 0; c < cols; ++c) dst[r * cols + c] = layer_elem(s, dr, p, role, l, k, r, c);
      });
    };
    fill(L.wq, WQ, std::size_t(qd));
    fill(L.wk, WK, std::size_t(kvd));
    fill(L.wv, WV, std::size_t(kvd));
    fill(L.wo, WO, d);
    fill(L.wg, WG, std::size_t(s.ffn));
    fill(L.wu, WU, std::size_t(s.ffn));
    fill(L.wd, WD, d);
  }
  rope_tables(s, cos_, sin_);
  kc_.assign(std::size_t(s.layers), {});
  vc_.assign(std::size_t(s.layers), {});
  x_.resize(d); hb_.resize(std::max<std::size_t>(d, std::size_t(s.ffn)));
  q_.resize(std::size_t(qd)); k_.resize(std::size_t(kvd)); v_.resize(std::size_t(kvd));
  att_.resize(std::size_t(qd)); g_.resize(std::size_t(s.ffn)); u_.resize(std::size_t(s.ffn));
  act_.resize(std::size_t(s.ffn)); tmp_.resize(d);
}

std::uint16_t TransformerLM::weight_bits(int layer, TensorKind k, std::size_t row, std::size_t col) const {
  const Layer& L = layers_[std::size_t(layer)];
  const int qd = s_.heads * s_.head_dim;
  switch (k) {
    case WQ: return L.wq[row * std::size_t(s_.d) + col];
    case WK: return L.wk[row * std::size_t(s_.d) + col];
    case WV: return L.wv[row * std::size_t(s_.d) + col];
    case WO: return L.wo[row * std::size_t(qd) + col];
    case WG: return L.wg[row * std::size_t(s_.d) + col];
    case WU: return L.wu[row * std::size_t(s_.d) + col];
    case WD: return L.wd[row * std::size_t(s_.ffn) + col];
    default: throw Error("weight_bits: bad kind");
  }
}
std::uint16_t TransformerLM::embed_bits(std::size_t v, std::size_t i) const { return embed_[v * std::size_t(s_.d) + i]; }
std::uint16_t TransformerLM::head_bits(std::size_t v, std::size_t i) const {
  return (s_.tied ? embed_ : head_)[v * std::size_t(s_.d) + i];
}

// y[r] = sum_c w[r][c] * x[c]; fp32, eight interleaved partial sums.
void TransformerLM::gemv(const std::vector<std::uint16_t>& w, int rows, int cols, const float* x, float* y) {
  const std::uint16_t* W = w.data();
  auto body = [&](long rb, long re) {
  for (int r = int(rb); r < int(re); ++r) {
    const std::uint16_t* row = W + std::size_t(r) * std::size_t(cols);
    if (f64_) {  // noise-floor reference: the same bf16 rounding points, fp64 sums
      double a = 0.0;
      for (int c = 0; c < cols; ++c) a += double(from_bf16(row[c])) * double(x[c]);
      y[r] = float(a);
      continue;
    }
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int c = 0;
    for (; c + 8 <= cols; c += 8)
      for (int j = 0; j < 8; ++j) {
        std::uint32_t u = std::uint32_t(row[c + j]) << 16;
        float wv;
        std::memcpy(&wv, &u, 4);
        acc[j] += wv * x[c + j];
      }
    float s = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
    for (; c < cols; ++c) s += from_bf16(row[c]) * x[c];
    y[r] = s;
  }
  };
  if (std::size_t(rows) * std::size_t(cols) >= (1u << 18)) pool_for(threads_).run(rows, body);
  else body(0, rows);
}

namespace {
// RMSNorm then bf16 rounding (the engine's GEMV input precision).
void rmsnorm_bf16(const float* x, const float* g, int n, float eps, float* out, bool f64 = false) {
  float ss = 0.f;
  if (f64) {
    double d = 0.0;
    for (int i = 0; i < n; ++i) d += double(x[i]) * double(x[i]);
    ss = float(d);
  } else {
    for (int i = 0; i < n; ++i) ss += x[i] * x[i];
  }
  const float r = 1.0f / std::sqrt(ss / float(n) + eps);
  for (int i = 0; i < n; ++i) out[i] = bf16_round(x[i] * r * (g ? g[i] : 1.0f));
}
}  // namespace

void TransformerLM::step(int token, int pos) {
  if (token < 0 || token >= s_.vocab) throw Error("TransformerLM: token out of range");
  if (pos >= s_.max_ctx) throw Error("TransformerLM: context exceeds max_ctx");
  const int d = s_.d, hd = s_.head_dim, half = hd / 2, H = s_.heads, KVH = s_.kv_heads;
  const int qd = H * hd, kvd = KVH * hd, grp = H / KVH;
  for (int i = 0; i < d; ++i) x_[std::size_t(i)] = from_bf16(embed_[std::size_t(token) * std::size_t(d) + std::size_t(i)]);
  const float* cs = &cos_[std::size_t(pos) * std::size_t(half)];
  const float* sn = &sin_[std::size_t(pos) * std::size_t(half)];
  const float scale = 1.0f / std::sqrt(float(hd));
  for (int l = 0; l < s_.layers; ++l) {
    Layer& L = layers_[std::size_t(l)];
    rmsnorm_bf16(x_.data(), nullptr, d, s_.norm_eps, hb_.data(), f64_);
    gemv(L.wq, qd, d, hb_.data(), q_.data());
    gemv(L.wk, kvd, d, hb_.data(), k_.data());
    gemv(L.wv, kvd, d, hb_.data(), v_.data());
    auto rope = [&](float* v) {
      for (int i = 0; i < half; ++i) {
        const float a = v[i], b = v[i + half];
        v[i] = a * cs[i] - b * sn[i];
        v[i + half] = b * cs[i] + a * sn[i];
      }
    };
    for (int h = 0; h < H; ++h) rope(&q_[std::size_t(h * hd)]);
    for (int h = 0; h < KVH; ++h) rope(&k_[std::size_t(h * hd)]);
    auto& KC = kc_[std::size_t(l)];
    auto& VC = vc_[std::size_t(l)];
    KC.resize(std::size_t(pos + 1) * std::size_t(kvd));
    VC.resize(std::size_t(pos + 1) * std::size_t(kvd));
    for (int i = 0; i < kvd; ++i) {
      KC[std::size_t(pos) * std::size_t(kvd) + std::size_t(i)] = bf16_round(k_[std::size_t(i)]);
      VC[std::size_t(pos) * std::size_t(kvd) + std::size_t(i)] = bf16_round(v_[std::size_t(i)]);
    }
    std::vector<float> sc(std::size_t(pos + 1));
    for (int h = 0; h < H; ++h) {
      const int kvh = h / grp;
      const float* q = &q_[std::size_t(h * hd)];
      float mx = -INFINITY;
      for (int j = 0; j <= pos; ++j) {
        const float* kr = &KC[std::size_t(j) * std::size_t(kvd) + std::size_t(kvh * hd)];
        float dot = 0.f;
        if (f64_) {
          double dd = 0.0;
          for (int i = 0; i < hd; ++i) dd += double(q[i]) * double(kr[i]);
          dot = float(dd);
        } else {
          for (int i = 0; i < hd; ++i) dot += q[i] * kr[i];
        }
        sc[std::size_t(j)] = dot * scale;
        mx = std::max(mx, sc[std::size_t(j)]);
      }
      float den = 0.f;
      for (int j = 0; j <= pos; ++j) { sc[std::size_t(j)] = std::exp(sc[std::size_t(j)] - mx); den += sc[std::size_t(j)]; }
      float* o = &att_[std::size_t(h * hd)];
      if (f64_) {
        double dden = 0.0;
        for (int j = 0; j <= pos; ++j) dden += double(sc[std::size_t(j)]);
        for (int i = 0; i < hd; ++i) {
          double a = 0.0;
          for (int j = 0; j <= pos; ++j)
            a += double(sc[std::size_t(j)]) * double(VC[std::size_t(j) * std::size_t(kvd) + std::size_t(kvh * hd + i)]);
          o[i] = bf16_round(float(a / dden));
        }
        continue;
      }
      for (int i = 0; i < hd; ++i) o[i] = 0.f;
      for (int j = 0; j <= pos; ++j) {
        const float* vr = &VC[std::size_t(j) * std::size_t(kvd) + std::size_t(kvh * hd)];
        const float pj = sc[std::size_t(j)];
        for (int i = 0; i < hd; ++i) o[i] += pj * vr[i];
      }
      for (int i = 0; i < hd; ++i) o[i] = bf16_round(o[i] / den);
    }
    gemv(L.wo, d, qd, att_.data(), tmp_.data());
    for (int i = 0; i < d; ++i) x_[std::size_t(i)] += tmp_[std::size_t(i)];
    rmsnorm_bf16(x_.data(), l == 0 ? ffn_gain0_.data() : nullptr, d, s_.norm_eps, hb_.data(), f64_);
    gemv(L.wg, s_.ffn, d, hb_.data(), g_.data());
    gemv(L.wu, s_.ffn, d, hb_.data(), u_.data());
    for (int i = 0; i < s_.ffn; ++i) {
      const float gv = g_[std::size_t(i)];
      act_[std::size_t(i)] = bf16_round(gv / (1.0f + std::exp(-gv)) * u_[std::size_t(i)]);
    }
    gemv(L.wd, d, s_.ffn, act_.data(), tmp_.data());
    for (int i = 0; i < d; ++i) x_[std::size_t(i)] += tmp_[std::size_t(i)];
  }
  rmsnorm_bf16(x_.data(), final_gain_.data(), d, s_.norm_eps, hb_.data(), f64_);
  out_f32_.resize(std::size_t(s_.vocab));
  gemv(s_.tied ? embed_ : head_, s_.vocab, d, hb_.data(), out_f32_.data());
  ++processed_;
}

// Incremental decoding with a longest-common-prefix KV cache: positions that
// agree with the previous call are reused, the rest recomputed one token at
// a time (the engine's decode order).
std::span<const double> TransformerLM::logits(std::span<const int> ctx) {
  const std::size_t n = ctx.size();
  if (n == 0) throw Error("TransformerLM: empty context");
  std::size_t l = 0;
  while (l < n && l < cached_.size() && cached_[l] == ctx[l]) ++l;
  if (l == n && memo_.size() >= n && !memo_[n - 1].empty()) {
    out_f32_ = memo_[n - 1];
  } else {
    if (l == n) l = n - 1;
    cached_.resize(l);
    memo_.resize(l);
    for (std::size_t p = l; p < n; ++p) {
      step(ctx[p], int(p));
      cached_.push_back(ctx[p]);
      memo_.push_back(out_f32_);
    }
  }
  out_.assign(out_f32_.begin(), out_f32_.end());
  return out_;
}

}  // namespace oracle
