// Vocabulary-row operations of the SSD round, split over many CTAs:
// greedy argmax, sampling under a scheme (dist::apply_scheme + dist::sample,
// categorical.cpp:65-92, 129-143) and the cache-key top-(F+1) selection
// (cache.cpp:249-270). A row of V = 128256 logits is 512 KB, so one CTA per
// row (the first version) was bound by a single SM's bandwidth; here phase 1
// runs (chunk, row) CTAs that each reduce ~1000 logits to a top-T candidate
// list plus an online-softmax partial (max, sum of exp), and phase 2 merges
// them per row and, for sampling, walks the chunk masses to the one chunk
// that holds the uniform's quantile, which a single warp then scans in index
// order. The (value desc, index asc) order of dist::top_indices is exact.
#pragma once

#include "kernels.cuh"

namespace ssd {

constexpr int kRowThreads = 256;
constexpr int kMaxChunks = 256;

struct RowChunk {
  float zmax;   // max logit of the chunk
  int pad;
  double esum;  // sum over the chunk of exp(z / tau - zmax / tau)
};

// Top-T over an array of candidates (value desc, index asc), block-wide.
template <int NT>
__device__ void block_topk_pairs(const VI* __restrict__ cand, int n, int T, VI* out, VI* wl) {
  VI L[kMaxTopF + 1];
  for (int t = 0; t < T; ++t) L[t] = VI{-INFINITY, 0x7fffffff};
  for (int j = threadIdx.x; j < n; j += NT) {
    const VI c = cand[j];
    if (ranks_before(c.v, c.i, L[T - 1].v, L[T - 1].i)) {
      int p = T - 1;
      while (p > 0 && ranks_before(c.v, c.i, L[p - 1].v, L[p - 1].i)) { L[p] = L[p - 1]; --p; }
      L[p] = c;
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int head = 0;
  for (int t = 0; t < T; ++t) {
    VI mine = head < T ? L[head] : VI{-INFINITY, 0x7fffffff};
    VI best = warp_best(mine);
    if (head < T && mine.v == best.v && mine.i == best.i) ++head;
    if (lane == 0) wl[w * T + t] = best;
  }
  __syncthreads();
  if (w == 0) {
    constexpr int NW = NT / 32;
    int h2 = 0;
    for (int t = 0; t < T; ++t) {
      VI mine = (lane < NW && h2 < T) ? wl[lane * T + h2] : VI{-INFINITY, 0x7fffffff};
      VI best = warp_best(mine);
      if (lane < NW && h2 < T && mine.v == best.v && mine.i == best.i) ++h2;
      if (lane == 0) out[t] = best;
    }
  }
  __syncthreads();
}

// Phase 1: CTA (chunk c, row r) over logits[r][c*C, (c+1)*C). Rows are
// base + r * row_stride (row_stride in floats); with row_ptrs the row
// pointers come from a device table instead (spec rows).
__global__ void __launch_bounds__(kRowThreads) row_phase1_kernel(const float* __restrict__ base, size_t row_stride,
                                                                 int V, int T, double tau, VI* __restrict__ cand,
                                                                 RowChunk* __restrict__ stat) {
  __shared__ VI top[kMaxTopF + 1];
  __shared__ VI wl[(kRowThreads / 32) * (kMaxTopF + 1)];
  __shared__ float shf[32];
  __shared__ double shd[32];
  const int c = blockIdx.x, r = blockIdx.y, nch = gridDim.x;
  const int C = (V + nch - 1) / nch;
  const int j0 = c * C, j1 = min(V, j0 + C);
  const float* z = base + size_t(r) * row_stride;
  // candidates: local lists over the chunk
  VI L[kMaxTopF + 1];
  for (int t = 0; t < T; ++t) L[t] = VI{-INFINITY, 0x7fffffff};
  float zm = -INFINITY;
  for (int j = j0 + threadIdx.x; j < j1; j += kRowThreads) {
    const float v = z[j];
    zm = fmaxf(zm, v);
    if (ranks_before(v, j, L[T - 1].v, L[T - 1].i)) {
      int p = T - 1;
      while (p > 0 && ranks_before(v, j, L[p - 1].v, L[p - 1].i)) { L[p] = L[p - 1]; --p; }
      L[p] = VI{v, j};
    }
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int head = 0;
  for (int t = 0; t < T; ++t) {
    VI mine = head < T ? L[head] : VI{-INFINITY, 0x7fffffff};
    VI best = warp_best(mine);
    if (head < T && mine.v == best.v && mine.i == best.i) ++head;
    if (lane == 0) wl[w * T + t] = best;
  }
  zm = warp_max(zm);
  if (lane == 0) shf[w] = zm;
  __syncthreads();
  if (w == 0) {
    constexpr int NW = kRowThreads / 32;
    int h2 = 0;
    for (int t = 0; t < T; ++t) {
      VI mine = (lane < NW && h2 < T) ? wl[lane * T + h2] : VI{-INFINITY, 0x7fffffff};
      VI best = warp_best(mine);
      if (lane < NW && h2 < T && mine.v == best.v && mine.i == best.i) ++h2;
      if (lane == 0) top[t] = best;
    }
    float m2 = lane < NW ? shf[lane] : -INFINITY;
    m2 = warp_max(m2);
    if (lane == 0) shf[0] = m2;
  }
  __syncthreads();
  VI* out = cand + (size_t(r) * nch + c) * T;
  for (int t = threadIdx.x; t < T; t += kRowThreads) out[t] = top[t];
  if (tau > 0.0) {
    const float cm = shf[0];
    const double mt = double(cm) / tau;
    double s = 0.0;
    for (int j = j0 + threadIdx.x; j < j1; j += kRowThreads) s += exp(double(z[j]) / tau - mt);
    s = block_sum(s, shd);
    if (threadIdx.x == 0) stat[size_t(r) * nch + c] = RowChunk{cm, 0, s};
  } else if (threadIdx.x == 0) {
    stat[size_t(r) * nch + c] = RowChunk{shf[0], 0, 0.0};
  }
}

// Phase 2, greedy / sampled draw: one CTA per row. Output token written to
// out[r * out_stride]; u[r * u_stride] is the row's uniform.
__global__ void __launch_bounds__(kRowThreads) row_sample_kernel(const float* __restrict__ base, size_t row_stride, int V,
                                                                 int nch, int T, DScheme s, const VI* __restrict__ cand,
                                                                 const RowChunk* __restrict__ stat,
                                                                 const double* __restrict__ u, int u_stride,
                                                                 int* __restrict__ out, int out_stride) {
  __shared__ VI top[kMaxTopF + 1];
  __shared__ VI wl[(kRowThreads / 32) * (kMaxTopF + 1)];
  __shared__ int s_chunk;
  __shared__ double s_before, s_target;
  const int r = blockIdx.x;
  block_topk_pairs<kRowThreads>(cand + size_t(r) * nch * T, nch * T, T, top, wl);
  if (s.tau == 0.0) {  // greedy: argmax (rank F when Saguaro removes the top-F set)
    if (threadIdx.x == 0) out[size_t(r) * out_stride] = (s.saguaro && s.C == 0.0) ? top[s.fan_out].i : top[0].i;
    return;
  }
  const float* z = base + size_t(r) * row_stride;
  const int C = (V + nch - 1) / nch;
  const RowChunk* st = stat + size_t(r) * nch;
  const double tau = s.tau;
  const int F = s.saguaro ? s.fan_out : 0;
  if (threadIdx.x == 0) {
    float zmax = -INFINITY;
    for (int c = 0; c < nch; ++c) zmax = fmaxf(zmax, st[c].zmax);
    const double M = double(zmax) / tau;
    // chunk masses (Saguaro: the top-F weights scaled by C)
    double total = 0.0;
    for (int c = 0; c < nch; ++c) total += st[c].esum * exp(double(st[c].zmax) / tau - M);
    double adj_total = 0.0;
    for (int t = 0; t < F; ++t) adj_total += (1.0 - s.C) * exp(double(top[t].v) / tau - M);
    const double S = total - adj_total;
    const double target = u[size_t(r) * u_stride] * S;
    double acc = 0.0;
    int pick = -1;
    for (int c = 0; c < nch; ++c) {
      double wc = st[c].esum * exp(double(st[c].zmax) / tau - M);
      for (int t = 0; t < F; ++t)
        if (top[t].i / C == c) wc -= (1.0 - s.C) * exp(double(top[t].v) / tau - M);
      if (target < acc + wc) { pick = c; break; }
      acc += wc;
    }
    s_chunk = pick;
    s_before = acc;
    s_target = target;
    // fallback (rounding left the total below u): the last positive token
    if (pick < 0) {
      int last = V - 1;
      while (last > 0) {
        bool zero = false;
        for (int t = 0; t < F; ++t) zero |= (top[t].i == last && s.C == 0.0);
        if (!zero) break;
        --last;
      }
      out[size_t(r) * out_stride] = last;
    }
  }
  __syncthreads();
  if (s_chunk < 0) return;
  // one warp scans the chunk in index order
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  float zmax = -INFINITY;
  for (int c = 0; c < nch; ++c) zmax = fmaxf(zmax, st[c].zmax);
  const double M = double(zmax) / tau;
  const int j0 = s_chunk * C, j1 = min(V, j0 + C);
  double acc = s_before;
  const double target = s_target;
  int result = j1 - 1;
  for (int b = j0; b < j1; b += 32) {
    const int j = b + lane;
    double w = 0.0;
    if (j < j1) {
      w = exp(double(z[j]) / tau - M);
      for (int t = 0; t < F; ++t)
        if (top[t].i == j) w *= s.C;
    }
    double incl = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double t2 = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t2;
    }
    const unsigned hit = __ballot_sync(0xffffffffu, j < j1 && target < acc + incl);
    if (hit) {
      result = b + __ffs(hit) - 1;
      break;
    }
    acc += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) out[size_t(r) * out_stride] = result;
}

// Phase 2, cache keys (cache.cpp:249-270): row k's first fan[k] candidates
// different from the in-flight token s_{k+1}; keys [rows][max_f] (-1 padded)
// and the flat branch list (bk, btok) at offset off[k]. Plans are [2][rows]
// (Primary, Backup); with `st` the plan follows the in-flight speculation's
// origin and the exclusions are its tokens.
__global__ void __launch_bounds__(kRowThreads) row_keys_kernel(int nch, int T, const VI* __restrict__ cand,
                                                               const int* __restrict__ fan2, const int* __restrict__ off2,
                                                               const LoopState* __restrict__ st,
                                                               const int* __restrict__ excl_explicit, int n_excl,
                                                               int max_f, int* __restrict__ keys, int* __restrict__ bk,
                                                               int* __restrict__ btok, int nrows, int bper) {
  // Batch lanes: grid = lanes x nrows; lane l's key table is
  // keys[l][nrows][max_f], its branches bk/btok[l * bper ..].
  __shared__ VI top[kMaxTopF + 1];
  __shared__ VI wl[(kRowThreads / 32) * (kMaxTopF + 1)];
  const int row = blockIdx.x, l = row / nrows, k = row % nrows;
  if (st) st += l;
  keys += size_t(l) * nrows * max_f;
  bk += l * bper;
  btok += l * bper;
  const int origin = st ? st->spec_origin : 0;
  const int F = fan2[origin * nrows + k];
  const int off = off2[origin * nrows + k];
  const int excl = k < n_excl ? (st ? st->spec[k] : excl_explicit[k]) : -1;
  if (F <= 0) {
    for (int j = threadIdx.x; j < max_f; j += kRowThreads) keys[k * max_f + j] = -1;
    return;
  }
  block_topk_pairs<kRowThreads>(cand + size_t(row) * nch * T, nch * T, min(F + 1, T), top, wl);
  if (threadIdx.x == 0) {
    int got = 0;
    for (int t = 0; t < min(F + 1, T) && got < F; ++t) {
      const int c = top[t].i;
      if (c == excl) continue;
      keys[k * max_f + got] = c;
      bk[off + got] = k;
      btok[off + got] = c;
      ++got;
    }
    for (int j = got; j < max_f; ++j) keys[k * max_f + j] = -1;
  }
}

}  // namespace ssd
