// Device kernels of the B200 Saguaro engine (sm_100a).
//
// Decode-step kernels (the replacement of lm::SyntheticLM::logits_at,
// reference lm.cpp:82-84) and the SSD control kernels (specdec.cpp:8-69,
// cache.cpp:232-277, sim.cpp:35-48, 258-601) that keep the whole round on
// the device. Layout conventions are in DESIGN.md §3.
#pragma once

#include "common.cuh"

namespace ssd {

typedef __nv_bfloat16 bf16;

// ------------------------------------------------------------------ params
// Per-forward token table (device memory, written by the prep kernels).
struct FwdParams {
  int tokens[kMaxM];
  int pos[kMaxM];       // RoPE position
  int slot[kMaxM];      // KV slot written by this token
  int main_len[kMaxM];  // visible main-cache keys: slots [mbase, mbase + main_len)
  int bbase[kMaxM];     // visible branch slots [bbase, bbase + blen)
  int blen[kMaxM];
  int mbase[kMaxM];     // first main slot of the token's sequence (batch lane; 0 at batch 1)
};

// Key index of `slot` among the keys query (mbase, main_len, bbase, blen)
// sees, or -1: main keys [0, main_len) live in slots mbase + j, branch keys
// main_len + i in slots bbase + i.
__device__ __forceinline__ int visible_key(int slot, int mbase, int main_len, int bbase, int blen) {
  if (slot >= mbase && slot < mbase + main_len) return slot - mbase;
  if (slot >= bbase && slot < bbase + blen) return main_len + slot - bbase;
  return -1;
}

// Paged main KV cache (the block manager is csrc/paged.cpp):
// main key j of the lane whose main region starts at slot mb lives at slot
// tab[lane][j >> shift] + (j & (page - 1)). tab == nullptr: the identity
// layout, slot mb + j. Branch slots are never paged.
struct KvMap {
  const int* tab;  // [lanes][ppl]: slot base of each logical page, this model's arena
  int shift;       // log2(page_tokens)
  int lane_S;      // slots of one lane (main + branch region)
  int ppl;         // pages per lane
};
__device__ __forceinline__ int main_slot(const KvMap& k, int mb, int j) {
  if (!k.tab) return mb + j;
  return k.tab[(mb / k.lane_S) * k.ppl + (j >> k.shift)] + (j & ((1 << k.shift) - 1));
}
// Key index of token t of this forward among the keys query (mb, main_len,
// bbase, blen) sees, or -1: a main-cache token (blen 0) is key pos[t] of its
// lane; a branch token is matched by slot (visible_key).
__device__ __forceinline__ int visible_token_key(const FwdParams* P, int t, int mb, int main_len, int bbase, int blen) {
  if (P->blen[t] == 0) return (P->mbase[t] == mb && P->pos[t] < main_len) ? P->pos[t] : -1;
  return visible_key(P->slot[t], mb, main_len, bbase, blen);
}

// Batch lanes (run_protocol_harness with batch_size > 1, sim.cpp:502-601):
// lane l's loop state is st[l], its history hist[l * hist_stride ..], its
// main KV slots start at l * lane_slots of each model, and its pre-speculation
// branches are the rows [l * bper, (l + 1) * bper) of the batched branch step.
struct Lanes {
  int hist_stride;
  int bper;
};

// Device-resident loop state: the harness' two processes' bookkeeping
// (sim.cpp:321-485) and the sim::RunStats counters (sim.hpp:55-104).
struct LoopState {
  int n;             // history length (tokens in hist[])
  int round;         // rounds completed
  int rounds;        // rounds requested
  int K;
  int spec[kMaxK];   // in-flight speculation
  int spec_origin;   // 0 Primary, 1 Backup
  int spec_src;      // 0 Initial, 1 CacheHit, 2 Backup
  int spec_uniform;  // dists are exactly uniform (FastRandom)
  const float* spec_rows[kMaxK];  // draft logit rows the tokens were drawn from
  int out_k, out_t;  // last verification outcome
  int hit;           // last lookup
  int error;         // ssd_status raised on the device (0 = ok)
  int backup_kind;   // 0 SamePrimaryJIT, 1 FastRandom
  int own;           // split speculator: the hit slot's branch is decoded here
  int seq_base;      // split runs: mailbox sequence numbers of this run start above it
  int Kb;            // pre-speculation continuation length (build_cache next_lookahead; K in the loops)
  double clock;      // harness virtual clock
  double primary_time, backup_time;
  long long tokens, p_lookups, p_hits, b_lookups, b_hits;
  long long hit_rounds, miss_rounds, initial_rounds, hit_round_tokens, miss_round_tokens;
  double accepted_sum;
  Mt64 vrng;         // verifier stream
  Mt64 drng;         // draft stream (the single stream for AR / SD)
};

// Scheme in device form (categorical.hpp:43-60).
struct DScheme {
  int saguaro;
  int fan_out;
  double tau;   // 0 = greedy
  double C;
};

// ------------------------------------------------------------------ weights
// Synthetic weight generator: a pure function of
// (seed, tensor id, flat index), bit-identical to oracle/transformer_lm.cpp.
struct GenShape { int d, heads, kv_heads, head_dim, ffn; };
struct GenPair { uint64_t seed; float embed_scale, shared_mlp_scale, block_out_scale, priv_embed, priv_head, gain_mix; };

__device__ __forceinline__ float unit_value(uint64_t key, uint64_t idx) {
  const uint64_t h = derive_seed(key, idx);
  const int32_t top = int32_t(uint32_t(h >> 32));
  return float(top >> 8) * 0x1.0p-23f;
}

__device__ __forceinline__ uint32_t layer_tensor_id(int role, int layer, int kind) {
  return (uint32_t(role) << 24) | (uint32_t(layer) << 8) | uint32_t(kind);
}

__device__ __forceinline__ size_t in_dim(const GenShape& s, int kind) {
  if (kind == 3) return size_t(s.heads) * size_t(s.head_dim);  // WO
  if (kind == 6) return size_t(s.ffn);                         // WD
  return size_t(s.d);
}

__device__ inline bf16 layer_elem(const GenShape& self, const GenShape& dr, const GenPair& p, int role, int l,
                                  int kind, size_t r, size_t c) {
  const GenShape* sh = &self;
  if (role == 0 && l == 0) {
    const bool gu = (kind == 4 || kind == 5) && r < size_t(dr.ffn) && c < size_t(dr.d);
    const bool dn = kind == 6 && r < size_t(dr.d) && c < size_t(dr.ffn);
    if (gu || dn) { role = 1; sh = &dr; }
  }
  const size_t in = in_dim(*sh, kind);
  float scale = 1.0f / sqrtf(float(in));
  if (kind == 3) scale = p.block_out_scale * scale;
  if (kind == 6) scale = ((role == 1 && l == 0) ? p.shared_mlp_scale : p.block_out_scale) * scale;
  const uint64_t key = derive_seed(p.seed, layer_tensor_id(role, l, kind));
  return __float2bfloat16_rn(unit_value(key, r * in + c) * scale);
}

// Element (r, c) of a [N][K] matrix in the pre-tiled GEMM layout
// (gemm_tc.cuh): 128 x 64 tiles, each a contiguous 16 KB run in the
// SWIZZLE_128B K-major order, tiles ordered (row tile, k block).
__host__ __device__ __forceinline__ size_t tiled_at(size_t r, size_t c, size_t KB) {
  const size_t t = r >> 7, rr = r & 127, kb = c >> 6, cc = c & 63;
  const size_t chunk = (cc >> 3) ^ (rr & 7);
  return ((t * KB + kb) * 128 + rr) * 64 + chunk * 8 + (cc & 7);
}

// Fill rows [row_off + row_stride * r] of the pre-tiled matrix dst (row
// length cols) with logical tensor (role, layer, kind) rows [lr0, lr0 + rows),
// columns [lc0, lc0 + cols): the tensor-parallel shard of the full logical
// tensor (lr0 = lc0 = 0 without TP), so every shard is bit-identical to the
// matching block of the unsharded model.
__global__ void gen_layer_kernel(bf16* dst, int rows, int cols, int row_stride, int row_off, GenShape self,
                                 GenShape dr, GenPair p, int role, int layer, int kind, int lr0, int lc0) {
  const size_t total = size_t(rows) * size_t(cols), KB = size_t(cols) / 64;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t r = e / size_t(cols), c = e % size_t(cols);
    dst[tiled_at(size_t(row_off) + size_t(row_stride) * r, c, KB)] =
        layer_elem(self, dr, p, role, layer, kind, size_t(lr0) + r, size_t(lc0) + c);
  }
}

// Embedding / LM head [V][d]: shared table S in dims [0, ds), target-private
// tables beyond (oracle transformer_lm.cpp constructor). `tiled` stores it in
// the GEMM layout (LM heads, and the tied draft table that is both).
// Rows [v0, v0 + V) of the table (vocabulary-parallel LM-head shard; v0 = 0
// for the whole table).
__global__ void gen_table_kernel(bf16* dst, int V, int d, int ds, GenPair p, int which /*0 embed 1 head*/, int tiled,
                                 int v0) {
  const uint64_t kS = derive_seed(p.seed, 0xE0000001u), kPE = derive_seed(p.seed, 0xE0000002u),
                 kPH = derive_seed(p.seed, 0xE0000003u);
  const size_t total = size_t(V) * size_t(d), dp = size_t(d - ds);
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t vl = e / size_t(d), i = e % size_t(d), v = size_t(v0) + vl;
    float val;
    if (i < size_t(ds)) {
      val = unit_value(kS, v * size_t(ds) + i) * p.embed_scale;
    } else {
      const size_t j = v * dp + (i - size_t(ds));
      val = which == 0 ? unit_value(kPE, j) * p.priv_embed : unit_value(kPH, j) * p.priv_head;
    }
    dst[tiled ? tiled_at(vl, i, size_t(d) / 64) : e] = __float2bfloat16_rn(val);
  }
}

__device__ __forceinline__ void pdl_wait_all() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// L2 prefetch window of the weight stream: the weight bytes
// that upcoming GEMMs will stream next, pulled into L2 by the kernel that
// runs before them, so HBM keeps streaming through latency-bound kernels
// (attention, norms, GEMM ramps / drains). A persistent stream-K GEMM reads
// its P unit ranges in parallel, so "the next bytes" of a GEMM are the
// fraction [f0, f1) of EVERY range: a segment names a GEMM (pre-tiled
// weights, U units of unit_bytes, P ranges) and that fraction. The issuing
// kernel's CTAs share the ranges round-robin; thread 0 issues bulk L2
// prefetches of <= 64 KB.
struct PfSeg {
  const char* w;
  int U, P;
  float f0, f1;
};
constexpr int kPfSegs = 4;
struct Prefetch {
  PfSeg seg[kPfSegs];
  int n;
};

__device__ __forceinline__ void prefetch_window(const Prefetch& w, int unit_bytes) {
  if (w.n <= 0 || threadIdx.x != 0 || threadIdx.y != 0 || threadIdx.z != 0) return;
  const int nct = int(gridDim.x * gridDim.y * gridDim.z);
  const int cta = int(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z));
  for (int k = 0; k < w.n && k < kPfSegs; ++k) {
    const PfSeg& sg = w.seg[k];
    for (int j = cta; j < sg.P; j += nct) {
      const long long u0 = (long long)j * sg.U / sg.P, u1 = (long long)(j + 1) * sg.U / sg.P;
      const long long len = (u1 - u0) * unit_bytes;
      long long b0 = u0 * unit_bytes + ((long long)(sg.f0 * float(len)) & ~1023LL);
      long long b1 = u0 * unit_bytes + (sg.f1 >= 1.0f ? len : ((long long)(sg.f1 * float(len)) & ~1023LL));
      for (long long b = b0; b < b1; b += 65536) {
        const long long n = (b1 - b) < 65536 ? (b1 - b) : 65536;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(sg.w + b), "r"(uint32_t(n & ~15LL))
                     : "memory");
      }
    }
  }
}

constexpr int kPfUnitBytes = 32768;  // GEMM unit = 2 k-blocks of 128 x 64 bf16 (gemm_tc.cuh kABytes)

// ------------------------------------------------------------------ forward
// x[m][:] = E[token_m][:] (fp32 residual stream); E row-major or pre-tiled.
__global__ void embed_kernel(const bf16* __restrict__ E, int d, int tiled, const FwdParams* __restrict__ P,
                             float* __restrict__ x, Prefetch pf) {
  KTL_ENTER(1);
  prefetch_window(pf, kPfUnitBytes);
  asm volatile("griddepcontrol.launch_dependents;");
  pdl_wait_all();
  KTL_READY();
  const int m = blockIdx.x;
  const size_t tok = size_t(P->tokens[m]);
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    const size_t at = tiled ? tiled_at(tok, size_t(i), size_t(d) / 64) : tok * size_t(d) + size_t(i);
    x[size_t(m) * d + i] = __bfloat162float(E[at]);
  }
  KTL_EXIT();
}

// Residual add + RMSNorm (gain optional) with bf16 rounding of the output:
// x += delta (the previous block's projection, when given), then
// out = bf16(x * rsqrt(mean(x^2) + eps) * g) — the GEMM input precision
// (oracle rmsnorm_bf16). Folding the residual add here keeps every GEMM
// epilogue a plain store. One CTA per token, float4 accesses, d <= 8192.
constexpr int kNormThreads = 256;

// zero / zero_n: rows [M][zero_n] of the next GEMM's output, cleared for its
// atomic split-K accumulation (gemm_tc.cuh GemmArgs::atomic).
__global__ void __launch_bounds__(kNormThreads) rmsnorm_kernel(float* __restrict__ x, const float* __restrict__ delta,
                                                               int d, const float* __restrict__ g, float eps,
                                                               bf16* __restrict__ out, Prefetch pf,
                                                               float* __restrict__ zero, int zero_n) {
  __shared__ float sh[32];
  KTL_ENTER(2);
  prefetch_window(pf, kPfUnitBytes);
  // let the next kernel (a GEMM) launch now and prefetch its weights; it
  // still waits for this grid, which waits for its own predecessor
  asm volatile("griddepcontrol.launch_dependents;");
  pdl_wait_all();
  KTL_READY();
  const int m = blockIdx.x;
  float4* xr = reinterpret_cast<float4*>(x + size_t(m) * d);
  const float4* dr = delta ? reinterpret_cast<const float4*>(delta + size_t(m) * d) : nullptr;
  const int n4 = d >> 2;
  float4 keep[8];  // n4 / kNormThreads <= 8
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = threadIdx.x + k * kNormThreads;
    if (i < n4) {
      float4 v = xr[i];
      if (dr) {
        const float4 e = dr[i];
        v.x += e.x; v.y += e.y; v.z += e.z; v.w += e.w;
        xr[i] = v;
      }
      keep[k] = v;
      ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
  }
  if (zero)
    for (int i = threadIdx.x; i < (zero_n >> 2); i += kNormThreads)
      reinterpret_cast<float4*>(zero + size_t(m) * zero_n)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  ss = block_sum(ss, sh);
  const float r = 1.0f / sqrtf(ss / float(d) + eps);
  __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(out + size_t(m) * d);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int i = threadIdx.x + k * kNormThreads;
    if (i >= n4) break;
    const float4 v = keep[k];
    float a = v.x * r, b = v.y * r, c = v.z * r, e = v.w * r;
    if (g) {
      const float4 gg = reinterpret_cast<const float4*>(g)[i];
      a *= gg.x; b *= gg.y; c *= gg.z; e *= gg.w;
    }
    o2[2 * i] = __floats2bfloat162_rn(a, b);
    o2[2 * i + 1] = __floats2bfloat162_rn(c, e);
  }
  KTL_EXIT();
}

enum Epi { EPI_STORE = 0, EPI_RESID = 1, EPI_SWIGLU = 2 };

// Decode attention, split over keys (flash-decoding) and fused with RoPE and
// the KV-cache append of this forward's tokens. CTA = (key chunk, kv head,
// query token); the G = H / KVH query heads of the group share every K/V
// read. Keys of query m are the main-cache prefix [0, main_len) plus a
// branch-local segment [bbase, bbase + blen): the tree/branch mask of
// pre-speculation, generated arithmetically instead of materialised. Each
// chunk writes (max, sum, unnormalised output) per head; the last chunk to
// finish for (kv head, token) merges them in chunk order (deterministic).
// qkv rows are [q: H*hd][k: KVH*hd][v: KVH*hd] (fp32, pre-RoPE).
constexpr int kAttnThreads = 128;
constexpr int kAttnChunk = 128;  // keys per CTA
constexpr int kMaxGroup = 8;

struct AttnWs {
  float* part;   // [M][KVH][chunks][G][hd + 2]
  int* counter;  // [M][KVH]
};

// Scores of one key chunk for the G query heads of a KV group: the hd/8
// 16-byte chunks of a K row are spread over hd/8 lanes (a warp covers
// 32/(hd/8) keys per step, its reads one contiguous run — conflict-free in
// shared memory, coalesced in global), partial dot products reduced with
// xor shuffles. rowp(jj) -> the K row of key jj of the chunk. hd: 16..128,
// a power of two.
template <int G, class RowPtr>
__device__ __forceinline__ void attn_scores(const float* qs, float* sc, int n, int hd, float scale, int warp, int lane,
                                            RowPtr rowp) {
  const int cpr = hd >> 3;
  const int kpi = 32 / cpr;
  const int sub = lane / cpr, ch = lane % cpr;
  float qv[G][8];
#pragma unroll
  for (int gg = 0; gg < G; ++gg)
#pragma unroll
    for (int i = 0; i < 8; ++i) qv[gg][i] = qs[gg * hd + ch * 8 + i];
  for (int jb = warp * kpi; jb < n; jb += (kAttnThreads / 32) * kpi) {
    const int jj = jb + sub;
    float part[G];
#pragma unroll
    for (int gg = 0; gg < G; ++gg) part[gg] = 0.f;
    if (jj < n) {
      float f[8];
      bf16x8_to_f32(rowp(jj)[ch], f);
#pragma unroll
      for (int gg = 0; gg < G; ++gg)
#pragma unroll
        for (int i = 0; i < 8; ++i) part[gg] += qv[gg][i] * f[i];
    }
    for (int o = cpr >> 1; o > 0; o >>= 1)
#pragma unroll
      for (int gg = 0; gg < G; ++gg) part[gg] += __shfl_xor_sync(0xffffffffu, part[gg], o);
    if (ch == 0 && jj < n)
#pragma unroll
      for (int gg = 0; gg < G; ++gg) sc[gg * kAttnChunk + jj] = part[gg] * scale;
  }
}

// Shared-memory scratch of one attention work item (kAttnSmemFloats(G, hd)
// floats + one int); static in attention_kernel.
struct AttnSmem {
  float* qs;      // [G][hd]
  float* sc;      // [G][kAttnChunk]
  float* stat;    // [G][2]
  float* pv_red;  // [key groups][G][hd]
  int* s_last;
};
__host__ __device__ constexpr int attn_pv_floats(int G, int hd) { return (kAttnThreads / (hd / 8)) * G * hd; }
__host__ __device__ constexpr int attn_smem_floats(int G, int hd) {
  return G * 128 + G * kAttnChunk + 2 * kMaxGroup + attn_pv_floats(G, hd) + 4;
}
__device__ __forceinline__ AttnSmem attn_smem_carve(float* base, int G, int hd) {
  AttnSmem a;
  a.qs = base;
  a.sc = a.qs + G * 128;
  a.stat = a.sc + G * kAttnChunk;
  a.pv_red = a.stat + 2 * kMaxGroup;
  a.s_last = reinterpret_cast<int*>(a.pv_red + attn_pv_floats(G, hd));
  return a;
}

struct BlockSync {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};

// One work item (key chunk, kv head, query token) of the split attention,
// executed by kAttnThreads threads (tid) that synchronise with sync().
template <int G, class Sync>
__device__ void attn_item(const float* __restrict__ qkv, const FwdParams* __restrict__ P, int M,
                          const float* __restrict__ cos_t, const float* __restrict__ sin_t, bf16* __restrict__ kc,
                          bf16* __restrict__ vc, int S, int H, int KVH, int hd, float scale, bf16* __restrict__ out,
                          AttnWs ws, int chunk, int kvh, int m, int nchunks, int tid, AttnSmem sm, Sync sync) {
  float* qs = sm.qs;
  float* sc = sm.sc;
  float* stat = sm.stat;
  float* pv_red = sm.pv_red;
  int* s_last = sm.s_last;
  const int lane = tid & 31, warp = tid >> 5;
  const int half = hd >> 1;
  const size_t row_len = size_t(H + 2 * KVH) * hd;
  const int main_len = P->main_len[m], bbase = P->bbase[m], blen = P->blen[m], mbase = P->mbase[m];
  const int nk = main_len + blen;
  const int j0 = chunk * kAttnChunk, j1 = min(nk, j0 + kAttnChunk);
  const int used = (nk + kAttnChunk - 1) / kAttnChunk;  // chunks holding keys of this query
  float* part = ws.part + ((size_t(m) * KVH + kvh) * nchunks) * G * (hd + 2);
  if (j0 < j1) {
    // 1) append (RoPE'd) K and V of this forward's tokens whose slot falls
    //    in this chunk (identical values wherever several CTAs write them)
    for (int e = tid; e < M * half; e += kAttnThreads) {
      const int t = e / half, i = e % half;
      const int slot = P->slot[t];
      const int j = visible_key(slot, mbase, main_len, bbase, blen);
      if (j < j0 || j >= j1) continue;
      const int pos = P->pos[t];
      const float c = cos_t[size_t(pos) * half + i], sn = sin_t[size_t(pos) * half + i];
      const float* ks = qkv + size_t(t) * row_len + size_t(H + kvh) * hd;
      const float* vs = qkv + size_t(t) * row_len + size_t(H + KVH + kvh) * hd;
      const float a = __ldcg(ks + i), b = __ldcg(ks + i + half);
      bf16* kd = kc + (size_t(kvh) * S + slot) * hd;
      bf16* vd = vc + (size_t(kvh) * S + slot) * hd;
      kd[i] = __float2bfloat16_rn(a * c - b * sn);
      kd[i + half] = __float2bfloat16_rn(b * c + a * sn);
      vd[i] = __float2bfloat16_rn(__ldcg(vs + i));
      vd[i + half] = __float2bfloat16_rn(__ldcg(vs + i + half));
    }
    // 2) rotated queries of the group
    {
      const int pos = P->pos[m];
      for (int e = tid; e < G * half; e += kAttnThreads) {
        const int gg = e / half, i = e % half;
        const float* src = qkv + size_t(m) * row_len + size_t(kvh * G + gg) * hd;
        const float c = cos_t[size_t(pos) * half + i], sn = sin_t[size_t(pos) * half + i];
        const float a = __ldcg(src + i), b = __ldcg(src + i + half);
        qs[gg * hd + i] = a * c - b * sn;
        qs[gg * hd + i + half] = b * c + a * sn;
      }
    }
    sync();
    // 3) scores, lane-cooperative (attn_scores): coalesced K row reads
    const bf16* kbase = kc + size_t(kvh) * S * hd;
    const bf16* vbase = vc + size_t(kvh) * S * hd;
    attn_scores<G>(qs, sc, j1 - j0, hd, scale, warp, lane, [&](int jj) {
      const int j = j0 + jj;
      const int slot = j < main_len ? mbase + j : bbase + (j - main_len);
      return reinterpret_cast<const uint4*>(kbase + size_t(slot) * hd);
    });
    sync();
    // 4) chunk softmax statistics (warp gg -> head gg)
    const int n = j1 - j0;
    for (int gg = warp; gg < G; gg += kAttnThreads / 32) {
      float mx = -INFINITY;
      for (int j = lane; j < n; j += 32) mx = fmaxf(mx, sc[gg * kAttnChunk + j]);
      mx = warp_max(mx);
      float den = 0.f;
      for (int j = lane; j < n; j += 32) {
        const float e = expf(sc[gg * kAttnChunk + j] - mx);
        sc[gg * kAttnChunk + j] = e;
        den += e;
      }
      den = warp_sum(den);
      if (lane == 0) { stat[2 * gg] = mx; stat[2 * gg + 1] = den; }
    }
    sync();
    // 5) unnormalised P.V of the chunk. Thread = (key group, 8-dim chunk);
    //    its <= 16 V vectors are loaded up front; partial sums are reduced
    //    over key groups through shared memory.
    {
      const int nd = hd >> 3;                 // 16-byte chunks per row
      const int ngrp = kAttnThreads / nd;     // key groups
      const int dc = tid % nd, kg = tid / nd;
      uint4 vv[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int jj = kg + u * ngrp;
        if (jj < n) {
          const int jabs = j0 + jj;
          const int slot = jabs < main_len ? mbase + jabs : bbase + (jabs - main_len);
          vv[u] = reinterpret_cast<const uint4*>(vbase + size_t(slot) * hd)[dc];
        }
      }
      float acc[kMaxGroup][8];
      
#pragma unroll
        for (int gg = 0; gg < G; ++gg)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[gg][i] = 0.f;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int jj = kg + u * ngrp;
        if (jj < n) {
          float f[8];
          bf16x8_to_f32(vv[u], f);
          
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
            const float p = sc[gg * kAttnChunk + jj];
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[gg][i] += p * f[i];
          }
        }
      }
      float* red = pv_red;  // [ngrp][G][hd]
      
#pragma unroll
        for (int gg = 0; gg < G; ++gg)
#pragma unroll
        for (int i = 0; i < 8; ++i) red[(kg * G + gg) * hd + dc * 8 + i] = acc[gg][i];
      sync();
      for (int e = tid; e < G * hd; e += kAttnThreads) {
        const int gg = e / hd, dd = e % hd;
        float o = 0.f;
        for (int k2 = 0; k2 < ngrp; ++k2) o += red[(k2 * G + gg) * hd + dd];
        part[(size_t(chunk) * G + gg) * (hd + 2) + dd] = o;
      }
    }
    if (tid < G) {
      part[(size_t(chunk) * G + tid) * (hd + 2) + hd] = stat[2 * tid];
      part[(size_t(chunk) * G + tid) * (hd + 2) + hd + 1] = stat[2 * tid + 1];
    }
  }
  // 6) the last of this query's chunks merges them in chunk order
  if (chunk >= used) return;
  __threadfence();
  sync();
  if (tid == 0) *s_last = atomicAdd(&ws.counter[m * KVH + kvh], 1) == used - 1;
  sync();
  if (!*s_last) return;
  __threadfence();
  for (int e = tid; e < G * hd; e += kAttnThreads) {
    const int gg = e / hd, dd = e % hd;
    float mx = -INFINITY;
    for (int c = 0; c < used; ++c) mx = fmaxf(mx, __ldcg(part + (size_t(c) * G + gg) * (hd + 2) + hd));
    float den = 0.f, o = 0.f;
    for (int c = 0; c < used; ++c) {
      const float* pc = part + (size_t(c) * G + gg) * (hd + 2);
      const float w = expf(__ldcg(pc + hd) - mx);
      den += w * __ldcg(pc + hd + 1);
      o += w * __ldcg(pc + dd);
    }
    out[size_t(m) * H * hd + size_t(kvh * G + gg) * hd + dd] = __float2bfloat16_rn(o / den);
  }
  if (tid == 0) ws.counter[m * KVH + kvh] = 0;
}

template <int G>
__global__ void __launch_bounds__(kAttnThreads) attention_kernel(const float* __restrict__ qkv, const FwdParams* __restrict__ P,
                                                                 int M, const float* __restrict__ cos_t,
                                                                 const float* __restrict__ sin_t, bf16* __restrict__ kc,
                                                                 bf16* __restrict__ vc, int S, int H, int KVH, int hd,
                                                                 float scale, bf16* __restrict__ out, AttnWs ws,
                                                                 Prefetch pf) {
  __shared__ float smem[attn_smem_floats(kMaxGroup, 128)];
  prefetch_window(pf, kPfUnitBytes);
  // let the next kernel (a GEMM) launch now and prefetch its weights; it
  // still waits for this grid, which waits for its own predecessor
  asm volatile("griddepcontrol.launch_dependents;");
  pdl_wait_all();
  attn_item<G>(qkv, P, M, cos_t, sin_t, kc, vc, S, H, KVH, hd, scale, out, ws, blockIdx.x, blockIdx.y, blockIdx.z,
               gridDim.x, threadIdx.x, attn_smem_carve(smem, G, hd), BlockSync());
}

// ------------------------------------------------------------------ top-k
// Block-wide top-T in the (value desc, index asc) order of
// dist::top_indices (categorical.cpp:35-48). Each thread keeps a sorted
// local list over a strided slice; warps merge by repeated warp argmax, then
// warp 0 merges the warp lists. Result in out[0..T) (shared memory).
template <int NT>
__device__ void block_topk(const float* __restrict__ z, int V, int T, VI* out, VI* wl /* (NT/32) * T */) {
  VI L[kMaxTopF + 1];
  for (int t = 0; t < T; ++t) L[t] = VI{-INFINITY, 0x7fffffff};
  for (int j = threadIdx.x; j < V; j += NT) {
    const float v = z[j];
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

// Cache keys (cache.cpp:249-270): for row k, the first fan[k] tokens of the
// ranking that differ from excl[k]. Writes keys[k*max_f + j] (-1 padded) and
// the flat branch list (bk, bt) at offset off[k]. grid = rows, 256 threads.
// Plans are [2][rows] (Primary, Backup); with `st` the plan follows the
// in-flight speculation's origin and the exclusions are its tokens.
__global__ void __launch_bounds__(256) keys_kernel(const float* __restrict__ rows, int V, const int* __restrict__ fan2,
                                                   const int* __restrict__ off2, const LoopState* __restrict__ st,
                                                   const int* __restrict__ excl_explicit, int n_excl, int max_f,
                                                   int* __restrict__ keys, int* __restrict__ bk, int* __restrict__ btok) {
  __shared__ VI top[kMaxTopF + 1];
  __shared__ VI wl[8 * (kMaxTopF + 1)];
  const int k = blockIdx.x, nrows = gridDim.x;
  const int origin = st ? st->spec_origin : 0;
  const int* fan = fan2 + origin * nrows;
  const int* off = off2 + origin * nrows;
  const int* excl_tok = st ? st->spec : excl_explicit;
  const int F = fan[k];
  if (F <= 0) {
    for (int j = threadIdx.x; j < max_f; j += blockDim.x) keys[k * max_f + j] = -1;
    return;
  }
  const int excl = k < n_excl ? excl_tok[k] : -1;
  const int T = min(F + 1, V);
  block_topk<256>(rows + size_t(k) * V, V, T, top, wl);
  if (threadIdx.x == 0) {
    int got = 0;
    for (int t = 0; t < T && got < F; ++t) {
      const int cand = top[t].i;
      if (cand == excl) continue;
      keys[k * max_f + got] = cand;
      bk[off[k] + got] = k;
      btok[off[k] + got] = cand;
      ++got;
    }
    for (int j = got; j < max_f; ++j) keys[k * max_f + j] = -1;
  }
}

// ------------------------------------------------------------------ sampling
// Greedy / sampled draw from one logit row under a scheme, with the uniform
// u[row] (dist::apply_scheme + dist::sample, categorical.cpp:65-92, 129-143).
// Probabilities in fp64 like the reference; the inverse CDF is a blocked
// prefix sum. grid = rows, 1024 threads.
constexpr int kSampleThreads = 1024;

__device__ inline int sample_row(const float* __restrict__ z, int V, const DScheme& s, double u) {
  __shared__ double shd[32];
  __shared__ VI shv[32];
  __shared__ VI top[kMaxTopF + 1];
  __shared__ VI wl[(kSampleThreads / 32) * (kMaxTopF + 1)];
  __shared__ int pick;
  const int tid = threadIdx.x;
  if (s.tau == 0.0) {
    if (s.saguaro && s.C == 0.0) {  // greedy with the top-F set removed: rank F
      block_topk<kSampleThreads>(z, V, s.fan_out + 1, top, wl);
      return top[s.fan_out].i;
    }
    VI b{-INFINITY, 0x7fffffff};
    for (int j = tid; j < V; j += blockDim.x)
      if (ranks_before(z[j], j, b.v, b.i)) b = VI{z[j], j};
    b = block_best(b, shv);
    return b.i;
  }
  VI thr{INFINITY, -1};  // F-th ranked element when Saguaro
  if (s.saguaro) {
    block_topk<kSampleThreads>(z, V, s.fan_out, top, wl);
    thr = top[s.fan_out - 1];
  }
  const double tau = s.tau;
  double mx = -INFINITY;
  for (int j = tid; j < V; j += blockDim.x) mx = fmax(mx, double(z[j]) / tau);
  mx = block_maxd(mx, shd);
  // contiguous chunk per thread for the ordered scan
  const int chunk = (V + blockDim.x - 1) / blockDim.x;
  const int b0 = min(V, tid * chunk), b1 = min(V, b0 + chunk);
  auto weight = [&](int j) {
    double w = exp(double(z[j]) / tau - mx);
    if (s.saguaro && (ranks_before(z[j], j, thr.v, thr.i) || j == thr.i)) w *= s.C;
    return w;
  };
  double loc = 0.0;
  for (int j = b0; j < b1; ++j) loc += weight(j);
  const double S = block_sum(loc, shd);
  // exclusive scan of per-thread probability mass
  double pm = 0.0;
  for (int j = b0; j < b1; ++j) pm += weight(j) / S;
  __shared__ double wsum[32];
  const int lane = tid & 31, w = tid >> 5;
  double incl = pm;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  __syncthreads();
  if (lane == 31) wsum[w] = incl;
  if (tid == 0) pick = 0x7fffffff;
  __syncthreads();
  double before = 0.0;
  for (int i = 0; i < w; ++i) before += wsum[i];
  const double excl = before + incl - pm;
  if (b0 < b1 && u < excl + pm) atomicMin(&pick, tid);
  __syncthreads();
  __shared__ int result;
  if (tid == pick) {
    double c = excl;
    int r = b1 - 1;
    for (int j = b0; j < b1; ++j) {
      c += weight(j) / S;
      if (u < c) { r = j; break; }
    }
    result = r;
  }
  __syncthreads();
  if (pick == 0x7fffffff) {  // rounding left the total below u: last positive
    int last = -1;
    for (int j = tid; j < V; j += blockDim.x) if (weight(j) > 0.0) last = max(last, j);
    VI lv{float(last), last};
    lv = block_best(lv, shv);
    return lv.i;
  }
  return result;
}

// Draw `n` uniforms from a device stream into u[] (the single-stream
// consumption of run_ar / run_sd, sim.cpp:64-121).
__global__ void draw_uniforms_kernel(Mt64* st, double* u, int n) {
  if (threadIdx.x == 0 && blockIdx.x == 0)
    for (int i = 0; i < n; ++i) u[i] = mt_unit(*st);
}

// Sample rows[r] with u[r]; token written to out[r * out_stride].
__global__ void __launch_bounds__(kSampleThreads) sample_rows_kernel(const float* __restrict__ rows, int V, DScheme s,
                                                                    const double* __restrict__ u, int u_stride,
                                                                    int* __restrict__ out, int out_stride) {
  const int r = blockIdx.x;
  const int t = sample_row(rows + size_t(r) * V, V, s, u ? u[size_t(r) * u_stride] : 0.0);
  if (threadIdx.x == 0) out[size_t(r) * out_stride] = t;
}

// ------------------------------------------------------------------ verify
// Per-row statistics for verification: max(z/tau) and sum of scheme weights
// for target rows [0, K] and draft rows [0, K), plus argmax (greedy) and the
// Saguaro threshold element. grid = 2K + 1, 1024 threads.
struct RowStat {
  double mx, S;
  int argmax;
  float thr_v;
  int thr_i;
};

__device__ inline double scheme_weight(float zj, int j, double mx, const DScheme& s, const RowStat& st) {
  double w = exp(double(zj) / s.tau - mx);
  if (s.saguaro && (ranks_before(zj, j, st.thr_v, st.thr_i) || j == st.thr_i)) w *= s.C;
  return w;
}

__global__ void __launch_bounds__(kSampleThreads) verify_stats_kernel(const float* __restrict__ trows,
                                                                     const LoopState* __restrict__ st, int V,
                                                                     DScheme ts, DScheme ds, RowStat* __restrict__ out) {
  __shared__ double shd[32];
  __shared__ VI shv[32];
  __shared__ VI top[kMaxTopF + 1];
  __shared__ VI wl[(kSampleThreads / 32) * (kMaxTopF + 1)];
  st += blockIdx.y;  // batch lane
  const int K = st->K;
  trows += size_t(blockIdx.y) * (K + 1) * V;
  out += size_t(blockIdx.y) * (2 * K + 1);
  const int r = blockIdx.x;
  const bool target = r <= K;
  if (!target && st->spec_uniform) return;
  const float* z = target ? trows + size_t(r) * V : st->spec_rows[r - K - 1];
  const DScheme s = target ? ts : ds;
  RowStat rs{0.0, 0.0, 0, INFINITY, -1};
  VI b{-INFINITY, 0x7fffffff};
  for (int j = threadIdx.x; j < V; j += blockDim.x)
    if (ranks_before(z[j], j, b.v, b.i)) b = VI{z[j], j};
  b = block_best(b, shv);
  rs.argmax = b.i;
  if (s.tau > 0.0) {
    if (s.saguaro) {
      block_topk<kSampleThreads>(z, V, s.fan_out, top, wl);
      rs.thr_v = top[s.fan_out - 1].v;
      rs.thr_i = top[s.fan_out - 1].i;
    }
    double mx = -INFINITY;
    for (int j = threadIdx.x; j < V; j += blockDim.x) mx = fmax(mx, double(z[j]) / s.tau);
    mx = block_maxd(mx, shd);
    rs.mx = mx;
    double loc = 0.0;
    for (int j = threadIdx.x; j < V; j += blockDim.x) loc += scheme_weight(z[j], j, mx, s, rs);
    rs.S = block_sum(loc, shd);
  } else if (s.saguaro && s.C == 0.0) {
    block_topk<kSampleThreads>(z, V, s.fan_out + 1, top, wl);
    rs.argmax = top[s.fan_out].i;
  }
  if (threadIdx.x == 0) out[r] = rs;
}

// Probability of token j in a row under scheme s (greedy: one-hot).
__device__ __forceinline__ double row_prob(const float* z, int j, const DScheme& s, const RowStat& st) {
  if (s.tau == 0.0) return j == st.argmax ? 1.0 : 0.0;
  return scheme_weight(z[j], j, st.mx, s, st) / st.S;
}

// The verification decision (specdec.cpp:27-69) and history append.
// One CTA of 1024 threads; thread 0 walks the accept coins on the
// verifier stream, then the block samples the bonus from the residual
// (or from the target row K when everything is accepted).
__global__ void __launch_bounds__(kSampleThreads) verify_decide_kernel(const float* __restrict__ trows, LoopState* st,
                                                                      int* __restrict__ hist, int V, DScheme ts, DScheme ds,
                                                                      double accept_scale, const RowStat* __restrict__ rs,
                                                                      int use_draft_stream, int hist_stride) {
  __shared__ int s_k;
  __shared__ double s_u;
  __shared__ int s_err;
  __shared__ double shd[32];
  __shared__ VI shv[32];
  st += blockIdx.x;  // batch lane: its stream, rows and history
  hist += size_t(blockIdx.x) * hist_stride;
  const int K = st->K;
  trows += size_t(blockIdx.x) * (K + 1) * V;
  rs += size_t(blockIdx.x) * (2 * K + 1);
  Mt64& rng = use_draft_stream ? st->drng : st->vrng;
  const bool uni = st->spec_uniform != 0;
  const double inv_v = 1.0 / double(V);
  if (threadIdx.x == 0) {
    int k = K;
    s_err = 0;
    for (int i = 0; i < K; ++i) {
      const int x = st->spec[i];
      const double pt = row_prob(trows + size_t(i) * V, x, ts, rs[i]);
      const double pd = uni ? inv_v : row_prob(st->spec_rows[i], x, ds, rs[K + 1 + i]);
      if (!(pd > 0.0)) { s_err = 1; k = i; break; }
      double a = fmin(1.0, pt / pd);
      a = fmin(1.0, a * accept_scale);
      if (mt_unit(rng) < a) continue;
      k = i;
      break;
    }
    s_k = k;
    s_u = mt_unit(rng);  // the bonus draw
  }
  __syncthreads();
  const int k = s_k;
  const double u = s_u;
  const float* zt = trows + size_t(k) * V;
  const RowStat& tst = rs[k];
  int bonus;
  if (k == K) {  // all accepted: bonus ~ target row K
    bonus = -1;
    if (ts.tau == 0.0) {
      bonus = tst.argmax;
    } else {
      // inverse CDF of the target row, thread-chunked like sample_row
      const int chunk = (V + blockDim.x - 1) / blockDim.x;
      const int b0 = min(V, int(threadIdx.x) * chunk), b1 = min(V, b0 + chunk);
      double pm = 0.0;
      for (int j = b0; j < b1; ++j) pm += row_prob(zt, j, ts, tst);
      __shared__ double wsum[32];
      __shared__ int pick;
      const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
      double incl = pm;
      for (int o = 1; o < 32; o <<= 1) { const double t = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl += t; }
      __syncthreads();
      if (lane == 31) wsum[w] = incl;
      if (threadIdx.x == 0) pick = 0x7fffffff;
      __syncthreads();
      double before = 0.0;
      for (int i = 0; i < w; ++i) before += wsum[i];
      const double ex = before + incl - pm;
      if (b0 < b1 && u < ex + pm) atomicMin(&pick, int(threadIdx.x));
      __syncthreads();
      __shared__ int res;
      if (int(threadIdx.x) == pick) {
        double c = ex;
        int r = b1 - 1;
        for (int j = b0; j < b1; ++j) { c += row_prob(zt, j, ts, tst); if (u < c) { r = j; break; } }
        res = r;
      }
      __syncthreads();
      if (pick == 0x7fffffff) {
        int last = -1;
        for (int j = threadIdx.x; j < V; j += blockDim.x) if (row_prob(zt, j, ts, tst) > 0.0) last = max(last, j);
        VI lv{float(last), last};
        lv = block_best(lv, shv);
        res = lv.i;
      }
      __syncthreads();
      bonus = res;
    }
  } else if (ts.tau == 0.0) {
    bonus = tst.argmax;  // residual of one-hot target against any draft law
  } else {
    // residual max(p_t - p_d, 0), normalised (categorical.cpp:94-110)
    const float* zd = uni ? nullptr : st->spec_rows[k];
    const RowStat& dst = rs[K + 1 + k];
    auto resid = [&](int j) {
      const double pt = row_prob(zt, j, ts, tst);
      const double pd = uni ? inv_v : row_prob(zd, j, ds, dst);
      return fmax(pt - pd, 0.0);
    };
    const int chunk = (V + blockDim.x - 1) / blockDim.x;
    const int b0 = min(V, int(threadIdx.x) * chunk), b1 = min(V, b0 + chunk);
    double loc = 0.0;
    for (int j = b0; j < b1; ++j) loc += resid(j);
    const double R = block_sum(loc, shd);
    if (!(R > 0.0)) {
      if (threadIdx.x == 0) s_err = 3;
      bonus = 0;
    } else {
      double pm = 0.0;
      for (int j = b0; j < b1; ++j) pm += resid(j) / R;
      __shared__ double wsum[32];
      __shared__ int pick;
      const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
      double incl = pm;
      for (int o = 1; o < 32; o <<= 1) { const double t = __shfl_up_sync(0xffffffffu, incl, o); if (lane >= o) incl += t; }
      __syncthreads();
      if (lane == 31) wsum[w] = incl;
      if (threadIdx.x == 0) pick = 0x7fffffff;
      __syncthreads();
      double before = 0.0;
      for (int i = 0; i < w; ++i) before += wsum[i];
      const double ex = before + incl - pm;
      if (b0 < b1 && u < ex + pm) atomicMin(&pick, int(threadIdx.x));
      __syncthreads();
      __shared__ int res;
      if (int(threadIdx.x) == pick) {
        double c = ex;
        int r = b1 - 1;
        for (int j = b0; j < b1; ++j) { c += resid(j) / R; if (u < c) { r = j; break; } }
        res = r;
      }
      __syncthreads();
      if (pick == 0x7fffffff) {
        int last = -1;
        for (int j = threadIdx.x; j < V; j += blockDim.x) if (resid(j) > 0.0) last = max(last, j);
        VI lv{float(last), last};
        lv = block_best(lv, shv);
        res = lv.i;
      }
      __syncthreads();
      bonus = res;
    }
  }
  if (threadIdx.x == 0) {
    if (s_err == 1) st->error = 1;
    if (s_err == 3) st->error = 3;
    st->out_k = k;
    st->out_t = bonus;
    const int n = st->n;
    for (int i = 0; i < k; ++i) hist[n + i] = st->spec[i];
    hist[n + k] = bonus;
    st->tokens += k + 1;
    st->accepted_sum += double(k);
  }
}

// ------------------------------------------------------------------ prep
// Chain inputs [hist[n-1], spec[0..M-2]] at positions n-1 .. (verify /
// extend / AR step). Causal visibility over the main cache. grid = batch
// lanes: lane l fills rows [l*M, (l+1)*M) from st[l] and its history, its
// main KV slots starting at l * lane_slots.
__global__ void prep_chain_kernel(const LoopState* __restrict__ st, const int* __restrict__ hist, FwdParams* P, int M,
                                  int hist_stride, int lane_slots, KvMap km) {
  const int l = blockIdx.x, m = threadIdx.x;
  if (m >= M) return;
  st += l;
  hist += size_t(l) * hist_stride;
  const int n = st->n;
  const int tok = m == 0 ? hist[n - 1] : st->spec[m - 1];
  const int pos = n - 1 + m, r = l * M + m, mb = l * lane_slots;
  P->tokens[r] = tok; P->pos[r] = pos; P->slot[r] = main_slot(km, mb, pos);
  P->main_len[r] = pos + 1; P->bbase[r] = 0; P->blen[r] = 0; P->mbase[r] = mb;
}

// Draft step i of specdec::draft: input hist[n-1] (i == 0) or spec[i-1].
// Row m drafts for lane lanes[m] (lanes == nullptr: lane 0, one row).
__global__ void prep_draft_step_kernel(const LoopState* __restrict__ st, const int* __restrict__ hist, FwdParams* P, int i,
                                       const int* __restrict__ lanes, int nl, int hist_stride, int lane_slots,
                                       KvMap km) {
  const int m = threadIdx.x;
  if (m >= (lanes ? nl : 1)) return;
  const int l = lanes ? lanes[m] : 0;
  st += l;
  hist += size_t(l) * hist_stride;
  const int n = st->n;
  const int pos = n - 1 + i, mb = l * lane_slots;
  P->tokens[m] = i == 0 ? hist[n - 1] : st->spec[i - 1];
  P->pos[m] = pos; P->slot[m] = main_slot(km, mb, pos); P->main_len[m] = pos + 1; P->bbase[m] = 0; P->blen[m] = 0;
  P->mbase[m] = mb;
}

// Prefill of hist[lo, hi) (chunked by the caller, M <= kMaxM) into the main
// KV slots starting at mb.
__global__ void prep_prefill_kernel(const int* __restrict__ hist, FwdParams* P, int lo, int M, int mb, KvMap km) {
  const int m = threadIdx.x;
  if (m >= M) return;
  const int pos = lo + m;
  P->tokens[m] = hist[pos]; P->pos[m] = pos; P->slot[m] = main_slot(km, mb, pos);
  P->main_len[m] = pos + 1; P->bbase[m] = 0; P->blen[m] = 0; P->mbase[m] = mb;
}

// Branch step j (cache.cpp:258-268 continuation drafts, batched): branch b
// = (k_b, t_b) continues prefix hist ++ spec[0..k_b) with t_b, then its own
// drafted tokens. KV of branch-local tokens lives in slots
// kv_base + b*K + j; its attention sees main slots [0, n + k_b) plus its own
// branch slots.
// Batch lanes (bper > 0): branch b belongs to lane b / bper, whose KV slots
// start at lane * lane_slots (main) and lane * lane_slots + kv_base (branches).
__global__ void prep_branch_kernel(const LoopState* __restrict__ st, const int* __restrict__ bk, const int* __restrict__ btok,
                                   const int* __restrict__ bt /* [B][K] */, FwdParams* P, int B, int j, int kv_base,
                                   int bper, int lane_slots) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int l = bper > 0 ? b / bper : 0, lb = bper > 0 ? b - l * bper : b;
  st += l;
  const int K = st->Kb, n = st->n, k = bk[b];
  const int mb = l * lane_slots, bb = mb + kv_base + lb * K;
  P->tokens[b] = j == 0 ? btok[b] : bt[b * K + j - 1];
  P->pos[b] = n + k + j;
  P->slot[b] = bb + j;
  P->main_len[b] = n + k;
  P->bbase[b] = bb;
  P->blen[b] = j + 1;
  P->mbase[b] = mb;
}

// Per-branch streams: base = one next_u64 of the draft stream (cache.cpp:245),
// branch b draws K uniforms from Stream(derive_seed(base, b)) (cache.cpp:264).
// grid = batch lanes (lane l: st[l], bu rows [l*B, (l+1)*B)).
__global__ void branch_streams_kernel(LoopState* st, int B, double* __restrict__ bu /* [B][K] */, int need) {
  __shared__ uint64_t base;
  st += blockIdx.x;
  bu += size_t(blockIdx.x) * B * st->Kb;
  if (threadIdx.x == 0) base = mt_next(st->drng);
  __syncthreads();
  if (!need) return;
  const int K = st->Kb;
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    Mt64 m;
    mt_seed(m, derive_seed(base, uint64_t(b)));
    for (int j = 0; j < K; ++j) bu[b * K + j] = mt_unit(m);
  }
}

// Lookup + backup + bookkeeping: the draft side's handle_outcomes
// (sim.cpp:418-463) and the harness clock (sim.cpp:528-577).
// cum: exact sequential fp64 cumulative of the uniform law (categorical.cpp
// :133-138 on a vector of 1/V), for the FastRandom tokens (sim.cpp:35-48).
// Branch sharding: this engine decodes branches [lo, lo + Bl)
// of the B keyed ones; bt / brows hold only those ([Bl][K], [K][Bl][V]).
// Per-round transcript log (sim.cpp:271-317 Channel, 489-500 to_jsonl):
// ints [round][lane][kTrInts] = (k, t, hit, emitted so far, next spec[K]),
// doubles [round][2] = (v2d vclock, d2v vclock).
constexpr int kTrInts = 4 + kMaxK;
struct TrLog {
  int* i;
  double* d;
  int n0;  // prompt length (seq_lens count emitted tokens)
};

// mode: 0 run_protocol_harness (sim.cpp:502-601: verifier / draft streams,
// cache ready at v0 + T_p, clock = all hit ? max(v1, ready) : v1 + T_b),
// 1 run_ssd_batch (sim.cpp:128-250: one stream per sequence, clock +=
// previous all hit ? max(1, T_p) : 1 + T_b).
__global__ void lookup_kernel(LoopState* st, int nb, const int* __restrict__ keys, int max_f,
                              const int* __restrict__ off2, const int* __restrict__ bt, const float* __restrict__ brows,
                              int lo, int Bl, int bper, int V, const double* __restrict__ cum,
                              int* __restrict__ log_outcomes, int* __restrict__ log_hits, int mode, TrLog tr) {
  if (threadIdx.x != 0) return;
  // Batch lanes (sim.cpp:548-577): every lane looks up its own outcome; the
  // round's virtual clock stalls the whole batch for the backup when any
  // lane missed. Per-round logs follow lane 0 (the harness' outcomes0 /
  // hits0).
  const double v0 = st[0].clock, v1 = v0 + 1.0, ready = v0 + st[0].primary_time;
  const int r = st[0].round;  // 0-based round being closed
  const bool last = r + 1 >= st[0].rounds;  // last round: no lookup, no backup
  // harness overlap invariant (sim.cpp:534-537)
  if (mode == 0 && st[0].primary_time < 1.0 && ready >= v1) {
    for (int l = 0; l < nb; ++l) st[l].error = 11;
    return;
  }
  bool all_hit = true;
  for (int l = 0; l < nb; ++l) {
    LoopState* s = st + l;
    const int K = s->K;
    const int k = s->out_k, t = s->out_t;
    // tokens attributed to the source of the verified speculation
    const long long emitted = k + 1;
    if (s->spec_src == 0) s->initial_rounds++;
    else if (s->spec_src == 1) { s->hit_rounds++; s->hit_round_tokens += emitted; }
    else { s->miss_rounds++; s->miss_round_tokens += emitted; }
    if (l == 0 && log_outcomes) { log_outcomes[2 * r] = k; log_outcomes[2 * r + 1] = t; }
    s->n += k + 1;
    s->round = r + 1;
    int* tl = tr.i ? tr.i + (size_t(r) * nb + l) * kTrInts : nullptr;
    if (tl) { tl[0] = k; tl[1] = t; tl[2] = 0; tl[3] = s->n - tr.n0; }
    if (last) {
      if (l == 0 && log_hits) log_hits[r] = -1;
      continue;
    }
    // the key table was built under the in-flight speculation's plan
    const int origin = s->spec_origin;
    const int* kl = keys + size_t(l) * (K + 1) * max_f;
    int b = -1;
    for (int j = 0; j < max_f; ++j)
      if (kl[k * max_f + j] == t) { b = l * bper + off2[origin * (K + 1) + k] + j; break; }
    const bool hit = b >= 0;
    const bool from_primary = origin == 0;
    if (from_primary) { s->p_lookups++; s->p_hits += hit; } else { s->b_lookups++; s->b_hits += hit; }
    if (l == 0 && log_hits) log_hits[r] = hit ? 1 : 0;
    s->hit = hit;
    if (hit) {
      const int lb = b - lo;
      s->own = lb >= 0 && lb < Bl;
      if (s->own) {  // otherwise the owning speculator broadcasts the tokens
        for (int i = 0; i < K; ++i) {
          s->spec[i] = bt[lb * K + i];
          s->spec_rows[i] = brows + (size_t(i) * Bl + lb) * size_t(V);
        }
      }
      s->spec_origin = 0; s->spec_src = 1; s->spec_uniform = 0;
    } else {
      all_hit = false;
      s->own = 0;
      s->spec_origin = 1; s->spec_src = 2;
      if (s->backup_kind == 1) {  // FastRandom: K uniform draws, exact CDF
        for (int i = 0; i < K; ++i) {
          const double u = mt_unit(s->drng);
          int a = 0, z = V;  // first idx with u < cum[idx]
          while (a < z) { const int mid = (a + z) >> 1; if (u < cum[mid]) z = mid; else a = mid + 1; }
          s->spec[i] = a < V ? a : V - 1;
          s->spec_rows[i] = nullptr;
        }
        s->spec_uniform = 1;
      } else {
        s->spec_uniform = 0;  // the host runs the JIT re-draft
      }
    }
    if (tl) {
      tl[2] = hit ? 1 : 0;
      for (int i = 0; i < K; ++i) tl[4 + i] = s->spec[i];  // JIT lanes: rewritten after the re-draft
    }
  }
  double clock;
  if (mode == 1) clock = last ? v0 : v0 + (all_hit ? fmax(1.0, st[0].primary_time) : 1.0 + st[0].backup_time);
  else clock = last ? v1 : (all_hit ? fmax(v1, ready) : v1 + st[0].backup_time);
  for (int l = 0; l < nb; ++l) st[l].clock = clock;
  if (tr.d) { tr.d[2 * r] = mode == 1 ? v0 : v1; tr.d[2 * r + 1] = clock; }
}

// Pre-speculation session (ssd_prespec_begin): origin of the in-flight
// speculation and the entries' continuation length, set on the device so the
// call needs no host round trip.
__global__ void set_spec_origin_kernel(LoopState* st, int origin, int Kb) {
  if (threadIdx.x != 0) return;
  st->spec_origin = origin;
  st->Kb = Kb;
}

// Transcript: the speculation each listed lane sends after a JIT re-draft.
__global__ void tr_log_spec_kernel(const LoopState* st, const int* __restrict__ lanes, int nl, int nb, TrLog tr) {
  if (threadIdx.x != 0 || !tr.i) return;
  for (int m = 0; m < nl; ++m) {
    const LoopState* s = st + lanes[m];
    int* tl = tr.i + (size_t(s->round - 1) * nb + lanes[m]) * kTrInts;
    for (int i = 0; i < s->K; ++i) tl[4 + i] = s->spec[i];
  }
}

// After a JIT / initial draft of spec[] from rows: origin bookkeeping.
__global__ void set_spec_rows_kernel(LoopState* st, const float* __restrict__ rows, int V, int origin, int src) {
  if (threadIdx.x != 0) return;
  for (int i = 0; i < st->K; ++i) st->spec_rows[i] = rows + size_t(i) * V;
  st->spec_origin = origin; st->spec_src = src; st->spec_uniform = 0;
}

// Batched draft (the initial drafts and the JIT backups of a batch): row m of
// draft step i drafted lane lanes[m]; its row is rows[(i * row_step + m) * V].
__global__ void set_lane_spec_rows_kernel(LoopState* st, const int* __restrict__ lanes, int nl, const float* __restrict__ rows,
                                          int row_step, int V, int origin, int src) {
  const int m = threadIdx.x;
  if (m >= nl) return;
  LoopState* s = st + lanes[m];
  for (int i = 0; i < s->K; ++i) s->spec_rows[i] = rows + (size_t(i) * row_step + m) * V;
  s->spec_origin = origin; s->spec_src = src; s->spec_uniform = 0;
}

// One uniform per row from its lane's draft stream (specdec.cpp:19).
__global__ void draw_lane_uniforms_kernel(LoopState* st, const int* __restrict__ lanes, int nl, double* u) {
  if (threadIdx.x == 0)
    for (int m = 0; m < nl; ++m) u[m] = mt_unit(st[lanes[m]].drng);
}

// Scatter the tokens drawn for rows m into st[lanes[m]].spec[i].
__global__ void scatter_spec_kernel(LoopState* st, const int* __restrict__ lanes, int nl, int i, const int* __restrict__ tok) {
  const int m = threadIdx.x;
  if (m < nl) st[lanes[m]].spec[i] = tok[m];
}

// SD / AR commit: n += k + 1 (history already appended by verify).
__global__ void commit_kernel(LoopState* st) {
  if (threadIdx.x == 0) { st->n += st->out_k + 1; st->round += 1; }
}

// AR: append sampled token.
__global__ void ar_commit_kernel(LoopState* st, int* hist, const int* tok) {
  if (threadIdx.x == 0) { hist[st->n] = tok[0]; st->n += 1; st->tokens += 1; st->round += 1; }
}

// Read-only HBM streaming probe (the achievable read bandwidth).
__global__ void __launch_bounds__(512) read_bw_kernel(const uint4* __restrict__ p, size_t n, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
  for (; i + 7 * stride < n; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = ldg_stream(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) { acc.x ^= v[u].x; acc.y ^= v[u].y; acc.z ^= v[u].z; acc.w ^= v[u].w; }
  }
  for (; i < n; i += stride) { const uint4 v = ldg_stream(p + i); acc.x ^= v.x; }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) *sink = acc;
}

__global__ void mt_init_kernel(Mt64* m, uint64_t seed) {
  if (threadIdx.x == 0) mt_seed(*m, seed);
}

__global__ void mt_draw_kernel(Mt64* m, int n, uint64_t* out) {
  if (threadIdx.x == 0) for (int i = 0; i < n; ++i) out[i] = mt_next(*m);
}

}  // namespace ssd
