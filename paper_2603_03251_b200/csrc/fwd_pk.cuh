// Persistent forward kernel ("pk"): ONE launch runs a whole decode / verify
// / branch step of a model for M <= 32 tokens — embedding, every layer's
// QKV, attention, O, gate/up, down, and the LM head (
// DESIGN.md §4).
//
// Why: a 1B draft step as separate kernels is ~115 dependent launches whose
// fixed costs (launch, ring ramp, split-K drain, PDL hop; ~5-10 us each)
// exceed the weight bytes of its small GEMMs (1.3-10 us at HBM speed). Here
// every SM runs one CTA for the whole step and the weight stream never stops
// at an op boundary: the producer warp issues the bulk copies of every GEMM
// back to back into one shared-memory ring. Only consumers wait on data
// dependencies, through per-op completion counters (dataflow, no grid
// barrier): op p's input needs op p-1 complete, i.e. every CTA has released
// its part of op p-1 (counters striped over 8 cache lines).
//
// Split-K: the stream-K segments of a tile accumulate into their fp32
// target with red.global.add (no partials, no last-arriver reduction round
// trips); targets are zero-filled by an earlier op of the same launch, once
// their last reader is complete; the residual stream x accumulates in place. Summation order is therefore not fixed (the split
// speculator roles, which must agree bit for bit, use the per-op path).
//
// RMSNorm: op NORM (one CTA per token) turns the final x rows into row scales
// rs[m] = 1 / sqrt(mean(x^2) + eps); the B-operand warps of the next normed
// GEMM write bf16(x * rs * gain) straight into the swizzled shared-memory
// tile (no normalised copy of x). SwiGLU is an elementwise op (SWIGLU) over
// the accumulated gate/up columns.
//
// Attention: op APPEND writes this forward's RoPE'd K and V rows (bf16) to
// the cache, then op ATTN runs items (kv head, key chunk, query block) over
// the CTAs on the 4 epilogue warps: every K / V row is loaded once per block
// of 16 (query, head) rows (the tree mask: shared main prefix, per-query
// lengths and branch tails), online softmax over 64-key passes, chunk
// partials merged by the last-arriving chunk.
//
// Warp roles (256 threads): w0 weight producer (+ L2 look-ahead), w1
// tcgen05.mma issuer (TMEM double buffer), w2-5 epilogue / attention /
// embedding / zero-fill, w6-7 B-operand producers (alternating units). The
// GEMM is gemm_tc.cuh's (swap-AB, pre-tiled K-major SWIZZLE_128B weights,
// persistent stream-K over (tile, unit)).
#pragma once

#include "gemm_tc.cuh"

namespace ssd {
namespace pk {

using tc::kABlock;
using tc::kABytes;
using tc::kBK;
using tc::kBM;
using tc::kKPS;

enum PkKind { OP_EMBED = 0, OP_GEMM = 1, OP_ATTN = 2, OP_SWIGLU = 3, OP_APPEND = 4, OP_NORM = 5 };
enum PkIn { IN_NORM = 0, IN_BF16 = 1 };

constexpr int kMaxTok = 32;   // tokens per forward
constexpr int kThreads = 256;
constexpr int kStripes = 8;   // completion counter stripes (CTA % kStripes)
constexpr int kLine = 32;     // ints per 128-byte line: one counter per line

struct PkOp {
  int kind;
  // ---- GEMM: out[m][n] (+)= sum_k W[n][k] B[m][k]
  const bf16* W;        // pre-tiled weights [N][K]
  int N, KU;            // rows, units per tile (K / 128)
  int in;               // IN_NORM: rmsnorm(x) * gain; IN_BF16: bf16 src
  const float* gain;    // IN_NORM gain (null: none)
  const bf16* src;      // IN_BF16 input [maxM][ld_src]
  int ld_src;
  // ---- SWIGLU: act[m][j] = silu(gu[m][2j]) * gu[m][2j + 1], j < ffn
  const float* gu;
  bf16* act;
  int ffn;
  float* out;           // fp32 accumulation target [M][ld_out] (zeroed, or the residual stream)
  int ld_out;
  // ---- zero-fill duty, run by every CTA's epilogue warps when it reaches this
  // op, once op zero_after (the buffer's last reader, -1: none) is complete
  float* zero;
  int zero_ld, zero_cols;  // rows [0, M) x cols [0, zero_cols) of a [.][zero_ld] buffer
  int zero_after;
  // ---- ATTN
  bf16* kc;             // this layer's cache [KVH][S][HD]
  bf16* vc;
  const float* qkv;     // accumulated QKV rows [M][(H + 2 KVH) HD]
  bf16* attn;           // output [M][H HD]
};

struct PkArgs {
  const PkOp* ops;
  int n_ops;
  int M;
  const FwdParams* P;
  const bf16* embed;
  int embed_tiled;
  int d, H, KVH, S;
  float eps, scale;
  const float* rope_cos;
  const float* rope_sin;
  float* x;             // residual stream [maxM][d] fp32
  float* rs;            // [kMaxTok] row scales 1 / sqrt(mean(x^2) + eps) of the last NORM (or EMBED)
  float* logits;        // accumulation target of a GEMM op whose out is null (the LM head; zeroed by its op)
  int chunk;            // attention main keys per chunk (a multiple of kKeysPass; chunks <= kMaxChunks)
  int* done;            // [n_ops][kStripes][kLine] completion counters + [kLine] exit count
  int* attn_cnt;        // [KVH * kMaxTok query blocks][kLine] chunk arrival counters (self-resetting)
  float* attn_part;     // [KVH][kMaxTok query blocks][kMaxChunks][kRows HD + 2 kRows] chunk partials
  int pf_units;         // L2 look-ahead of the weight stream beyond the ring (32 KB units)
  unsigned long long* trace;  // profiling (SSD_B200_PK_TRACE): [grid][kTrSlots] stamps, or null
  int trace_ops;        // ops traced (first trace_ops of the launch)
};

// Trace slots per CTA: 0 entry, 1 exit, then per traced op p (base 2 + 6 p):
// 0 weight copies start, 1 end, 2 input dependency met (B warps / attention),
// 3 first MMA, 4 last MMA, 5 epilogue / attention of the op done.
constexpr int kTrOps = 16;
constexpr int kTrSlots = 2 + 6 * kTrOps;

template <int NP, int HD, int G>
struct Cfg {
  static constexpr int kBBlock = NP * kBK * 2;
  static constexpr int kBBytes = kBBlock * kKPS;
  static constexpr int kStageBytes = kABytes + kBBytes;
  // attention scratch (AttnSm): V rows [64][HD] bf16, query rows [16][HD],
  // probabilities [16][64], row state; aliased onto the B ring when it fits
  // (no B tile is in flight while a CTA runs attention items: the next
  // GEMM's B operand waits for the whole attention op)
  static constexpr int kAttnBytes = 64 * HD * 2 + 16 * HD * 4 + 16 * 64 * 4 + 3 * 16 * 4 + 8 * 4;  // attn_smem_bytes<HD>()
  static constexpr int kMisc = 1024;
  static constexpr int kBudget = 227 * 1024 - 1024 - kMisc;
  static constexpr int kStages0 = kBudget / kStageBytes > 6 ? 6 : kBudget / kStageBytes;
  static constexpr bool kAlias = kStages0 * kBBytes >= kAttnBytes;
  static constexpr int kStages1 = kAlias ? kStages0 : (kBudget - kAttnBytes) / kStageBytes;
  static constexpr int S = kStages1 > 6 ? 6 : kStages1;
  static_assert(S >= 3, "pk: shared memory");
  static constexpr int kAccCols = NP < 32 ? 32 : NP;
  static constexpr int kTmemCols = 2 * kAccCols <= 64 ? 64 : 128;
  static constexpr size_t kSmem = 1024 + size_t(S) * kStageBytes + (kAlias ? 0 : kAttnBytes) + kMisc;
};

constexpr unsigned long long kWatchNs = 4000000000ull;  // a wait beyond this is a protocol bug: trap
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __noinline__ void watch_fail(int code, int aux) {
  printf("pk watchdog: block %d thread %d code %d aux %d\n", blockIdx.x, threadIdx.x, code, aux);
  __trap();
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_add_f32(float* p, float v) {
  asm volatile("red.relaxed.gpu.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
// Whole warp: spin until op p is complete (every CTA released its part).
__device__ __forceinline__ void wait_op(const PkArgs& a, int p, int code) {
  if (p < 0) return;
  const int lane = threadIdx.x & 31;
  const int* c = a.done + (size_t(p) * kStripes + (lane & (kStripes - 1))) * kLine;
  const int target = int(gridDim.x);
  unsigned long long t0 = 0;
  while (true) {
    int v = lane < kStripes ? ld_acquire(c) : 0;
    v = warp_sum(v);
    if (v >= target) break;
    const unsigned long long t = gtimer();
    if (!t0) t0 = t;
    else if (t - t0 > kWatchNs) watch_fail(code, p);
  }
  __syncwarp();
}
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t parity, int code) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok) : "r"(tc::smem_u32(b)), "r"(parity) : "memory");
  if (ok) return;
  const unsigned long long t0 = gtimer();
  while (true) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok) : "r"(tc::smem_u32(b)), "r"(parity) : "memory");
    if (ok) return;
    if (gtimer() - t0 > kWatchNs) watch_fail(code, int(parity));
  }
}
__device__ __forceinline__ void tr(const PkArgs& a, int p, int slot) {
  if (a.trace && p < a.trace_ops && p < kTrOps) a.trace[size_t(blockIdx.x) * kTrSlots + 2 + 6 * p + slot] = gtimer();
}
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
__device__ __forceinline__ void bprod_sync() { asm volatile("bar.sync 2, 64;" ::: "memory"); }

__device__ __forceinline__ int op_tiles(const PkOp& o) { return (o.N + kBM - 1) / kBM; }
// Stream-K partition (32-bit): CTA i owns units [ub(i), ub(i + 1)).
__device__ __forceinline__ int ub(int i, int U, int P) { return int(unsigned(i) * unsigned(U) / unsigned(P)); }

__device__ __forceinline__ uint4 pack8(const float* f) {
  __nv_bfloat162 b[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) b[j] = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
  return *reinterpret_cast<uint4*>(b);
}

// RoPE'd element d of a head row x (fp32): attention_dec's rope_elem.
__device__ __forceinline__ float rope_at(const float* x, int d, int half, const float* c, const float* s) {
  if (d < half) return __fsub_rn(__fmul_rn(__ldcg(x + d), c[d]), __fmul_rn(__ldcg(x + d + half), s[d]));
  const int i = d - half;
  return __fadd_rn(__fmul_rn(__ldcg(x + d), c[i]), __fmul_rn(__ldcg(x + i), s[i]));
}

// ---------------------------------------------------------------- attention
// Items (kv head, key chunk, query block): a block is kRows / G queries, i.e.
// kRows rows (query, head) that share every K / V row of a pass (branch steps:
// all branches see the same main prefix; verify / extend chains: the same
// slots under per-query length masks). A pass covers kKeysPass main keys;
// chunk 0 also runs the tail pass over each query's own branch keys. Rows
// keep online-softmax state; chunk partials are merged by the last arriver.
constexpr int kRows = 16;
constexpr int kKeysPass = 64;
constexpr int kMaxChunks = 16;

struct AttnSm {
  bf16* vs;      // [kKeysPass][HD]
  float* qs;     // [kRows][HD]
  float* ps;     // [kRows][kKeysPass]
  float* rmax;   // [kRows] running max
  float* rsum;   // [kRows] running sum
  float* ralpha; // [kRows] rescale of this pass
  int* misc;     // [8]
};
template <int HD>
__host__ __device__ constexpr int attn_smem_bytes() {
  return kKeysPass * HD * 2 + kRows * HD * 4 + kRows * kKeysPass * 4 + 3 * kRows * 4 + 8 * 4;
}

template <int HD, int G>
__device__ void attn_item(const PkArgs& a, const PkOp& o, int kvh, int c, int qb, int nch_eff, int chunk,
                          const AttnSm& sm, int tid) {
  constexpr int HALF = HD / 2;
  constexpr int QB = kRows / G;
  constexpr int OPT = kRows * HD / 128;  // outputs per thread: rows (tid / HD) + (128 / HD) i, dim tid % HD
  constexpr int RSTEP = 128 / HD;
  const int lane = tid & 31, warp = tid >> 5;
  const FwdParams* P = a.P;
  const int q0 = qb * QB, q1 = min(a.M, q0 + QB);
  const size_t row_len = size_t(a.H + 2 * a.KVH) * HD;
  // 1) rotated, scaled query rows; row state
  for (int e = tid; e < kRows * HD; e += 128) {
    const int r = e / HD, d = e % HD, m = q0 + r / G;
    float v = 0.f;
    if (m < q1) {
      const int pos = P->pos[m];
      v = rope_at(o.qkv + size_t(m) * row_len + size_t(kvh * G + r % G) * HD, d, HALF, a.rope_cos + size_t(pos) * HALF,
                  a.rope_sin + size_t(pos) * HALF) * a.scale;
    }
    sm.qs[e] = v;
  }
  if (tid < kRows) { sm.rmax[tid] = -INFINITY; sm.rsum[tid] = 0.f; }
  float acc[OPT];
#pragma unroll
  for (int i = 0; i < OPT; ++i) acc[i] = 0.f;
  const bf16* kb = o.kc + size_t(kvh) * a.S * HD;
  const bf16* vb = o.vc + size_t(kvh) * a.S * HD;
  const int kk = tid % kKeysPass, h = tid / kKeysPass;  // key of the pass, row half (rows 8 h .. 8 h + 7)
  // passes: main keys of chunk c (sub-blocks of equal mbase), then (chunk 0) the tail
  int m = q0;
  bool tail = false;
  int j0 = 0, jend = 0, mb = 0, sb0 = q0, sbe = q0, tb = 0;
  // the next (sub-block of equal mbase, key range) span; every thread
  // derives the same sequence
  auto next_span = [&]() -> bool {
    while (true) {
      if (j0 < jend) return true;
      if (tail) return false;
      if (m >= q1) {
        if (c != 0) return false;
        tail = true;
        j0 = 0;
        tb = 0;
        for (int mm = q0; mm < q1; ++mm) tb = max(tb, P->blen[mm]);
        jend = tb * (q1 - q0);  // tail pairs (query, branch key), blocked by query
        sb0 = q0;
        sbe = q1;
        continue;
      }
      mb = P->mbase[m];
      sb0 = m;
      int ml = 0;
      while (m < q1 && P->mbase[m] == mb) { ml = max(ml, P->main_len[m]); ++m; }
      sbe = m;
      j0 = c * chunk;
      jend = min(ml, (c + 1) * chunk);
    }
  };
  epi_sync();
  while (next_span()) {
    const int jj = j0 + kk;
    // 2) this thread's key: slot and the queries that see it
    int slot = -1, only = -1;
    if (jj < jend) {
      if (!tail) {
        slot = mb + jj;
      } else {
        const int qm = q0 + jj / tb, bi = jj % tb;
        if (bi < P->blen[qm]) { slot = P->bbase[qm] + bi; only = qm; }
      }
    }
    // V row into smem (the two row halves load one half of the row each), K row scores
    {
      uint4* vdst = reinterpret_cast<uint4*>(sm.vs + size_t(kk) * HD);
      constexpr int NV = HD / 16;
#pragma unroll
      for (int i = 0; i < NV; ++i)
        vdst[h * NV + i] = slot >= 0 ? __ldcg(reinterpret_cast<const uint4*>(vb + size_t(slot) * HD) + h * NV + i)
                                     : make_uint4(0u, 0u, 0u, 0u);
    }
    float sc[kRows / 2];
#pragma unroll
    for (int r = 0; r < kRows / 2; ++r) sc[r] = 0.f;
    if (slot >= 0) {
      const uint4* ks = reinterpret_cast<const uint4*>(kb + size_t(slot) * HD);
      constexpr int KG = HD / 8 < 8 ? HD / 8 : 8;
#pragma unroll
      for (int i0 = 0; i0 < HD / 8; i0 += KG) {
        uint4 kr[KG];
#pragma unroll
        for (int i = 0; i < KG; ++i) kr[i] = __ldcg(ks + i0 + i);
#pragma unroll
        for (int i = 0; i < KG; ++i) {
          float kf[8];
          bf16x8_to_f32(kr[i], kf);
#pragma unroll
          for (int r = 0; r < kRows / 2; ++r) {
            const float4* q4 = reinterpret_cast<const float4*>(sm.qs + (h * (kRows / 2) + r) * HD + 8 * (i0 + i));
            const float4 qa = q4[0], qb4 = q4[1];
            sc[r] = fmaf(qa.x, kf[0], fmaf(qa.y, kf[1], fmaf(qa.z, kf[2], fmaf(qa.w, kf[3], sc[r]))));
            sc[r] = fmaf(qb4.x, kf[4], fmaf(qb4.y, kf[5], fmaf(qb4.z, kf[6], fmaf(qb4.w, kf[7], sc[r]))));
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kRows / 2; ++r) {
      const int row = h * (kRows / 2) + r, qm = q0 + row / G;
      bool vis = slot >= 0 && qm >= sb0 && qm < sbe && (only < 0 ? jj < P->main_len[qm] : qm == only);
      sm.ps[row * kKeysPass + kk] = vis ? sc[r] : -INFINITY;
    }
    epi_sync();
    // 3) online softmax, one warp per 4 rows (lanes own keys lane, lane + 32)
#pragma unroll
    for (int rr = 0; rr < kRows / 4; ++rr) {
      const int row = warp * (kRows / 4) + rr;
      float* pr = sm.ps + row * kKeysPass;
      const float s0 = pr[lane], s1 = pr[lane + 32];
      const float pm = warp_max(fmaxf(s0, s1));
      const float mo = sm.rmax[row];
      const float mn = fmaxf(mo, pm);
      const float p0 = s0 == -INFINITY ? 0.f : expf(s0 - mn), p1 = s1 == -INFINITY ? 0.f : expf(s1 - mn);
      pr[lane] = p0;
      pr[lane + 32] = p1;
      const float ts = warp_sum(p0 + p1);
      if (lane == 0) {
        const float al = mo == -INFINITY ? 0.f : expf(mo - mn);
        sm.ralpha[row] = al;
        sm.rsum[row] = sm.rsum[row] * al + ts;
        sm.rmax[row] = mn;
      }
    }
    epi_sync();
    // 4) P.V
#pragma unroll
    for (int i = 0; i < OPT; ++i) {
      const int row = tid / HD + RSTEP * i, d = tid % HD;
      const float* pr = sm.ps + row * kKeysPass;
      float o0 = 0.f, o1 = 0.f;
#pragma unroll 4
      for (int k2 = 0; k2 < kKeysPass; k2 += 2) {
        o0 = fmaf(pr[k2], __bfloat162float(sm.vs[size_t(k2) * HD + d]), o0);
        o1 = fmaf(pr[k2 + 1], __bfloat162float(sm.vs[size_t(k2 + 1) * HD + d]), o1);
      }
      acc[i] = acc[i] * sm.ralpha[row] + (o0 + o1);
    }
    epi_sync();
    j0 += kKeysPass;
  }
  // 5) outputs: one chunk writes them; several merge through the last arriver
  const int nrows = (q1 - q0) * G;
  if (nch_eff == 1) {
#pragma unroll
    for (int i = 0; i < OPT; ++i) {
      const int row = tid / HD + RSTEP * i, d = tid % HD;
      if (row < nrows) {
        const int mm = q0 + row / G, g = row % G;
        const float den = sm.rsum[row];
        o.attn[size_t(mm) * a.H * HD + size_t(kvh * G + g) * HD + d] = __float2bfloat16_rn(den > 0.f ? acc[i] / den : 0.f);
      }
    }
    return;
  }
  constexpr int PS = kRows * HD + 2 * kRows;
  float* part = a.attn_part + (size_t(kvh) * kMaxTok + qb) * kMaxChunks * PS;
#pragma unroll
  for (int i = 0; i < OPT; ++i) __stcg(part + size_t(c) * PS + (tid / HD + RSTEP * i) * HD + tid % HD, acc[i]);
  if (tid < kRows) {
    __stcg(part + size_t(c) * PS + kRows * HD + 2 * tid, sm.rmax[tid]);
    __stcg(part + size_t(c) * PS + kRows * HD + 2 * tid + 1, sm.rsum[tid]);
  }
  epi_sync();
  int* cnt = a.attn_cnt + size_t(kvh * kMaxTok + qb) * kLine;
  if (tid == 0) {
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(cnt) : "memory");
    sm.misc[3] = old == nch_eff - 1;
  }
  epi_sync();
  if (!sm.misc[3]) return;
  // merge: chunk weights per row into smem (ps reused), then the outputs
  float* w = sm.ps;  // [kMaxChunks][kRows] weights, [kRows] denominators after
  if (tid < kRows) {
    float mx = -INFINITY;
    float mc[kMaxChunks], sc2[kMaxChunks];
#pragma unroll
    for (int c2 = 0; c2 < kMaxChunks; ++c2) {
      mc[c2] = c2 < nch_eff ? __ldcg(part + size_t(c2) * PS + kRows * HD + 2 * tid) : -INFINITY;
      sc2[c2] = c2 < nch_eff ? __ldcg(part + size_t(c2) * PS + kRows * HD + 2 * tid + 1) : 0.f;
    }
#pragma unroll
    for (int c2 = 0; c2 < kMaxChunks; ++c2) mx = fmaxf(mx, mc[c2]);
    float den = 0.f;
#pragma unroll
    for (int c2 = 0; c2 < kMaxChunks; ++c2) {
      const float wc = mc[c2] == -INFINITY ? 0.f : expf(mc[c2] - mx);
      w[c2 * kRows + tid] = wc;
      den += wc * sc2[c2];
    }
    w[kMaxChunks * kRows + tid] = den;
  }
  epi_sync();
#pragma unroll
  for (int i = 0; i < OPT; ++i) {
    const int row = tid / HD + RSTEP * i, d = tid % HD;
    float v[kMaxChunks];
#pragma unroll
    for (int c2 = 0; c2 < kMaxChunks; ++c2) v[c2] = c2 < nch_eff ? __ldcg(part + size_t(c2) * PS + row * HD + d) : 0.f;
    float num = 0.f;
#pragma unroll
    for (int c2 = 0; c2 < kMaxChunks; ++c2) num = fmaf(w[c2 * kRows + row], v[c2], num);
    if (row < nrows) {
      const int mm = q0 + row / G, g = row % G;
      const float den = w[kMaxChunks * kRows + row];
      o.attn[size_t(mm) * a.H * HD + size_t(kvh * G + g) * HD + d] = __float2bfloat16_rn(den > 0.f ? num / den : 0.f);
    }
  }
  epi_sync();
  if (tid == 0) *cnt = 0;
}

// ---------------------------------------------------------------- kernel
template <int NP, int HD, int G>
__global__ void __launch_bounds__(kThreads, 1) pk_kernel(const __grid_constant__ PkArgs a) {
  using C = Cfg<NP, HD, G>;
  constexpr int S = C::S;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * kABytes;
  uint8_t* sAttn = C::kAlias ? sB : sB + S * C::kBBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + S * C::kBBytes + (C::kAlias ? 0 : C::kAttnBytes));
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;   // [2]
  uint64_t* tempty = tfull + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  float* s_rs = reinterpret_cast<float*>(tmem_slot + 4);  // [kMaxTok] row scales of a normed B operand

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int P = gridDim.x;
  if (threadIdx.x == 0 && a.trace) a.trace[size_t(blockIdx.x) * kTrSlots] = gtimer();

  if (threadIdx.x == 0) {
    // full: the weight copy (expect_tx) + the 32 lanes of the B warp of that unit
    for (int s = 0; s < S; ++s) { tc::mbar_init(&full[s], 1 + 32); tc::mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { tc::mbar_init(&tfull[b], 1); tc::mbar_init(&tempty[b], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tmem_slot)),
                 "r"(C::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  tc::pdl_launch();

  if (warp == 0) {
    // ---------------- weight producer: every GEMM of the step, back to back
    if (lane == 0) {
      uint64_t pol_w;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_w));
      uint32_t it = 0, pit = 0;       // units loaded / L2-prefetched
      int pp = -1, pu = 0, pu1 = 0;   // prefetch cursor: op, unit range
      const bf16* pw = nullptr;
      for (int p = 0; p < a.n_ops; ++p) {
        const PkOp& op = a.ops[p];
        if (op.kind != OP_GEMM) continue;
        const int U = op_tiles(op) * op.KU;
        const int u0 = ub(blockIdx.x, U, P), u1 = ub(blockIdx.x + 1, U, P);
        tr(a, p, 0);
        for (int u = u0; u < u1; ++u, ++it) {
          const int s = int(it % S);
          while (pit < it + uint32_t(a.pf_units)) {  // keep HBM ahead of the ring through dependency waits
            if (pu >= pu1) {
              do { ++pp; } while (pp < a.n_ops && a.ops[pp].kind != OP_GEMM);
              if (pp >= a.n_ops) break;
              const PkOp& q = a.ops[pp];
              const int Uq = op_tiles(q) * q.KU;
              pu = ub(blockIdx.x, Uq, P);
              pu1 = ub(blockIdx.x + 1, Uq, P);
              pw = q.W;
              continue;
            }
            if (pit >= it + uint32_t(S))
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pw + size_t(pu) * (kABytes / 2)),
                           "r"(uint32_t(kABytes)) : "memory");
            ++pu;
            ++pit;
          }
          if (it >= uint32_t(S)) mwait(&empty[s], ((it / S) - 1) & 1, 1);
          tc::mbar_expect_tx(&full[s], kABytes);
          tc::bulk_load(sA + s * kABytes, op.W + size_t(u) * (kABytes / 2), kABytes, &full[s], pol_w);
        }
        tr(a, p, 1);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16(kBM, NP);
      uint32_t it = 0;
      int seg = -1;
      for (int p = 0; p < a.n_ops; ++p) {
        const PkOp& op = a.ops[p];
        if (op.kind != OP_GEMM) continue;
        const int U = op_tiles(op) * op.KU;
        const int u0 = ub(blockIdx.x, U, P), u1 = ub(blockIdx.x + 1, U, P);
        int cur_tile = -1;
        for (int u = u0; u < u1; ++u, ++it) {
          const int t = u / op.KU, s = int(it % S);
          const bool first = t != cur_tile;
          if (first) {
            ++seg;
            cur_tile = t;
            if (seg >= 2) mwait(&tempty[seg & 1], ((seg >> 1) - 1) & 1, 2);
          }
          mwait(&full[s], (it / S) & 1, 3);
          if (u == u0) tr(a, p, 3);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t dcol = tmem + uint32_t((seg & 1) * C::kAccCols);
#pragma unroll
          for (int h = 0; h < kKPS; ++h) {
            const uint32_t a0 = tc::smem_u32(sA + s * kABytes + h * kABlock);
            const uint32_t b0 = tc::smem_u32(sB + s * C::kBBytes + h * C::kBBlock);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              tc::mma_bf16(dcol, tc::sw128_desc(a0 + k * 32), tc::sw128_desc(b0 + k * 32), idesc,
                           (!first || h || k) ? 1u : 0u);
          }
          tc::mma_commit(&empty[s]);
          const bool last = (u + 1 == u1) || ((u + 1) / op.KU != t);
          if (last) tc::mma_commit(&tfull[seg & 1]);
        }
        if (u1 > u0) tr(a, p, 4);
      }
    }
  } else if (warp >= 6) {
    // ---------------- B-operand producers: warp 6 even units, warp 7 odd units
    const int bw = warp - 6, tid64 = threadIdx.x - 192;
    uint32_t it = 0;
    bool waited_pdl = false;
    for (int p = 0; p < a.n_ops; ++p) {
      const PkOp& op = a.ops[p];
      if (op.kind != OP_GEMM) continue;
      const int U = op_tiles(op) * op.KU;
      const int u0 = ub(blockIdx.x, U, P), u1 = ub(blockIdx.x + 1, U, P);
      if (u0 == u1) continue;
      if (!waited_pdl) { tc::pdl_wait(); waited_pdl = true; }
      wait_op(a, p - 1, 10);  // the input: op p - 1 complete (both warps poll)
      if (tid64 == 0) tr(a, p, 2);
      if (op.in == IN_NORM) {  // row scales of the preceding NORM op
        if (tid64 < a.M) s_rs[tid64] = __ldcg(a.rs + tid64);
        bprod_sync();
      }
      for (int u = u0; u < u1; ++u, ++it) {
        if (int(it & 1) != bw) continue;
        const int s = int(it % S);
        if (it >= uint32_t(S)) mwait(&empty[s], ((it / S) - 1) & 1, 4);
        const int col0 = (u % op.KU) * (kKPS * kBK);
        uint8_t* dst = sB + s * C::kBBytes;
        // NP x 16 chunks of 16 bytes (2 k-blocks x NP rows x 8 chunks) over 32
        // lanes; every load of the unit is issued before the first use.
        // SWIZZLE_128B K-major: row m's chunk c sits at position c ^ (m & 7).
        constexpr int CPL = NP * 8 * kKPS / 32;
        if (op.in == IN_NORM) {
          constexpr int CG = CPL < 8 ? CPL : 8;  // chunks per load group (register budget)
#pragma unroll
          for (int g0 = 0; g0 < CPL; g0 += CG) {
            float4 xv[CG][2];
#pragma unroll
            for (int i = 0; i < CG; ++i) {
              const int e = lane + 32 * (g0 + i), h = e / (NP * 8), rem = e % (NP * 8), m = rem >> 3, c = rem & 7;
              if (m < a.M) {
                const float4* xs = reinterpret_cast<const float4*>(a.x + size_t(m) * a.d + col0 + h * kBK + c * 8);
                xv[i][0] = __ldcg(xs);
                xv[i][1] = __ldcg(xs + 1);
              }
            }
#pragma unroll
            for (int i = 0; i < CG; ++i) {
              const int e = lane + 32 * (g0 + i), h = e / (NP * 8), rem = e % (NP * 8), m = rem >> 3, c = rem & 7;
              const int col = col0 + h * kBK + c * 8;
              uint4 val = make_uint4(0u, 0u, 0u, 0u);
              if (m < a.M) {
                const float rs = s_rs[m];
                float f[8] = {xv[i][0].x * rs, xv[i][0].y * rs, xv[i][0].z * rs, xv[i][0].w * rs,
                              xv[i][1].x * rs, xv[i][1].y * rs, xv[i][1].z * rs, xv[i][1].w * rs};
                if (op.gain) {
                  const float4 g0v = __ldg(reinterpret_cast<const float4*>(op.gain + col));
                  const float4 g1v = __ldg(reinterpret_cast<const float4*>(op.gain + col) + 1);
                  f[0] *= g0v.x; f[1] *= g0v.y; f[2] *= g0v.z; f[3] *= g0v.w;
                  f[4] *= g1v.x; f[5] *= g1v.y; f[6] *= g1v.z; f[7] *= g1v.w;
                }
                val = pack8(f);
              }
              *reinterpret_cast<uint4*>(dst + h * C::kBBlock + m * 128 + ((c ^ (m & 7)) << 4)) = val;
            }
          }
        } else {
          const bf16* src = op.src;
          uint4 bv[CPL];
#pragma unroll
          for (int i = 0; i < CPL; ++i) {
            const int e = lane + 32 * i, h = e / (NP * 8), rem = e % (NP * 8), m = rem >> 3, c = rem & 7;
            bv[i] = m < a.M ? __ldcg(reinterpret_cast<const uint4*>(src + size_t(m) * op.ld_src + col0 + h * kBK + c * 8))
                            : make_uint4(0u, 0u, 0u, 0u);
          }
#pragma unroll
          for (int i = 0; i < CPL; ++i) {
            const int e = lane + 32 * i, h = e / (NP * 8), rem = e % (NP * 8), m = rem >> 3, c = rem & 7;
            *reinterpret_cast<uint4*>(dst + h * C::kBBlock + m * 128 + ((c ^ (m & 7)) << 4)) = bv[i];
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc::mbar_arrive(&full[s]);
      }
    }
  } else {
    // ---------------- epilogue / attention / embedding / zero-fill (warps 2-5)
    const int tid = threadIdx.x - 64;
    const int q = warp & 3;
    const int rl = q * 32 + lane;
    int seg = -1;
    tc::pdl_wait();
    AttnSm sm;
    sm.vs = reinterpret_cast<bf16*>(sAttn);
    sm.qs = reinterpret_cast<float*>(sAttn + kKeysPass * HD * 2);
    sm.ps = sm.qs + kRows * HD;
    sm.rmax = sm.ps + kRows * kKeysPass;
    sm.rsum = sm.rmax + kRows;
    sm.ralpha = sm.rsum + kRows;
    sm.misc = reinterpret_cast<int*>(sm.ralpha + kRows);
    for (int p = 0; p < a.n_ops; ++p) {
      const PkOp& op = a.ops[p];
      // zero-fill duty of this op: this CTA's slice of rows [0, M) x cols [0, zero_cols)
      float* zbuf = op.zero == reinterpret_cast<float*>(1) ? a.logits : op.zero;  // (float*)1: the logits
      if (zbuf) {
        if (op.zero_after >= 0) {
          if (warp == 2) wait_op(a, op.zero_after, 30);
          epi_sync();
        }
        const int per_row = op.zero_cols / 4, total = a.M * per_row;
        const int lo = int((long long)blockIdx.x * total / P), hi = int((long long)(blockIdx.x + 1) * total / P);
        for (int i = lo + tid; i < hi; i += 128) {
          const int m = i / per_row, c4 = i % per_row;
          __stcg(reinterpret_cast<float4*>(zbuf + size_t(m) * op.zero_ld) + c4, make_float4(0.f, 0.f, 0.f, 0.f));
        }
      }
      if (op.kind == OP_EMBED || op.kind == OP_NORM) {
        // x rows (EMBED: from the table) and their row scales, one CTA per token
        if (op.kind == OP_NORM) {
          if (warp == 2) wait_op(a, p - 1, 50);
          epi_sync();
          if (tid == 0) tr(a, p, 2);
        }
        for (int m = blockIdx.x; m < a.M; m += P) {
          float ss = 0.f;
          if (op.kind == OP_EMBED) {
            const size_t tok = size_t(a.P->tokens[m]);
            for (int i = tid; i < a.d; i += 128) {
              const size_t at =
                  a.embed_tiled ? tiled_at(tok, size_t(i), size_t(a.d) / 64) : tok * size_t(a.d) + size_t(i);
              const float v = __bfloat162float(a.embed[at]);
              __stcg(a.x + size_t(m) * a.d + i, v);
              ss = fmaf(v, v, ss);
            }
          } else {
            const float4* xr = reinterpret_cast<const float4*>(a.x + size_t(m) * a.d);
            for (int i = tid; i < a.d / 4; i += 128) {
              const float4 v = __ldcg(xr + i);
              ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
            }
          }
          ss = warp_sum(ss);
          if (lane == 0) sm.rmax[q] = ss;
          epi_sync();
          if (tid == 0)
            __stcg(a.rs + m, 1.0f / sqrtf(((sm.rmax[0] + sm.rmax[1]) + (sm.rmax[2] + sm.rmax[3])) / float(a.d) + a.eps));
          epi_sync();
        }
      } else if (op.kind == OP_APPEND) {
        // this forward's K (RoPE'd) and V rows into the cache, items (kv head, token)
        if (warp == 2) wait_op(a, p - 1, 60);
        epi_sync();
        if (tid == 0) tr(a, p, 2);
        constexpr int HALF = HD / 2;
        const size_t row_len = size_t(a.H + 2 * a.KVH) * HD;
        for (int w = blockIdx.x; w < a.KVH * a.M; w += P) {
          const int kvh = w % a.KVH, m = w / a.KVH;
          const int slot = a.P->slot[m], pos = a.P->pos[m];
          const float* cs = a.rope_cos + size_t(pos) * HALF;
          const float* sn = a.rope_sin + size_t(pos) * HALF;
          const float* xk = op.qkv + size_t(m) * row_len + size_t(a.H + kvh) * HD;
          const float* xv = op.qkv + size_t(m) * row_len + size_t(a.H + a.KVH + kvh) * HD;
          for (int d2 = tid; d2 < HD; d2 += 128) {
            op.kc[(size_t(kvh) * a.S + slot) * HD + d2] = __float2bfloat16_rn(rope_at(xk, d2, HALF, cs, sn));
            op.vc[(size_t(kvh) * a.S + slot) * HD + d2] = __float2bfloat16_rn(__ldcg(xv + d2));
          }
        }
      } else if (op.kind == OP_SWIGLU) {
        if (warp == 2) wait_op(a, p - 1, 40);
        epi_sync();
        if (tid == 0) tr(a, p, 2);
        // this CTA's slice of the M x ffn activations, 4 per thread-step
        const int per_row = op.ffn / 4, total = a.M * per_row;
        const int lo = int((long long)blockIdx.x * total / P), hi = int((long long)(blockIdx.x + 1) * total / P);
        for (int i = lo + tid; i < hi; i += 128) {
          const int m = i / per_row, j4 = (i % per_row) * 4;
          const float4* gs = reinterpret_cast<const float4*>(op.gu + size_t(m) * 2 * op.ffn + 2 * j4);
          const float4 v0 = __ldcg(gs), v1 = __ldcg(gs + 1);
          const float f0 = v0.x / (1.0f + expf(-v0.x)) * v0.y, f1 = v0.z / (1.0f + expf(-v0.z)) * v0.w;
          const float f2 = v1.x / (1.0f + expf(-v1.x)) * v1.y, f3 = v1.z / (1.0f + expf(-v1.z)) * v1.w;
          __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(op.act + size_t(m) * op.ffn + j4);
          o2[0] = __floats2bfloat162_rn(f0, f1);
          o2[1] = __floats2bfloat162_rn(f2, f3);
        }
      } else if (op.kind == OP_ATTN) {
        if (warp == 2) wait_op(a, p - 1, 20);
        epi_sync();
        if (tid == 0) tr(a, p, 2);
        // chunks that hold main keys of some query (every CTA derives the same count)
        int main_max = 1;
        for (int mm = 0; mm < a.M; ++mm) main_max = max(main_max, a.P->main_len[mm]);
        // at most kMaxChunks chunks: widen the chunk for long contexts
        const int need = (((main_max + kMaxChunks - 1) / kMaxChunks) + kKeysPass - 1) / kKeysPass * kKeysPass;
        const int chunk_eff = max(a.chunk, need);
        const int nch_eff = (main_max + chunk_eff - 1) / chunk_eff;
        constexpr int QB = kRows / G;
        const int nqb = (a.M + QB - 1) / QB;
        const int items = a.KVH * nqb * nch_eff;
        for (int w = blockIdx.x; w < items; w += P) {
          const int c = w % nch_eff, kvh = (w / nch_eff) % a.KVH, qb = w / (nch_eff * a.KVH);
          attn_item<HD, G>(a, op, kvh, c, qb, nch_eff, chunk_eff, sm, tid);
          epi_sync();
        }
      } else {
        // GEMM epilogue: accumulate this CTA's segments into op.out
        const int U = op_tiles(op) * op.KU;
        const int u0 = ub(blockIdx.x, U, P), u1 = ub(blockIdx.x + 1, U, P);
        int u = u0;
        while (u < u1) {
          const int t = u / op.KU;
          const int seg_end = min(u1, (t + 1) * op.KU);
          ++seg;
          const int b = seg & 1;
          mwait(&tfull[b], (seg >> 1) & 1, 5);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t taddr = tmem + (uint32_t(q * 32) << 16) + uint32_t(b * C::kAccCols);
          const int r = t * kBM + rl;
#pragma unroll 1
          for (int c = 0; c < NP; c += 8) {
            uint32_t v[8];
            tc::tmem_ld8(taddr + c, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (c + 8 >= NP) {
              asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
              __syncwarp();
              if (lane == 0) tc::mbar_arrive(&tempty[b]);
            }
            float* out = op.out ? op.out : a.logits;
            const int ld = op.out ? op.ld_out : op.N;
            if (r < op.N)
#pragma unroll
              for (int j = 0; j < 8; ++j)
                if (c + j < a.M) red_add_f32(out + size_t(c + j) * ld + r, __uint_as_float(v[j]));
          }
          u = seg_end;
        }
      }
      // release this CTA's part of op p (its accumulations / writes / zero-fills)
      epi_sync();
      if (tid == 0) {
        tr(a, p, 5);
        red_release_add(a.done + (size_t(p) * kStripes + (blockIdx.x & (kStripes - 1))) * kLine, 1);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::kTmemCols));
  // the last CTA out resets the completion counters for the next launch (a
  // CTA must not count itself out before the previous launch completed: PDL
  // may start this grid early)
  if (threadIdx.x == 0) {
    tc::pdl_wait();
    int* exitc = a.done + size_t(a.n_ops) * kStripes * kLine;
    int old;
    asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(exitc) : "memory");
    if (old == P - 1) {
      for (int i = 0; i < a.n_ops * kStripes; ++i) a.done[size_t(i) * kLine] = 0;
      *exitc = 0;
    }
    if (a.trace) a.trace[size_t(blockIdx.x) * kTrSlots + 1] = gtimer();
  }
}

}  // namespace pk
}  // namespace ssd
