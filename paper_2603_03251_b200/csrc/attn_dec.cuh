// Decode / verify / branch-step attention: ONE CTA of 256 threads per
// (kv head, query token) over all of the query's keys.
//
// Why: the chunked kernels (attention_kernel, attention_cl_kernel) put 128
// keys on a 128-thread CTA and run 6-7 dependent phases with warp-shuffle
// reductions per key; at 4 warps per SM every instruction waits on its
// predecessor (ncu: ~10 cycles per issued instruction), so a 1 MB KV read
// took ~15 us per layer. Here 8 warps share the work, each lane group of
// HD/16 lanes owns one key per pass (16 dims per lane, two 16-byte loads),
// and the query's KV rows are read BEFORE the PDL wait (they were written by
// earlier forwards), overlapping the tail of the QKV GEMM: with few CTAs
// (decode / verify, MINB = 1) the first `nst` main rows are bulk-copied into
// shared memory, so scores and P.V run from SMEM; with many CTAs (branch
// steps, MINB = 2 for two CTAs per SM) they are bulk-prefetched into L2 and
// read in batches of 4 passes (every load of a batch issued before use).
//
// Same contract as attention_kernel: RoPE + KV append of this forward's
// tokens fused, the tree/branch mask generated from FwdParams (main keys
// [0, main_len) in slots mbase + j, branch keys in [bbase, bbase + blen)),
// the G query heads of a KV group share every K/V load. Keys produced by
// THIS forward (another CTA appends them to the cache concurrently) are
// recomputed from the QKV row with the same rounding as the writer, so the
// kernel never reads a cache row written in the same launch.
#pragma once

#include "kernels.cuh"

namespace ssd {

constexpr int kDecThreads = 256;
constexpr int kDecBatch = 4;  // K-row passes whose loads are in flight together
#ifndef SSD_DEC_BATCH_MINB2
#define SSD_DEC_BATCH_MINB2 2  // two CTAs per SM (128 registers): 4 spilled (d20 1.27 -> 1.23 ms)
#endif
constexpr size_t kDecStaticSmem = 2 * kMaxM * sizeof(int);  // s_tj + s_tp

// RoPE'd key element d of a K row x (fp32, head_dim hd) at cos / sin row
// (c, s): the writer and the in-kernel recomputation use this one function
// (explicit _rn intrinsics: no contraction differences).
__device__ __forceinline__ float rope_elem(const float* x, int d, int half, const float* c, const float* s) {
  if (d < half) return __fsub_rn(__fmul_rn(x[d], c[d]), __fmul_rn(x[d + half], s[d]));
  const int i = d - half;
  return __fadd_rn(__fmul_rn(x[d], c[i]), __fmul_rn(x[i], s[i]));
}

__host__ __device__ constexpr int dec_nkg(int HD) { return kDecThreads / (HD / 8); }

// RoPE + KV append of every token of a wide forward (prefill chunks), one
// CTA per (token, kv head), with the writer rounding of attention_dec; the
// attention that follows (appended = 1) then reads every key from the cache
// instead of recomputing this forward's keys per query (quadratic in M).
__global__ void __launch_bounds__(128) rope_append_kernel(const float* __restrict__ qkv,
                                                          const FwdParams* __restrict__ P, const float* __restrict__ cos_t,
                                                          const float* __restrict__ sin_t, bf16* __restrict__ kc,
                                                          bf16* __restrict__ vc, int S, int H, int KVH, int HD) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int m = blockIdx.x, kvh = blockIdx.y, half = HD >> 1;
  const size_t row_len = size_t(H + 2 * KVH) * HD;
  const int pos = P->pos[m], slot = P->slot[m];
  const float* c = cos_t + size_t(pos) * half;
  const float* s = sin_t + size_t(pos) * half;
  const float* xk = qkv + size_t(m) * row_len + size_t(H + kvh) * HD;
  const float* xv = qkv + size_t(m) * row_len + size_t(H + KVH + kvh) * HD;
  for (int d = threadIdx.x; d < HD; d += blockDim.x) {
    kc[(size_t(kvh) * S + slot) * HD + d] = __float2bfloat16_rn(rope_elem(xk, d, half, c, s));
    vc[(size_t(kvh) * S + slot) * HD + d] = __float2bfloat16_rn(__ldcg(xv + d));
  }
}

// Shared memory: [qs][sc][red][stat][ovr] then (16-byte aligned) the staged
// K and V rows ([nst][HD] bf16 each) and one mbarrier.
__host__ __device__ constexpr size_t attn_dec_base(int G, int HD, int kcap) {
  return ((size_t(G) * HD + size_t(G) * kcap + size_t(dec_nkg(HD)) * G * HD + 2 * G) * 4 + size_t(kcap) * 4 + 15) &
         ~size_t(15);
}
__host__ __device__ constexpr size_t attn_dec_smem(int G, int HD, int kcap, int nst) {
  return attn_dec_base(G, HD, kcap) + size_t(2) * nst * HD * 2 + 16;
}

template <int G, int HD, int MINB>
__global__ void __launch_bounds__(kDecThreads, MINB) attention_dec_kernel(
    const float* __restrict__ qkv, const FwdParams* __restrict__ P, int M, const float* __restrict__ cos_t,
    const float* __restrict__ sin_t, bf16* __restrict__ kc, bf16* __restrict__ vc, int S, int H, int KVH, float scale,
    bf16* __restrict__ out, int kcap, int nst, int appended, Prefetch pf, KvMap km) {
  constexpr int NW = kDecThreads / 32;
  constexpr int LPK = HD / 16;   // lanes per key
  constexpr int KPW = 32 / LPK;  // keys per warp pass
  constexpr int HALF = HD / 2;
  constexpr int NDC = HD / 8;    // 8-dim chunks of a row
  constexpr int NBT = MINB == 2 ? SSD_DEC_BATCH_MINB2 : kDecBatch;
  constexpr int NKG = dec_nkg(HD);
  extern __shared__ __align__(16) float dsm[];
  float* qs = dsm;                       // [G][HD] rotated, scaled queries
  float* sc = qs + G * HD;               // [G][kcap] scores -> probabilities
  float* red = sc + size_t(G) * kcap;    // [NKG][G][HD] P.V partials
  float* stat = red + NKG * G * HD;      // [G][2] max, sum
  int* ovr = reinterpret_cast<int*>(stat + 2 * G);  // [kcap] key -> token of this forward (or -1)
  bf16* Ks = reinterpret_cast<bf16*>(reinterpret_cast<char*>(dsm) + attn_dec_base(G, HD, kcap));  // [nst][HD]
  bf16* Vs = Ks + size_t(nst) * HD;
  uint64_t* bar = reinterpret_cast<uint64_t*>(Vs + size_t(nst) * HD);

  KTL_ENTER(4);
  const int kvh = blockIdx.x, m = blockIdx.y, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // P was written before this forward's first kernel started: readable
  // before the PDL wait, like the KV rows of earlier forwards.
  const int main_len = P->main_len[m], bbase = P->bbase[m], blen = P->blen[m], mb = P->mbase[m];
  const int nk = main_len + blen;
  const bf16* kb = kc + size_t(kvh) * S * HD;
  const bf16* vb = vc + size_t(kvh) * S * HD;
  const int ns = min(nst, main_len);  // main keys [0, ns) served from shared memory
  // Stage main rows [0, ns) into shared memory with two bulk copies (rows of
  // THIS forward's tokens among them are stale and patched after the wait).
  // The mbarrier is initialised, and the initialisation made visible to every
  // thread by the CTA barrier, before anyone can wait on it (a wait issued
  // before that barrier faulted: scripts/ssd_stress.py, compute-sanitizer).
  if (tid == 0 && nst > 0) {
    tc::mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    // main rows are contiguous within a page (one run when unpaged)
    const int run = km.tab ? (1 << km.shift) : (1 << 30);
    if (nst > 0) {
      const uint32_t sbytes = uint32_t(ns) * HD * 2;
      tc::mbar_expect_tx(bar, 2 * sbytes);
      if (sbytes) {
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        for (int j0 = 0; j0 < ns; j0 += run) {
          const uint32_t rb = uint32_t(min(run, ns - j0)) * HD * 2;
          const int sl = main_slot(km, mb, j0);
          tc::bulk_load(Ks + size_t(j0) * HD, kb + size_t(sl) * HD, rb, bar, pol);
          tc::bulk_load(Vs + size_t(j0) * HD, vb + size_t(sl) * HD, rb, bar, pol);
        }
      }
    }
    prefetch_window(pf, kPfUnitBytes);
    for (int j0 = ns; j0 < main_len; j0 += run) {
      const int rows = km.tab ? min(run - (j0 & (run - 1)), main_len - j0) : main_len - j0;
      const uint32_t mbytes = uint32_t(rows) * HD * 2;
      const int sl = main_slot(km, mb, j0);
      if (mbytes >= 16) {
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(kb + size_t(sl) * HD), "r"(mbytes & ~15u)
                     : "memory");
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(vb + size_t(sl) * HD), "r"(mbytes & ~15u)
                     : "memory");
      }
      if (km.tab) j0 -= j0 & (run - 1);  // continue at the next page boundary
    }
    const uint32_t bbytes = uint32_t(blen) * HD * 2;
    if (bbytes >= 16) {
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(kb + size_t(bbase) * HD), "r"(bbytes & ~15u) : "memory");
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(vb + size_t(bbase) * HD), "r"(bbytes & ~15u) : "memory");
    }
  }
  // Everything that depends only on P and the RoPE tables happens before the
  // PDL wait (P and the tables predate this forward): the key -> token map of
  // this forward's tokens, the staged-key patch list, the query's and the
  // appended key's cos / sin. After the wait only the QKV row is read.
  __shared__ int s_tj[kMaxM], s_tp[kMaxM];  // token t -> visible key j (or -1), RoPE position (kDecStaticSmem)
  for (int j = tid; j < nk; j += kDecThreads) ovr[j] = -1;
  const int pos_m = P->pos[m];
  constexpr int NQE = (G * HD + kDecThreads - 1) / kDecThreads;
  float qcv[NQE], qsv[NQE];
#pragma unroll
  for (int r = 0; r < NQE; ++r) {
    const int e = tid + r * kDecThreads, dd = (e % HD) % HALF;
    qcv[r] = e < G * HD ? cos_t[size_t(pos_m) * HALF + dd] : 0.f;
    qsv[r] = e < G * HD ? sin_t[size_t(pos_m) * HALF + dd] : 0.f;
  }
  __syncthreads();  // ovr initialised before the sets below
  for (int t = tid; t < M; t += kDecThreads) {
    const int j = visible_token_key(P, t, mb, main_len, bbase, blen);
    s_tj[t] = j;
    s_tp[t] = P->pos[t];
    // appended: rope_append_kernel wrote this forward's rows before this
    // launch (wide forwards), so every key is read from the cache
    if (j >= 0 && !appended) ovr[j] = t;
  }
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  KTL_READY();

  const size_t row_len = size_t(H + 2 * KVH) * HD;
  // 1) rotated queries; append of token m's K / V (this kv head) to the cache;
  //    keys of this forward in the staged range patched
  if (nst > 0) tc::mbar_wait(bar, 0);  // staged rows landed before they are patched below
  __syncthreads();
  // keys of this forward that fall in the staged range: patch the stale
  // staged rows with the recomputed ones (the writer's rounding), so scores
  // and P.V read every staged key from shared memory
  for (int e = tid; e < M * HD && ns > 0; e += kDecThreads) {
    const int t = e / HD, d = e % HD;
    const int j = s_tj[t];
    if (j < 0 || j >= ns) continue;
    const int pos = s_tp[t];
    const float* x = qkv + size_t(t) * row_len + size_t(H + kvh) * HD;
    Ks[size_t(j) * HD + d] =
        __float2bfloat16_rn(rope_elem(x, d, HALF, cos_t + size_t(pos) * HALF, sin_t + size_t(pos) * HALF));
    Vs[size_t(j) * HD + d] = __float2bfloat16_rn(__ldcg(x + KVH * HD + d));
  }
  {
#pragma unroll
    for (int r = 0; r < NQE; ++r) {
      const int e = tid + r * kDecThreads;
      if (e >= G * HD) break;
      const int gg = e / HD, d = e % HD;
      const float* x = qkv + size_t(m) * row_len + size_t(kvh * G + gg) * HD;
      const float a = __ldcg(x + d), b = __ldcg(x + (d < HALF ? d + HALF : d - HALF));
      const float rr = d < HALF ? __fsub_rn(__fmul_rn(a, qcv[r]), __fmul_rn(b, qsv[r]))
                                : __fadd_rn(__fmul_rn(a, qcv[r]), __fmul_rn(b, qsv[r]));
      qs[e] = rr * scale;
    }
    const float* c = cos_t + size_t(pos_m) * HALF;
    const float* sn = sin_t + size_t(pos_m) * HALF;
    const float* xk = qkv + size_t(m) * row_len + size_t(H + kvh) * HD;
    const float* xv = qkv + size_t(m) * row_len + size_t(H + KVH + kvh) * HD;
    const int slot = P->slot[m];
    for (int d = tid; d < HD && !appended; d += kDecThreads) {
      kc[(size_t(kvh) * S + slot) * HD + d] = __float2bfloat16_rn(rope_elem(xk, d, HALF, c, sn));
      vc[(size_t(kvh) * S + slot) * HD + d] = __float2bfloat16_rn(__ldcg(xv + d));
    }
  }
  __syncthreads();
  KTL_SUB(0);

  // 2) scores: lane group (lane / LPK) takes one key per pass, lane sub
  //    (lane % LPK) its dims [16 sub, 16 sub + 16)
  {
    const int sub = lane % LPK, grp = lane / LPK;
    float qr[G][16];
#pragma unroll
    for (int gg = 0; gg < G; ++gg)
#pragma unroll
      for (int i = 0; i < 16; ++i) qr[gg][i] = qs[gg * HD + sub * 16 + i];
    for (int jb = warp * KPW; jb < nk; jb += NW * KPW * NBT) {
      uint4 kr[NBT][2];
      int tk[NBT];
#pragma unroll
      for (int u = 0; u < NBT; ++u) {  // issue every load of the batch first
        const int j = jb + u * NW * KPW + grp;
        tk[u] = j < nk ? (j < ns ? -1 : ovr[j]) : -2;
        if (tk[u] == -1) {
          const int slot = j < main_len ? main_slot(km, mb, j) : bbase + (j - main_len);
          const uint4* src = j < ns ? reinterpret_cast<const uint4*>(Ks + size_t(j) * HD + sub * 16)
                                    : reinterpret_cast<const uint4*>(kb + size_t(slot) * HD + sub * 16);
          kr[u][0] = j < ns ? src[0] : __ldcg(src);
          kr[u][1] = j < ns ? src[1] : __ldcg(src + 1);
        }
      }
#pragma unroll
      for (int u = 0; u < NBT; ++u) {
        const int j = jb + u * NW * KPW + grp;
        float kf[16];
        if (tk[u] == -1) {
          bf16x8_to_f32(kr[u][0], kf);
          bf16x8_to_f32(kr[u][1], kf + 8);
        } else if (tk[u] >= 0) {  // a key of this forward: recompute the written row
          const int t = tk[u];
          const int pos = P->pos[t];
          const float* x = qkv + size_t(t) * row_len + size_t(H + kvh) * HD;
          const float* c = cos_t + size_t(pos) * HALF;
          const float* s = sin_t + size_t(pos) * HALF;
#pragma unroll
          for (int i = 0; i < 16; ++i)
            kf[i] = __bfloat162float(__float2bfloat16_rn(rope_elem(x, sub * 16 + i, HALF, c, s)));
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) kf[i] = 0.f;
        }
        float part[G];
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
          float a0 = 0.f, a1 = 0.f;
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            a0 = fmaf(qr[gg][i], kf[i], a0);
            a1 = fmaf(qr[gg][i + 1], kf[i + 1], a1);
          }
          part[gg] = a0 + a1;
        }
#pragma unroll
        for (int o = LPK >> 1; o > 0; o >>= 1)
#pragma unroll
          for (int gg = 0; gg < G; ++gg) part[gg] += __shfl_xor_sync(0xffffffffu, part[gg], o);
        if (sub == 0 && j < nk)
#pragma unroll
          for (int gg = 0; gg < G; ++gg) sc[gg * kcap + j] = part[gg];
      }
    }
  }
  __syncthreads();
  KTL_SUB(1);
  // 3) softmax statistics (warp gg -> head gg), probabilities in place
  for (int gg = warp; gg < G; gg += NW) {
    float mx = -INFINITY;
    for (int j = lane; j < nk; j += 32) mx = fmaxf(mx, sc[gg * kcap + j]);
    mx = warp_max(mx);
    float den = 0.f;
    for (int j = lane; j < nk; j += 32) {
      const float e = expf(sc[gg * kcap + j] - mx);
      sc[gg * kcap + j] = e;
      den += e;
    }
    den = warp_sum(den);
    if (lane == 0) { stat[2 * gg] = mx; stat[2 * gg + 1] = den; }
  }
  __syncthreads();
  KTL_SUB(2);
  // 4) P.V: thread = (8-dim chunk dc, key group kg), V rows in batches
  {
    const int dc = tid % NDC, kg = tid / NDC;
    float acc[G][8];
#pragma unroll
    for (int gg = 0; gg < G; ++gg)
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[gg][i] = 0.f;
    for (int jb = kg; jb < nk; jb += NKG * NBT) {
      uint4 vr[NBT];
      int tv[NBT];
#pragma unroll
      for (int u = 0; u < NBT; ++u) {
        const int j = jb + u * NKG;
        tv[u] = j < nk ? (j < ns ? -1 : ovr[j]) : -2;
        if (tv[u] == -1) {
          const int slot = j < main_len ? main_slot(km, mb, j) : bbase + (j - main_len);
          vr[u] = j < ns ? reinterpret_cast<const uint4*>(Vs + size_t(j) * HD)[dc]
                         : __ldcg(reinterpret_cast<const uint4*>(vb + size_t(slot) * HD) + dc);
        }
      }
#pragma unroll
      for (int u = 0; u < NBT; ++u) {
        const int j = jb + u * NKG;
        if (tv[u] == -2) continue;
        float f[8];
        if (tv[u] == -1) {
          bf16x8_to_f32(vr[u], f);
        } else {
          const float* x = qkv + size_t(tv[u]) * row_len + size_t(H + KVH + kvh) * HD + dc * 8;
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = __bfloat162float(__float2bfloat16_rn(__ldcg(x + i)));
        }
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
          const float p = sc[gg * kcap + j];
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[gg][i] = fmaf(p, f[i], acc[gg][i]);
        }
      }
    }
#pragma unroll
    for (int gg = 0; gg < G; ++gg)
#pragma unroll
      for (int i = 0; i < 8; ++i) red[(kg * G + gg) * HD + dc * 8 + i] = acc[gg][i];
  }
  __syncthreads();
  KTL_SUB(3);
  for (int e = tid; e < G * HD; e += kDecThreads) {
    const int gg = e / HD, dd = e % HD;
    float o = 0.f;
#pragma unroll 4
    for (int k2 = 0; k2 < NKG; ++k2) o += red[(k2 * G + gg) * HD + dd];
    out[size_t(m) * H * HD + size_t(kvh * G + gg) * HD + dd] = __float2bfloat16_rn(o / stat[2 * gg + 1]);
  }
  KTL_SUB(4);
  KTL_EXIT();
}

}  // namespace ssd
