// Decode attention with the chunk merge done in a thread-block cluster
// (DSMEM) instead of through global memory, and the chunk's K/V rows pulled
// into shared memory by one bulk copy BEFORE the PDL wait, so the KV-cache
// read overlaps the tail of the QKV GEMM that precedes it.
//
// Same contract as attention_kernel (kernels.cuh): CTA = (key chunk, kv
// head, query token), RoPE + KV append of this forward's tokens fused, the
// tree/branch mask generated from FwdParams; the G query heads of a KV group
// share every K/V row. The nch <= 8 chunks of one (kv head, token) form one
// cluster; after each CTA has its chunk's (max, sum, unnormalised P.V) in
// shared memory, rank 0 merges them in chunk order over DSMEM (deterministic)
// and writes the head outputs. No global partials, fences or atomics.
#pragma once

#include <cooperative_groups.h>

#include "gemm_tc.cuh"

namespace ssd {

constexpr int kAttnClMaxChunks = 8;  // portable cluster size

__host__ __device__ constexpr size_t attn_cl_smem(int G, int hd) {
  return size_t(2) * kAttnChunk * hd * 2                    // K, V rows (bf16)
         + size_t(G) * hd * 4 + size_t(G) * kAttnChunk * 4  // q, scores
         + size_t(kAttnThreads / (hd / 8)) * G * hd * 4     // P.V key-group partials
         + size_t(G) * (hd + 2) * 4                         // chunk result
         + 64;                                              // mbarrier
}

template <int G>
__global__ void __launch_bounds__(kAttnThreads) attention_cl_kernel(
    const float* __restrict__ qkv, const FwdParams* __restrict__ P, int M, const float* __restrict__ cos_t,
    const float* __restrict__ sin_t, bf16* __restrict__ kc, bf16* __restrict__ vc, int S, int H, int KVH, int hd,
    float scale, bf16* __restrict__ out, int ctx_bound, Prefetch pf) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(128) uint8_t smem[];
  bf16* Ks = reinterpret_cast<bf16*>(smem);
  bf16* Vs = Ks + size_t(kAttnChunk) * hd;
  float* qs = reinterpret_cast<float*>(Vs + size_t(kAttnChunk) * hd);
  float* sc = qs + G * hd;
  float* pv_red = sc + G * kAttnChunk;
  const int ngrp = kAttnThreads / (hd >> 3);
  float* res = pv_red + ngrp * G * hd;  // [G][hd + 2]: unnormalised o, max, sum
  uint64_t* bar = reinterpret_cast<uint64_t*>(res + G * (hd + 2) + 2);
  bar = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(bar) + 15) & ~uintptr_t(15));

  KTL_ENTER(3);
  const int chunk = blockIdx.x, kvh = blockIdx.y, m = blockIdx.z, tid = threadIdx.x;
  const int nch = gridDim.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int half = hd >> 1;
  const int j0 = chunk * kAttnChunk;
  const bf16* kbase = kc + size_t(kvh) * S * hd;
  const bf16* vbase = vc + size_t(kvh) * S * hd;
  // 0) main-cache rows [j0, j0 + npre) of this head: written by earlier
  //    forwards (or patched below), so they are fetched before the PDL wait.
  //    (P was written before this forward's first kernel started.)
  const int mb = P->mbase[m];
  const int npre = max(0, min(min(kAttnChunk, ctx_bound - j0), S - mb - j0));
  if (tid == 0) {
    tc::mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    prefetch_window(pf, kPfUnitBytes);
    const uint32_t bytes = uint32_t(npre) * hd * 2;
    tc::mbar_expect_tx(bar, 2 * bytes);
    if (bytes) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      tc::bulk_load(Ks, kbase + size_t(mb + j0) * hd, bytes, bar, pol);
      tc::bulk_load(Vs, vbase + size_t(mb + j0) * hd, bytes, bar, pol);
    }
  }
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  KTL_READY();
  KTL_SUB(0);

  const size_t row_len = size_t(H + 2 * KVH) * hd;
  const int main_len = P->main_len[m], bbase = P->bbase[m], blen = P->blen[m];
  const int nk = main_len + blen;
  const int j1 = min(nk, j0 + kAttnChunk);
  tc::mbar_wait(bar, 0);
  KTL_SUB(1);
  if (j0 < j1) {
    // 1) branch-local keys of this chunk (j >= main_len) from their slots
    for (int e = tid; e < (j1 - max(j0, main_len)) * (hd >> 3); e += kAttnThreads) {
      const int jj = max(j0, main_len) + e / (hd >> 3), q8 = e % (hd >> 3);
      const int slot = bbase + (jj - main_len);
      reinterpret_cast<uint4*>(Ks + size_t(jj - j0) * hd)[q8] = reinterpret_cast<const uint4*>(kbase + size_t(slot) * hd)[q8];
      reinterpret_cast<uint4*>(Vs + size_t(jj - j0) * hd)[q8] = reinterpret_cast<const uint4*>(vbase + size_t(slot) * hd)[q8];
    }
    __syncthreads();
    // 2) append (RoPE'd) K and V of this forward's tokens whose key falls in
    //    this chunk: to the cache and to the staged rows
    for (int e = tid; e < M * half; e += kAttnThreads) {
      const int t = e / half, i = e % half;
      const int slot = P->slot[t];
      const int j = visible_key(slot, mb, main_len, bbase, blen);
      if (j < j0 || j >= j1) continue;
      const int pos = P->pos[t];
      const float c = cos_t[size_t(pos) * half + i], sn = sin_t[size_t(pos) * half + i];
      const float* ks = qkv + size_t(t) * row_len + size_t(H + kvh) * hd;
      const float* vs = qkv + size_t(t) * row_len + size_t(H + KVH + kvh) * hd;
      const float a = __ldcg(ks + i), b = __ldcg(ks + i + half);
      const bf16 k0 = __float2bfloat16_rn(a * c - b * sn), k1 = __float2bfloat16_rn(b * c + a * sn);
      const bf16 v0 = __float2bfloat16_rn(__ldcg(vs + i)), v1 = __float2bfloat16_rn(__ldcg(vs + i + half));
      bf16* kd = kc + (size_t(kvh) * S + slot) * hd;
      bf16* vd = vc + (size_t(kvh) * S + slot) * hd;
      kd[i] = k0; kd[i + half] = k1; vd[i] = v0; vd[i + half] = v1;
      bf16* kr = Ks + size_t(j - j0) * hd;
      bf16* vr = Vs + size_t(j - j0) * hd;
      kr[i] = k0; kr[i + half] = k1; vr[i] = v0; vr[i + half] = v1;
    }
    // 3) rotated queries of the group
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
    __syncthreads();
    KTL_SUB(2);
    // 4) scores from the staged K rows (lane-cooperative, conflict-free)
    const int n = j1 - j0;
    attn_scores<G>(qs, sc, n, hd, scale, warp, lane,
                   [&](int jj) { return reinterpret_cast<const uint4*>(Ks + size_t(jj) * hd); });
    __syncthreads();
    KTL_SUB(3);
    // 5) chunk softmax statistics (warp gg -> head gg)
    for (int gg = warp; gg < G; gg += kAttnThreads / 32) {
      float mx = -INFINITY;
      for (int j = lane; j < n; j += 32) mx = fmaxf(mx, sc[gg * kAttnChunk + j]);
      mx = warp_max(mx);
      float den = 0.f;
      for (int j = lane; j < n; j += 32) {
        const float e2 = expf(sc[gg * kAttnChunk + j] - mx);
        sc[gg * kAttnChunk + j] = e2;
        den += e2;
      }
      den = warp_sum(den);
      if (lane == 0) { res[gg * (hd + 2) + hd] = mx; res[gg * (hd + 2) + hd + 1] = den; }
    }
    __syncthreads();
    // 6) unnormalised P.V: thread = (key group, 8 dims), V rows from shared memory
    {
      const int nd = hd >> 3, dc = tid % nd, kg = tid / nd;
      float acc[G][8];
#pragma unroll
      for (int gg = 0; gg < G; ++gg)
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[gg][i] = 0.f;
      for (int jj = kg; jj < n; jj += ngrp) {
        float f[8];
        bf16x8_to_f32(reinterpret_cast<const uint4*>(Vs + size_t(jj) * hd)[dc], f);
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
          const float p = sc[gg * kAttnChunk + jj];
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[gg][i] += p * f[i];
        }
      }
#pragma unroll
      for (int gg = 0; gg < G; ++gg)
#pragma unroll
        for (int i = 0; i < 8; ++i) pv_red[(kg * G + gg) * hd + dc * 8 + i] = acc[gg][i];
      __syncthreads();
      for (int e = tid; e < G * hd; e += kAttnThreads) {
        const int gg = e / hd, dd = e % hd;
        float o = 0.f;
        for (int k2 = 0; k2 < ngrp; ++k2) o += pv_red[(k2 * G + gg) * hd + dd];
        res[gg * (hd + 2) + dd] = o;
      }
    }
  } else if (tid < G) {  // chunk beyond this query's keys: empty partial
    res[tid * (hd + 2) + hd] = -INFINITY;
    res[tid * (hd + 2) + hd + 1] = 0.f;
  }
  KTL_SUB(4);
  // 7) merge the cluster's chunks in chunk order (rank 0, over DSMEM)
  cluster.sync();
  KTL_SUB(5);
  if (chunk == 0) {
    for (int e = tid; e < G * hd; e += kAttnThreads) {
      const int gg = e / hd, dd = e % hd;
      float mx = -INFINITY;
      for (int c = 0; c < nch; ++c) {
        const float* r = cluster.map_shared_rank(res, c);
        mx = fmaxf(mx, r[gg * (hd + 2) + hd]);
      }
      float den = 0.f, o = 0.f;
      for (int c = 0; c < nch; ++c) {
        const float* r = cluster.map_shared_rank(res, c);
        const float mc = r[gg * (hd + 2) + hd];
        if (mc == -INFINITY) continue;
        const float w = expf(mc - mx);
        den += w * r[gg * (hd + 2) + hd + 1];
        o += w * r[gg * (hd + 2) + dd];
      }
      out[size_t(m) * H * hd + size_t(kvh * G + gg) * hd + dd] = __float2bfloat16_rn(o / den);
    }
  }
  KTL_SUB(6);
  cluster.sync();  // keep every rank's shared memory alive until rank 0 has read it
  KTL_SUB(7);
  KTL_EXIT();
}

}  // namespace ssd
