// Weight-streaming GEMV for decode steps with M <= 4 tokens (the north star's
// "HBM-bound weight streaming through 16-byte-vectorised loads").
//
// Why not tcgen05 at M = 1: the tensor-core kernel pads the tokens to a
// 16-wide N operand and, to keep every SM streaming, splits each 128-row tile
// over several CTAs along K; the partial sums then cost an L2 round trip,
// an atomic ticket and a last-arriver reduction at the end of every GEMM
// (~6 us, scripts/ktl.py) — a fixed cost paid 129 times per 8B step. Here a
// CTA owns 16 whole rows (one 2 KB run of every 16 KB k-block of the
// pre-tiled layout), so no partial ever leaves the CTA; the grid is
// N / 16 CTAs of 256 threads, several resident per SM.
//
// Layout: the pre-tiled SWIZZLE_128B blocks of gemm_tc.cuh; row r of a tile
// holds logical 16-byte chunk c at physical chunk c ^ (r & 7). Warp w takes
// k-blocks kb = w, w + 8, ...; lane l reads physical chunks l, l+32, l+64,
// l+96 of the 2 KB run (rows l/8 + {0,4,8,12}, chunk l%8): every warp load
// is 512 contiguous bytes. The weights of the first k-blocks are loaded
// BEFORE the PDL wait (they do not depend on the previous kernel); the
// activations are staged in shared memory after it. Fixed-order reductions
// (lane shuffles, then warps through shared memory): deterministic.
#pragma once

#include "kernels.cuh"

namespace ssd {

constexpr int kGemvThreads = 256;
constexpr int kGemvRows = 16;   // rows per CTA
constexpr int kGemvPre = 2;     // k-blocks per warp loaded before the PDL wait
constexpr size_t kGemvSmemMax = 160 * 1024;

template <int EPI, int MT>
__global__ void __launch_bounds__(kGemvThreads) gemv_kernel(const bf16* __restrict__ W, int N, int K,
                                                            const bf16* __restrict__ X, int M, float* __restrict__ Y,
                                                            int ldy, bf16* __restrict__ Yb, int ldyb, Prefetch pf) {
  extern __shared__ __align__(16) float gsm[];
  float* xs = gsm;                          // [MT][K] activations (fp32)
  float* red = xs + size_t(MT) * K;         // [8 warps][MT][16 rows]
  KTL_ENTER(30 + EPI);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KB = K >> 6;
  const int groups = ((N + 127) >> 7) * 8;  // 16-row groups (rows padded to whole tiles)
  int g = blockIdx.x;                       // row group: tile g / 8, rows (g % 8) * 16 .. (persistent loop)
  const uint4* base0 = reinterpret_cast<const uint4*>(W) + (size_t(g >> 3) * KB * 1024 + size_t(g & 7) * 128);
  const int rl = lane >> 3, p = lane & 7;   // rows rl + {0,4,8,12}; physical chunk p
  // 1) first k-blocks of this warp's slice: independent of the previous kernel
  uint4 wpre[kGemvPre][4];
#pragma unroll
  for (int u = 0; u < kGemvPre; ++u) {
    const int kb = warp + 8 * u;
    if (kb < KB) {
      const uint4* blk = base0 + size_t(kb) * 1024;
#pragma unroll
      for (int q = 0; q < 4; ++q) wpre[u][q] = __ldcs(blk + lane + 32 * q);
    }
  }
  if (threadIdx.x == 0) prefetch_window(pf, kPfUnitBytes);
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  KTL_READY();
  // 2) activations -> shared memory (fp32)
  for (int e = threadIdx.x; e < M * (K >> 3); e += kGemvThreads) {
    const int t = e / (K >> 3), c8 = e % (K >> 3);
    float f[8];
    bf16x8_to_f32(reinterpret_cast<const uint4*>(X + size_t(t) * K)[c8], f);
#pragma unroll
    for (int i = 0; i < 8; ++i) xs[size_t(t) * K + c8 * 8 + i] = f[i];
  }
  for (int e = M * K + threadIdx.x; e < MT * K; e += kGemvThreads) xs[e] = 0.f;
  __syncthreads();
  for (bool first = true; g < groups; g += gridDim.x, first = false) {
  const uint4* base = reinterpret_cast<const uint4*>(W) + (size_t(g >> 3) * KB * 1024 + size_t(g & 7) * 128);
  if (!first) {
#pragma unroll
    for (int u = 0; u < kGemvPre; ++u) {
      const int kb = warp + 8 * u;
      if (kb < KB) {
        const uint4* blk = base + size_t(kb) * 1024;
#pragma unroll
        for (int q = 0; q < 4; ++q) wpre[u][q] = __ldcs(blk + lane + 32 * q);
      }
    }
  }
  // 3) stream: acc[token][row slot]
  float acc[MT][4];
#pragma unroll
  for (int t = 0; t < MT; ++t)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[t][q] = 0.f;
  auto consume = [&](const uint4 (&w)[4], int kb) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int row = rl + 4 * q;            // row within the 16-row group (row & 7 == (rl + 4q) & 7)
      const int c = p ^ (row & 7);           // logical chunk held by physical chunk p
      float f[8];
      bf16x8_to_f32(w[q], f);
      const float* xk = xs + kb * 64 + c * 8;
#pragma unroll
      for (int t = 0; t < MT; ++t) {
        const float4 a = *reinterpret_cast<const float4*>(xk + size_t(t) * K);
        const float4 b = *reinterpret_cast<const float4*>(xk + size_t(t) * K + 4);
        float s = acc[t][q];
        s = fmaf(f[0], a.x, s); s = fmaf(f[1], a.y, s); s = fmaf(f[2], a.z, s); s = fmaf(f[3], a.w, s);
        s = fmaf(f[4], b.x, s); s = fmaf(f[5], b.y, s); s = fmaf(f[6], b.z, s); s = fmaf(f[7], b.w, s);
        acc[t][q] = s;
      }
    }
  };
#pragma unroll
  for (int u = 0; u < kGemvPre; ++u)
    if (warp + 8 * u < KB) consume(wpre[u], warp + 8 * u);
  constexpr int B = 4;  // k-blocks in flight per warp
  for (int kb0 = warp + 8 * kGemvPre; kb0 < KB; kb0 += 8 * B) {
    uint4 w[B][4];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int kb = kb0 + 8 * u;
      if (kb < KB) {
        const uint4* blk = base + size_t(kb) * 1024;
#pragma unroll
        for (int q = 0; q < 4; ++q) w[u][q] = __ldcs(blk + lane + 32 * q);
      }
    }
#pragma unroll
    for (int u = 0; u < B; ++u)
      if (kb0 + 8 * u < KB) consume(w[u], kb0 + 8 * u);
  }
  // 4) reduce: the 8 lanes of a row (xor 1, 2, 4), then the 8 warps
#pragma unroll
  for (int t = 0; t < MT; ++t)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      float v = acc[t][q];
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      if (p == 0) red[(warp * MT + t) * kGemvRows + rl + 4 * q] = v;
    }
  __syncthreads();
  if (warp < (MT * kGemvRows + 31) / 32) {  // whole warps: the SwiGLU pairing shuffles
    const int t = threadIdx.x / kGemvRows, r = threadIdx.x % kGemvRows;
    const bool ok = t < MT;
    float v = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < 8; ++w2) v += ok ? red[(w2 * MT + t) * kGemvRows + r] : 0.f;
    const int row = g * kGemvRows + r;
    if (EPI == EPI_SWIGLU) {
      const float up = __shfl_xor_sync(0xffffffffu, v, 1);  // rows 2j (gate), 2j+1 (up) in adjacent lanes
      if (ok && (r & 1) == 0 && row < N && t < M)
        Yb[size_t(t) * ldyb + (row >> 1)] = __float2bfloat16_rn(v / (1.0f + expf(-v)) * up);
    } else if (ok && row < N && t < M) {
      Y[size_t(t) * ldy + row] = v;
    }
  }
  __syncthreads();  // red[] is reused by the next row group
  }
  KTL_EXIT();
}

__host__ __device__ constexpr size_t gemv_smem(int MT, int K) {
  return (size_t(MT) * K + size_t(8) * MT * kGemvRows) * 4;
}

}  // namespace ssd
