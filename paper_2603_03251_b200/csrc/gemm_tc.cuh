// tcgen05 weight-streaming GEMM for the small-M forwards of the Saguaro loop:
// the (K+1)-token verify / extend forwards and the M = B branch steps of
// pre-speculation. Swap-AB: the weight tile is the
// M = 128 operand (A, K-major), the M tokens are the N operand (B, K-major,
// padded to a multiple of 16); D = W_tile · X^T accumulates in TMEM.
//
// One CTA = one 128-row weight tile x one K split. Warp 0 / lane 0 streams
// A and B stages with TMA (SWIZZLE_128B) into a 6-deep mbarrier ring; warp 1
// / lane 0 issues tcgen05.mma; all four warps then drain TMEM (tcgen05.ld,
// lane i = weight row i) and either apply the epilogue (store / residual add
// / SwiGLU) or, with split-K, write fp32 partials that the last-arriving CTA
// of the tile reduces in a fixed order (deterministic).
#pragma once

#include <cuda.h>

#include "kernels.cuh"

namespace ssd {
namespace tc {

constexpr int kBM = 128;        // weight rows per tile (UMMA M)
constexpr int kBK = 64;         // K per stage: one 128-byte swizzle atom of bf16
constexpr int kStages = 6;
constexpr int kThreads = 128;
constexpr int kABytes = kBM * kBK * 2;  // 16 KB

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// sm100 shared-memory matrix descriptor, K-major SWIZZLE_128B (CUTLASS
// UMMA::SmemDescriptor): start>>4 | LBO 1 | SBO 1024B>>4 | version 1 | layout 2.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

// kind::f16 instruction descriptor: bf16 x bf16 -> f32, both K-major.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

struct GemmArgs {
  int N;        // weight rows
  int K;        // reduction length
  int M;        // tokens (valid columns)
  int splits;   // K splits
  int kb_per;   // 64-wide K blocks per split
  float* Y;     // EPI_STORE / EPI_RESID output [M][ldy]
  int ldy;
  bf16* Yb;     // EPI_SWIGLU output [M][ldyb]
  int ldyb;
  float* ws;    // split-K partials [splits][M][N]
  int* counters;  // per-tile arrival counters (zeroed, self-resetting)
};

template <int EPI, int NP>
__device__ __forceinline__ void apply_epi(const GemmArgs& g, int row, int tok, float v) {
  if (EPI == EPI_SWIGLU) {
    const float up = __shfl_xor_sync(0xffffffffu, v, 1);
    if ((row & 1) == 0 && row < g.N && tok < g.M) {
      const float act = v / (1.0f + expf(-v)) * up;
      g.Yb[size_t(tok) * g.ldyb + (row >> 1)] = __float2bfloat16_rn(act);
    }
  } else if (row < g.N && tok < g.M) {
    float* y = g.Y + size_t(tok) * g.ldy + row;
    if (EPI == EPI_RESID) *y += v;
    else *y = v;
  }
}

// NP: padded token count (UMMA N), multiple of 16 in [16, 256].
template <int EPI, int NP>
__global__ void __launch_bounds__(kThreads, 1) gemm_tc_kernel(const __grid_constant__ CUtensorMap mapW,
                                                              const __grid_constant__ CUtensorMap mapX, GemmArgs g) {
  constexpr int kBBytes = NP * kBK * 2;
  constexpr int kTmemCols = NP <= 32 ? 32 : (NP <= 64 ? 64 : (NP <= 128 ? 128 : 256));
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kBBytes);
  uint64_t* empty = full + kStages;
  uint64_t* accf = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accf + 1);
  __shared__ int s_last;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles = (g.N + kBM - 1) / kBM;
  const int tile = blockIdx.x % tiles, split = blockIdx.x / tiles;
  const int row0 = tile * kBM;
  const int kb0 = split * g.kb_per;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(accf, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // TMA producer: weights are streamed once (evict-first), activations
    // are re-read by every tile (evict-last).
    uint64_t pol_w, pol_x;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_w));
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_x));
    for (int i = 0; i < g.kb_per; ++i) {
      const int s = i % kStages;
      if (i >= kStages) mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
      mbar_expect_tx(&full[s], kABytes + kBBytes);
      const int kc = (kb0 + i) * kBK;
      tma_load_2d(sA + s * kABytes, &mapW, &full[s], kc, row0, pol_w);
      tma_load_2d(sB + s * kBBytes, &mapX, &full[s], kc, 0, pol_x);
    }
  } else if (warp == 1 && lane == 0) {
    // MMA issuer
    constexpr uint32_t idesc = idesc_bf16(kBM, NP);
    for (int i = 0; i < g.kb_per; ++i) {
      const int s = i % kStages;
      mbar_wait(&full[s], (i / kStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t a0 = smem_u32(sA + s * kABytes), b0 = smem_u32(sB + s * kBBytes);
#pragma unroll
      for (int k = 0; k < kBK / 16; ++k)
        mma_bf16(tmem, sw128_desc(a0 + k * 32), sw128_desc(b0 + k * 32), idesc, (i | k) ? 1u : 0u);
      mma_commit(&empty[s]);
    }
    mma_commit(accf);
  }
  __syncwarp();
  mbar_wait(accf, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");

  const int r = row0 + threadIdx.x;  // TMEM lane == weight row within the tile
  const uint32_t taddr = tmem + (uint32_t(warp * 32) << 16);
  if (g.splits == 1) {
#pragma unroll 1
    for (int c = 0; c < NP; c += 8) {
      float v[8];
      tmem_ld8(taddr + c, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) apply_epi<EPI, NP>(g, r, c + j, v[j]);
    }
  } else {
    float* part = g.ws + size_t(split) * g.M * g.N;
#pragma unroll 1
    for (int c = 0; c < NP; c += 8) {
      float v[8];
      tmem_ld8(taddr + c, v);
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (c + j < g.M && r < g.N) part[size_t(c + j) * g.N + r] = v[j];
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(&g.counters[tile], 1) == g.splits - 1;
    __syncthreads();
    if (s_last) {
      __threadfence();
      for (int t = 0; t < g.M; ++t) {
        float acc = 0.f;
        if (r < g.N)
          for (int sp = 0; sp < g.splits; ++sp) acc += __ldcg(g.ws + (size_t(sp) * g.M + t) * g.N + r);
        apply_epi<EPI, NP>(g, r, t, acc);
      }
      if (threadIdx.x == 0) g.counters[tile] = 0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
}

template <int NP>
constexpr size_t smem_bytes() {
  return 1024 + size_t(kStages) * (kABytes + NP * kBK * 2) + (2 * kStages + 1) * 8 + 16;
}

}  // namespace tc
}  // namespace ssd
