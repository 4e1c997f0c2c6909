// tcgen05 weight-streaming GEMM for every linear layer of the decode step
// (SURVEY §2.3 K1/K2/K3): Y[m][n] (+)= sum_k W[n][k] X[m][k] for M = 1..256
// tokens. Swap-AB: the weight tile is the M = 128 operand (A, K-major), the
// tokens are the N operand (B, K-major, padded to NP, a multiple of 16);
// D = W_tile · X^T accumulates in TMEM.
//
// Weights live pre-tiled in HBM: block (tile t, k-block kb)
// is one contiguous 16 KB run holding the 128 x 64 bf16 tile already in the
// SWIZZLE_128B K-major order of the UMMA descriptor, and the k-blocks of a
// tile are adjacent, so one 1-D bulk copy (cp.async.bulk) streams KPS
// k-blocks (a "unit") at full DRAM efficiency.
//
// Persistent stream-K: the tiles x units work items are split into gridDim.x
// contiguous ranges; a range crosses tile boundaries, so every CTA streams
// the same number of bytes. Warp 0 / lane 0 is the producer (weights are
// issued before griddepcontrol.wait: they do not depend on the previous
// kernel — PDL overlaps the weight stream with its tail), warp 1 / lane 0
// issues tcgen05.mma into a double-buffered TMEM accumulator, warps 2-5
// drain TMEM and apply the epilogue. A tile split between CTAs is reduced by
// its last-arriving segment in a fixed order (deterministic).
#pragma once

#include <cuda.h>

#include "kernels.cuh"

// Measured on B200 (scripts/tma_probe.py, scripts/gemm_trace.py, profiles/):
// bulk copies need >= 16 KB blocks (8 KB blocks halve the bandwidth), the
// loaded issue->land latency is ~2.6 us, so one SM needs ~140 KB in flight
// for its 1/148 share of 7.1 TB/s: 6 stages of 32 KB (two k-blocks per
// stage, which also halves the per-stage barrier round trips). With this
// ring the 8B LM head streams at ~7.1 TB/s; the per-kernel cold start is
// hidden by the L2 prefetch chain (GemmArgs::nextW).
#ifndef SSD_GEMM_SMEM_KB
#define SSD_GEMM_SMEM_KB 220
#endif
#ifndef SSD_GEMM_KPS
#define SSD_GEMM_KPS 2
#endif
#ifndef SSD_GEMM_MAX_STAGES
#define SSD_GEMM_MAX_STAGES 6
#endif
#ifndef SSD_GEMM_SPIN
#define SSD_GEMM_SPIN 0
#endif
#ifndef SSD_GEMM_SLEEP_EPI
#define SSD_GEMM_SLEEP_EPI 0
#endif
#ifndef SSD_GEMM_NO_B_RELOAD
#define SSD_GEMM_NO_B_RELOAD 0
#endif

namespace ssd {
namespace tc {

#ifndef SSD_GEMM_TRACE
#define SSD_GEMM_TRACE 0
#endif
#if SSD_GEMM_TRACE
// [0][i]: producer issue of unit i; [1][i]: MMA saw full; [2][i]: MMA
// committed; [3][i]: producer saw empty (slot reuse); [4][0..1]: start/end.
__device__ unsigned long long g_trace[5][512];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(row, i) \
  do { if (blockIdx.x == 0 && (i) < 512) g_trace[row][i] = gtime(); } while (0)
#else
#define TRACE(row, i) do {} while (0)
#endif

constexpr int kBM = 128;        // weight rows per tile (UMMA M)
constexpr int kBK = 64;         // K per block: one 128-byte swizzle atom of bf16
constexpr int kKPS = SSD_GEMM_KPS;          // k-blocks per pipeline stage
constexpr int kABlock = kBM * kBK * 2;      // 16 KB
constexpr int kABytes = kABlock * kKPS;
constexpr int kThreads = 192;   // 6 warps
static_assert(kABytes == kPfUnitBytes, "prefetch windows assume 32 KB units");
// Stage budget per CTA; the host launches enough CTAs per SM to fill it.
constexpr int kSmemBudget = SSD_GEMM_SMEM_KB * 1024;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// Blocking wait (try_wait suspends the thread in hardware between probes).
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// Sleeping wait for threads that idle for the whole main loop (epilogue):
// keeps 128 waiting threads off the shared-memory barrier unit.
__device__ __forceinline__ void mbar_sleep_wait(uint64_t* b, uint32_t parity) {
#if SSD_GEMM_SLEEP_EPI
  uint32_t ok = 0;
  while (true) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    if (ok) break;
    __nanosleep(SSD_GEMM_SLEEP_EPI);
  }
#else
  mbar_wait(b, parity);
#endif
}

// Polling wait for the latency-critical producer / MMA threads.
__device__ __forceinline__ void mbar_spin(uint64_t* b, uint32_t parity) {
#if SSD_GEMM_SPIN
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "SPIN_%=:\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra SPIN_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
#else
  mbar_wait(b, parity);
#endif
}

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// Converged-warp producer steps (one elected lane issues; warp-uniform
// operands stay in uniform registers, see the MMA issuer).
__device__ __forceinline__ void expect_bulk_elect(uint64_t* bar, uint32_t tx, void* dst, const void* src, uint32_t bytes,
                                                  uint64_t policy) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n\t"
      "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%2], [%3], %4, [%0], %5;\n\t}"
      ::"r"(smem_u32(bar)), "r"(tx), "r"(smem_u32(dst)), "l"(src), "r"(bytes), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_elect(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n\t}" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// PDL (programmatic dependent launch)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

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

// Issued by a converged warp: one elected lane issues (operands warp-uniform).
__device__ __forceinline__ void mma_bf16_elect(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// The four K = 16 MMAs of one 64-wide k-block (one swizzle atom: the
// descriptors advance by 32 bytes = 2 in the >> 4 address field), in one asm
// block so the descriptor adds stay next to the MMAs (fewer uniform-register
// moves per MMA). acc: accumulate into D on the first MMA.
__device__ __forceinline__ void mma4_bf16_elect(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, q, e;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "setp.eq.b32 q, %4, %4;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, q;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, q;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}

struct GemmArgs {
  const bf16* W;  // pre-tiled weights
  int N;          // weight rows (logical)
  int KU;         // units per tile (K / (64 * KPS))
  int M;          // tokens (valid columns)
  float* Y;       // EPI_STORE / EPI_RESID output [M][ldy]
  int ldy;
  bf16* Yb;       // EPI_SWIGLU output [M][ldyb]
  int ldyb;
  float* ws;      // partials [2 * gridDim][M][128]
  int* counters;  // per-tile arrival counters (zeroed, self-resetting)
  // L2 prefetch window of the weight stream ahead of this GEMM (kernels.cuh
  // prefetch_window), issued once this CTA's own weight stream is issued:
  // it covers the drain / epilogue / next-launch gap.
  Prefetch pf;
  int dbg_seq;  // profiling build: launch sequence number (per-CTA timeline)
  // 1: a tile split between CTAs is summed with fp32 atomics straight into Y
  // (pre-zeroed for EPI_STORE; the residual stream itself for EPI_RESID)
  // instead of partials + a last-arriver reduction: no ticket / reduce round
  // trips after the last MMA, summation order not fixed.
  int atomic;
};

template <int EPI>
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

// Unit range of CTA i: [i*U/P, (i+1)*U/P).
__device__ __forceinline__ int unit_begin(long long i, long long U, long long P) { return int(i * U / P); }
// CTA owning unit u.
__device__ __forceinline__ int cta_of(int u, long long U, long long P) {
  long long i = ((long long)u * P) / U;
  while (i + 1 < P && unit_begin(i + 1, U, P) <= u) ++i;
  while (i > 0 && unit_begin(i, U, P) > u) --i;
  return int(i);
}

// BUDGET_KB: shared-memory stage budget. The full budget (one CTA per SM,
// ~190 KB in flight) streams large GEMMs at HBM speed; the small budget
// (kSmallBudgetKB) lets the next GEMM's CTA be resident beside the current
// one, so under PDL it launches, allocates and starts its weight stream
// while the current one drains (what the small per-layer GEMMs of a 1B
// draft step are bound by).
constexpr int kSmallBudgetKB = 108;
template <int NP, int BUDGET_KB = SSD_GEMM_SMEM_KB>
struct Cfg {
  static constexpr int kBudget = BUDGET_KB * 1024;
  static constexpr int kBBlock = NP * kBK * 2;
  static constexpr int kBBytes = kBBlock * kKPS;
  static constexpr int kStageBytes = kABytes + kBBytes;
  // staging tile of the atomic split-K epilogue: [NP tokens][128 rows] fp32,
  // added into Y with one TMA bulk reduce per token row (NP = 32: the M = 17..32
  // branch steps; at M <= 16 a few atomics per thread are cheaper)
  static constexpr int kCBytes = NP == 32 ? NP * kBM * 4 : 0;
  // (the staging tile comes out of the 227 KB CTA limit, not the stage budget,
  // while both fit: NP = 16 keeps its 6 stages)
  static constexpr int kRing = kBudget < 227 * 1024 - 1280 - kCBytes ? kBudget : 227 * 1024 - 1280 - kCBytes;
  static constexpr int kStages = (kRing / kStageBytes) < 2 ? 2
                                 : ((kRing / kStageBytes) > SSD_GEMM_MAX_STAGES ? SSD_GEMM_MAX_STAGES
                                                                                : kRing / kStageBytes);
  static constexpr int kAccCols = NP < 32 ? 32 : NP;
  static constexpr int kTmemCols = 2 * kAccCols <= 64 ? 64 : (2 * kAccCols <= 128 ? 128 : (2 * kAccCols <= 256 ? 256 : 512));
  static constexpr size_t kSmem = 1024 + size_t(kStages) * kStageBytes + kCBytes + 256;
};

// Add `bytes` of fp32 from shared memory into global memory (TMA bulk
// reduce-add at L2: one instruction per contiguous row instead of a red per
// element).
__device__ __forceinline__ void bulk_reduce_add_f32(float* dst, const float* src, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}

template <int EPI, int NP, int BUDGET_KB = SSD_GEMM_SMEM_KB>
__global__ void __launch_bounds__(kThreads, 1) gemm_tc_kernel(const __grid_constant__ CUtensorMap mapX, GemmArgs g) {
  using C = Cfg<NP, BUDGET_KB>;
  constexpr int S = C::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * kABytes;
  float* sC = reinterpret_cast<float*>(sB + S * C::kBBytes);  // [NP][128] (kCBytes)
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + S * C::kBBytes + C::kCBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;   // [2]
  uint64_t* tempty = tfull + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  __shared__ int s_last;

  KTL_ENTER(10 + EPI);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles = (g.N + kBM - 1) / kBM;
  const long long U = (long long)tiles * g.KU, P = gridDim.x;
  const int u0 = unit_begin(blockIdx.x, U, P), u1 = unit_begin(blockIdx.x + 1, U, P);

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  pdl_launch();  // let the next kernel start its own prologue / weight prefetch

  if (warp == 0) {
    // ---------------- producer (converged warp, elected issue)
    uint64_t pol_w;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_w));
    if (lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&mapX) : "memory");
    const int n = u1 - u0;
    const int pre = n < S ? n : S;
    if (threadIdx.x == 0) TRACE(4, 0);
    for (int i = 0; i < pre; ++i) {  // weights only: independent of the previous kernel
      expect_bulk_elect(&full[i], C::kStageBytes, sA + i * kABytes, g.W + size_t(u0 + i) * (kABytes / 2), kABytes,
                        pol_w);
      if (lane == 0) TRACE(0, i);
    }
    pdl_wait();  // activations are produced by the previous kernel
    KTL_READY();
#if SSD_KTL
    if (lane == 0 && blockIdx.x < 160) g_ktl_cta[g.dbg_seq & 63][blockIdx.x][0] = ktl_now();
#endif
    for (int i = 0; i < pre; ++i) {
      const int kb = ((u0 + i) % g.KU) * kKPS;
#pragma unroll
      for (int h = 0; h < kKPS; ++h)
        tma_load_2d_elect(sB + i * C::kBBytes + h * C::kBBlock, &mapX, &full[i], (kb + h) * kBK, 0);
    }
    int ku = (u0 + pre) % g.KU, s = pre % S;  // kept incrementally (no divisions in the loop)
    uint32_t ph = pre / S - 1;                // parity of the empty phase awaited for unit i >= S
    for (int i = pre; i < n; ++i) {
      mbar_spin(&empty[s], ph & 1);
      if (lane == 0) TRACE(3, i);
      const int u = u0 + i;
#if SSD_GEMM_NO_B_RELOAD  // bandwidth experiment only: stale activations
      expect_bulk_elect(&full[s], kABytes, sA + s * kABytes, g.W + size_t(u) * (kABytes / 2), kABytes, pol_w);
#else
      expect_bulk_elect(&full[s], C::kStageBytes, sA + s * kABytes, g.W + size_t(u) * (kABytes / 2), kABytes, pol_w);
      const int kb = ku * kKPS;
#pragma unroll
      for (int h = 0; h < kKPS; ++h)
        tma_load_2d_elect(sB + s * C::kBBytes + h * C::kBBlock, &mapX, &full[s], (kb + h) * kBK, 0);
#endif
      if (lane == 0) TRACE(0, i);
      if (++ku == g.KU) ku = 0;
      if (++s == S) { s = 0; ++ph; }
    }
    if (lane == 0) prefetch_window(g.pf, kABytes);
  } else if (warp == 1) {
    // ---------------- MMA issuer. The whole warp runs the loop, so the
    // descriptors are warp-uniform values the compiler keeps in uniform
    // registers, and one elected lane issues each tcgen05.mma / commit. (A
    // lone lane-0 branch made every MMA a divergent ELECT / R2UR.BROADCAST
    // loop of ~20 instructions: ~150 cycles per MMA, the issue rate, not the
    // tensor core or HBM, bounded a CTA at ~55 GB/s — scripts/gemm_trace.py,
    // profiles/r02g_summary.md.)
    constexpr uint32_t idesc = idesc_bf16(kBM, NP);
    const uint64_t adesc0 = sw128_desc(smem_u32(sA)), bdesc0 = sw128_desc(smem_u32(sB));
    int seg = -1;
    // tile position of unit u0 + i, kept incrementally (no divisions in the loop)
    int ku = u0 % g.KU, s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < u1 - u0; ++i) {
      const int u = u0 + i;
      const bool first = i == 0 || ku == 0;
      if (first) {
        ++seg;
        if (seg >= 2) mbar_spin(&tempty[seg & 1], ((seg >> 1) - 1) & 1);
      }
      mbar_spin(&full[s], ph);
      if (lane == 0) TRACE(1, i);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t d = tmem + uint32_t((seg & 1) * C::kAccCols);
      static_assert(kBK == 64, "mma4: four K = 16 MMAs per k-block");
#pragma unroll
      for (int h = 0; h < kKPS; ++h) {
        // descriptor start address field = smem address >> 4 (< 2^14: no carry)
        const uint64_t ad = adesc0 + uint64_t((s * kABytes + h * kABlock) >> 4);
        const uint64_t bd = bdesc0 + uint64_t((s * C::kBBytes + h * C::kBBlock) >> 4);
        mma4_bf16_elect(d, ad, bd, idesc, (!first || h) ? 1u : 0u);
      }
      mma_commit_elect(&empty[s]);
      if (lane == 0) TRACE(2, i);
#if SSD_KTL
      if (lane == 0 && i + 1 == u1 - u0 && blockIdx.x < 160) g_ktl_cta[g.dbg_seq & 63][blockIdx.x][1] = ktl_now();
#endif
      const bool last = (u + 1 == u1) || (ku + 1 == g.KU);
      if (last) mma_commit_elect(&tfull[seg & 1]);
#if SSD_KTL
      if (last && u + 1 == u1 && blockIdx.x < 160) {  // profiling: when the accumulator is complete
        mbar_wait(&tfull[seg & 1], (seg >> 1) & 1);
        if (lane == 0) g_ktl_cta[g.dbg_seq & 63][blockIdx.x][7] = ktl_now();
      }
#endif
      if (++ku == g.KU) ku = 0;
      if (++s == S) { s = 0; ph ^= 1u; }
    }
  } else if (warp >= 2) {
    // ---------------- epilogue: TMEM lanes (warp % 4) * 32 + lane
    const int q = warp & 3;
    const int rl = q * 32 + lane;
    int seg = -1;
    int u = u0;
    while (u < u1) {
      const int t = u / g.KU;
      const int ku_lo = u % g.KU;
      const int seg_end = min(u1, (t + 1) * g.KU);
      const bool whole = ku_lo == 0 && seg_end == (t + 1) * g.KU;
      ++seg;
      const int b = seg & 1;
      if (lane == 0) mbar_sleep_wait(&tfull[b], (seg >> 1) & 1);
      __syncwarp();
      mbar_wait(&tfull[b], (seg >> 1) & 1);
#if SSD_KTL
      if (threadIdx.x == 64 && blockIdx.x < 160) g_ktl_cta[g.dbg_seq & 63][blockIdx.x][3] = ktl_now();
#endif
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t taddr = tmem + (uint32_t(q * 32) << 16) + uint32_t(b * C::kAccCols);
      const int r = t * kBM + rl;
      // partial slot: first segment of this CTA -> 2*cta, later -> 2*cta+1
      float* part = g.ws + (size_t(2 * blockIdx.x + (u == u0 ? 0 : 1)) * g.M) * kBM;
      // atomic mode: split segments (and whole residual tiles) are staged in
      // shared memory and added with TMA bulk reduces (NP = 32)
      const bool bulk = C::kCBytes > 0 && EPI != EPI_SWIGLU && g.atomic && (!whole || EPI == EPI_RESID);
#pragma unroll 1
      for (int c = 0; c < NP; c += 8) {
        uint32_t v[8];
        tmem_ld8(taddr + c, v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (c + 8 >= NP) {  // accumulator drained: hand it back to the MMA warp
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[b]);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float f = __uint_as_float(v[j]);
          if (bulk) {
            if (c + j < g.M) sC[(c + j) * kBM + rl] = f;
          } else if (whole) apply_epi<EPI>(g, r, c + j, f);
          else if (EPI != EPI_SWIGLU && g.atomic) {
            if (r < g.N && c + j < g.M) atomicAdd(g.Y + size_t(c + j) * g.ldy + r, f);
          } else if (c + j < g.M) part[size_t(c + j) * kBM + rl] = f;
        }
      }
      if (C::kCBytes > 0 && bulk) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // staged rows visible to the TMA unit
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 64) {
          const int rows = min(kBM, g.N - t * kBM);
          for (int m = 0; m < g.M; ++m)
            bulk_reduce_add_f32(g.Y + size_t(m) * g.ldy + size_t(t) * kBM, sC + m * kBM, uint32_t(rows) * 4);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // sC free again
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        u = seg_end;
        continue;
      }
#if SSD_KTL
      if (threadIdx.x == 64 && blockIdx.x < 160) g_ktl_cta[g.dbg_seq & 63][blockIdx.x][4] = ktl_now();
#endif
      if (!whole && !(EPI != EPI_SWIGLU && g.atomic)) {
        // last-arriving segment of tile t reduces the partials in CTA order
        const int cf = cta_of(t * g.KU, U, P), cl = cta_of((t + 1) * g.KU - 1, U, P);
        // The CTA barrier orders the 128 threads' partial stores before the
        // arrival; one acq_rel atomic (cumulative release of those stores,
        // acquire of the other contributors') replaces two full fences.
        // (Deferring the ticket past the next segment's drain was measured
        // slower: profiles/r01_summary.md.)
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 64) {
          int old;
          asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;" : "=r"(old) : "l"(&g.counters[t]) : "memory");
          s_last = old == (cl - cf);
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
#if SSD_KTL
        if (threadIdx.x == 64 && blockIdx.x < 160) g_ktl_cta[g.dbg_seq & 63][blockIdx.x][5] = ktl_now();
#endif
        if (s_last) {
          // only the first contributing CTA can start before the tile
          const int first_slot = 2 * cf + (unit_begin(cf, U, P) >= t * g.KU ? 0 : 1);
          // All partial loads of a (kC contributors x kT tokens) block are in
          // flight together, then summed in CTA order: the same order, hence
          // the same bits, as a sequential reduction. kT covers every token
          // up to NP = 32 (one L2 round trip for the usual <= 3 contributors
          // of a stream-K tile; 4 tokens per round trip took ~9 us at M = 20,
          // scripts/ktl.py)
          constexpr int kT = NP <= 32 ? NP : 16, kC = NP <= 16 ? 4 : 3;
          for (int t0 = 0; t0 < g.M; t0 += kT) {
            float acc[kT];
#pragma unroll
            for (int j = 0; j < kT; ++j) acc[j] = 0.f;
            for (int cb = cf; cb <= cl; cb += kC) {
              float v[kC][kT];
#pragma unroll
              for (int k = 0; k < kC; ++k) {
                const int c2 = cb + k;
                const int slot = c2 == cf ? first_slot : 2 * c2;
                const float* src = g.ws + (size_t(slot) * g.M) * kBM + rl;
#pragma unroll
                for (int j = 0; j < kT; ++j)
                  v[k][j] = (c2 <= cl && t0 + j < g.M) ? __ldcg(src + size_t(t0 + j) * kBM) : 0.f;
              }
#pragma unroll
              for (int k = 0; k < kC; ++k)
#pragma unroll
                for (int j = 0; j < kT; ++j)
                  if (cb + k <= cl) acc[j] += v[k][j];
            }
#pragma unroll
            for (int j = 0; j < kT; ++j) apply_epi<EPI>(g, r, t0 + j, acc[j]);
          }
          if (threadIdx.x == 64) g.counters[t] = 0;
#if SSD_KTL
          if (threadIdx.x == 64 && blockIdx.x < 160) g_ktl_cta[g.dbg_seq & 63][blockIdx.x][6] = ktl_now();
#endif
        }
      }
      u = seg_end;
    }
  }
  if (C::kCBytes > 0 && threadIdx.x == 64) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::kTmemCols));
  if (threadIdx.x == 0) TRACE(4, 1);
#if SSD_KTL
  if (threadIdx.x == 64 && blockIdx.x < 160) g_ktl_cta[g.dbg_seq & 63][blockIdx.x][2] = ktl_now();
#endif
  KTL_EXIT();
}

}  // namespace tc
}  // namespace ssd
