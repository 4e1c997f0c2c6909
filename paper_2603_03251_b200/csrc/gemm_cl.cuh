// Cluster split-K variant of the weight-streaming GEMM (gemm_tc.cuh) for the
// small per-layer matrices of a decode step.
//
// Why: with stream-K over 148 CTAs, a small GEMM (8-50 MB) gives each CTA
// 2-10 units and splits every tile over several CTAs; the partial sums then
// go through global memory, an atomic ticket and a last-arriver reduction —
// ~6 us of round trips after the last MMA (scripts/ktl.py), longer than the
// weight streaming itself. Here the CS CTAs of a thread-block cluster split
// the K range of the same tiles; each drains its TMEM partial into its own
// shared memory, signals the other ranks' mbarriers (remote arrive over
// DSMEM), and each rank reduces a 128/CS-row slice of the tile by reading
// all CS partials over DSMEM in rank order (deterministic). No global
// partials, fences or atomics; the shared partial buffers are
// double-buffered by tile parity with a "free" barrier for reuse.
//
// Work split: cluster i owns tiles [i*T/NC, (i+1)*T/NC); rank r owns k-units
// [r*KU/CS, (r+1)*KU/CS) of each of them. Same producer (1-D bulk weights +
// 2-D TMA activations), tcgen05 swap-AB MMA into a double-buffered TMEM
// accumulator, and epilogues as gemm_tc_kernel.
#pragma once

#include "gemm_tc.cuh"

namespace ssd {
namespace tc {

__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAITC_%=;\n}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ float ld_dsmem_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <int NP, int BUDGET_KB = 224>
struct ClCfg {
  static constexpr int kBBlock = NP * kBK * 2;
  static constexpr int kBBytes = kBBlock * kKPS;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kPart = NP * kBM * 4;  // one partial [NP][128] fp32
  static constexpr int kBudget = BUDGET_KB * 1024 - 2 * kPart - 2048;
  static constexpr int kStages = (kBudget / kStageBytes) > SSD_GEMM_MAX_STAGES ? SSD_GEMM_MAX_STAGES
                                                                               : kBudget / kStageBytes;
  static_assert(kStages >= 2, "cluster GEMM: shared memory");
  static constexpr int kAccCols = NP < 32 ? 32 : NP;
  static constexpr int kTmemCols = 2 * kAccCols <= 64 ? 64 : (2 * kAccCols <= 128 ? 128 : 256);
  static constexpr size_t kSmem = 1024 + size_t(kStages) * kStageBytes + 2 * size_t(kPart) + 512;
};

// Unit range of rank r in a tile of KU units split over CS ranks.
__device__ __forceinline__ int kbeg(int r, int KU, int CS) { return r * KU / CS; }

template <int EPI, int NP, int CS, int BUDGET_KB = 224>
__global__ void __launch_bounds__(kThreads, 1) gemm_cl_kernel(const __grid_constant__ CUtensorMap mapX, GemmArgs g) {
  using C = ClCfg<NP, BUDGET_KB>;
  constexpr int S = C::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * kABytes;
  float* pbuf = reinterpret_cast<float*>(sB + S * C::kBBytes);  // [2][NP][128]
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(pbuf) + 2 * C::kPart);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;   // [2]
  uint64_t* tempty = tfull + 2;  // [2]
  uint64_t* pready = tempty + 2; // [2] all CS partials of a tile are in place
  uint64_t* pfree = pready + 2;  // [2] every rank finished reading a partial buffer
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pfree + 2);

  KTL_ENTER(20 + EPI);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = int(cluster_rank());
  const int cl = blockIdx.x / CS, NC = gridDim.x / CS;
  const int T = (g.N + kBM - 1) / kBM;
  const int t0 = int((long long)cl * T / NC), t1 = int((long long)(cl + 1) * T / NC);
  const int k0 = kbeg(rank, g.KU, CS), k1 = kbeg(rank + 1, g.KU, CS);
  const int nk = k1 - k0;  // units of each tile this rank accumulates (may be 0)

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 4);
      mbar_init(&pready[b], CS);
      mbar_init(&pfree[b], CS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  // every rank's barriers are initialised before any remote arrive
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  pdl_launch();

  if (warp == 0) {
    // ---------------- producer: the rank's k-slice of every tile of the cluster
    // (converged warp, elected issue: gemm_tc.cuh)
    uint64_t pol_w;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_w));
    if (lane == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&mapX) : "memory");
    const int n = (t1 - t0) * nk;
    const int pre = n < S ? n : S;
    for (int i = 0; i < pre; ++i) {  // weights only: independent of the previous kernel
      const int u = (t0 + i / nk) * g.KU + k0 + i % nk;
      expect_bulk_elect(&full[i], C::kStageBytes, sA + i * kABytes, g.W + size_t(u) * (kABytes / 2), kABytes, pol_w);
    }
    pdl_wait();  // activations are produced by the previous kernel
    KTL_READY();
    // (tile, k-slice, stage, parity) kept incrementally: no divisions in the loop
    int tt = t0, j = 0, s = 0;
    uint32_t ph = 0xffffffffu;  // (i / S) - 1: the empty phase awaited for i >= S
    for (int i = 0; i < n; ++i) {
      const int kk = k0 + j;
      if (i >= pre) {
        mbar_wait(&empty[s], ph & 1);
        const int u = tt * g.KU + kk;
        expect_bulk_elect(&full[s], C::kStageBytes, sA + s * kABytes, g.W + size_t(u) * (kABytes / 2), kABytes,
                          pol_w);
      }
#pragma unroll
      for (int h = 0; h < kKPS; ++h)
        tma_load_2d_elect(sB + s * C::kBBytes + h * C::kBBlock, &mapX, &full[s], (kk * kKPS + h) * kBK, 0);
      if (++j == nk) { j = 0; ++tt; }
      if (++s == S) { s = 0; ++ph; }
    }
    if (lane == 0) prefetch_window(g.pf, kABytes);
  } else if (warp == 1 && nk > 0) {
    // ---------------- MMA issuer: one accumulation segment per tile
    // (converged warp, elected issue: gemm_tc.cuh)
    constexpr uint32_t idesc = idesc_bf16(kBM, NP);
    const uint64_t adesc0 = sw128_desc(smem_u32(sA)), bdesc0 = sw128_desc(smem_u32(sB));
    int s = 0;
    uint32_t ph = 0;  // ring stage and parity, kept incrementally
    for (int t = t0; t < t1; ++t) {
      const int seg = t - t0;
      if (seg >= 2) mbar_wait(&tempty[seg & 1], ((seg >> 1) - 1) & 1);
      const uint32_t d = tmem + uint32_t((seg & 1) * C::kAccCols);
      for (int j = 0; j < nk; ++j) {
        mbar_wait(&full[s], ph & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int h = 0; h < kKPS; ++h) {
          const uint64_t ad = adesc0 + uint64_t((s * kABytes + h * kABlock) >> 4);
          const uint64_t bd = bdesc0 + uint64_t((s * C::kBBytes + h * C::kBBlock) >> 4);
          mma4_bf16_elect(d, ad, bd, idesc, (j || h) ? 1u : 0u);
        }
        mma_commit_elect(&empty[s]);
        if (++s == S) { s = 0; ph ^= 1u; }
      }
      mma_commit_elect(&tfull[seg & 1]);
    }
  } else if (warp >= 2) {
    // ---------------- epilogue: drain -> own smem partial -> signal -> reduce a row slice over DSMEM
    const int q = warp & 3;
    const int rl = q * 32 + lane;
    const int tid = threadIdx.x - 64;
    constexpr int RPR = kBM / CS;  // rows reduced by each rank
    for (int t = t0; t < t1; ++t) {
      const int seg = t - t0, b = seg & 1;
      float* mine = pbuf + b * (C::kPart / 4);
      if (seg >= 2) mbar_wait_cluster(&pfree[b], ((seg >> 1) - 1) & 1);  // all ranks done with tile seg-2
      if (nk > 0) {
        mbar_wait(&tfull[b], (seg >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t taddr = tmem + (uint32_t(q * 32) << 16) + uint32_t(b * C::kAccCols);
#pragma unroll 1
        for (int c = 0; c < NP; c += 8) {
          uint32_t v[8];
          tmem_ld8(taddr + c, v);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (c + 8 >= NP) {
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[b]);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) mine[(c + j) * kBM + rl] = __uint_as_float(v[j]);
        }
      } else {
        for (int c = 0; c < NP; ++c) mine[c * kBM + rl] = 0.f;  // no k-units: a zero partial
      }
      // Every writer's partial must be visible cluster-wide before the one
      // remote release-arrive below: a CTA barrier alone does not order other
      // threads' shared-memory writes for the peer ranks' DSMEM reads
      // (measured: first-launch garbage in ~1 of 10 processes sharing a GPU,
      // scripts/share_diag.py; with this fence 0 of 40).
      asm volatile("fence.acq_rel.cluster;" ::: "memory");
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (tid == 0)
        for (int r = 0; r < CS; ++r) mbar_arrive_remote(mapa_shared(smem_u32(&pready[b]), r));
      mbar_wait_cluster(&pready[b], (seg >> 1) & 1);
      // rows [rank*RPR, (rank+1)*RPR) x tokens: lanes cover consecutive rows
      // of one token (SwiGLU pairs rows 2j, 2j+1 in adjacent lanes)
      const uint32_t base = smem_u32(mine);
      const int items = RPR * g.M;
      for (int it0 = 0; it0 < items; it0 += 128) {
        const int it = it0 + tid;
        const bool ok = it < items;
        const int rr = rank * RPR + (ok ? it % RPR : 0), tok = ok ? it / RPR : 0;
        float acc = 0.f;
        if (ok) {
          const uint32_t off = uint32_t((tok * kBM + rr) * 4);
#pragma unroll
          for (int r = 0; r < CS; ++r) acc += ld_dsmem_f32(mapa_shared(base + off, r));
        }
        apply_epi<EPI>(g, t * kBM + rr, ok ? tok : g.M, acc);  // tok = M: no store, shuffle still taken
      }
      asm volatile("fence.acq_rel.cluster;" ::: "memory");  // this thread's DSMEM reads are done
      asm volatile("bar.sync 1, 128;" ::: "memory");
      if (tid == 0)
        for (int r = 0; r < CS; ++r) mbar_arrive_remote(mapa_shared(smem_u32(&pfree[b]), r));
    }
    // keep this rank's partial buffers alive until every rank has read them
    const int ns = t1 - t0;
    for (int seg = ns - 2 < 0 ? 0 : ns - 2; seg < ns; ++seg) mbar_wait_cluster(&pfree[seg & 1], (seg >> 1) & 1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::kTmemCols));
  KTL_EXIT();
}

}  // namespace tc
}  // namespace ssd
