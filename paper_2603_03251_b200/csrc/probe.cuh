// Bandwidth probes used to choose the GEMM's weight-streaming layout
// (bench/profiling only; not on the decode path).
#pragma once

#include "gemm_tc.cuh"

namespace ssd {

// One producer lane streams `units` blocks of `ublk` bytes with S stages of
// 1-D bulk copies; one consumer lane releases each stage as it lands.
// mode 0: CTA i owns the contiguous range [i*U/P, (i+1)*U/P) of blocks;
// mode 1: block u goes to CTA u % P (all CTAs read one contiguous window).
__global__ void __launch_bounds__(64, 1) tma_stream_probe(const uint8_t* __restrict__ buf, long long units, int ublk,
                                                         int stages, int mode, unsigned* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + size_t(stages) * ublk);
  uint64_t* empty = full + stages;
  const long long P = gridDim.x, i0 = blockIdx.x;
  long long n;
  if (mode == 0) n = (i0 + 1) * units / P - i0 * units / P;
  else n = (units - i0 + P - 1) / P;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (long long i = 0; i < n; ++i) {
      const int s = int(i % stages);
      if (i >= stages) tc::mbar_wait(&empty[s], uint32_t(((i / stages) - 1) & 1));
      const long long u = mode == 0 ? i0 * units / P + i : i0 + i * P;
      tc::mbar_expect_tx(&full[s], uint32_t(ublk));
      tc::bulk_load(sm + size_t(s) * ublk, buf + size_t(u) * ublk, uint32_t(ublk), &full[s], pol);
    }
  } else if (threadIdx.x == 32) {
    unsigned acc = 0;
    for (long long i = 0; i < n; ++i) {
      const int s = int(i % stages);
      tc::mbar_wait(&full[s], uint32_t((i / stages) & 1));
      acc ^= *reinterpret_cast<const unsigned*>(sm + size_t(s) * ublk);
      tc::mbar_arrive(&empty[s]);
    }
    if (acc == 0x9e3779b9u) *sink = acc;
  }
}

// tcgen05.mma issue-to-completion rate for the GEMM's shape (M=128 weight
// tile x N tokens, K-major SW128 operands in shared memory): `iters` x 8 MMAs
// (one 32 KB unit: 2 k-blocks x 4 K=16 steps), a commit per unit, one wait
// at the end. out[0] = total cycles, out[1] = cycles of the final wait.
template <int NP>
__global__ void __launch_bounds__(64, 1) mma_rate_probe(int iters, unsigned long long* out) {
  using C = tc::Cfg<NP>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = sm;
  uint8_t* sB = sm + tc::kABytes;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sB + C::kBBytes);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 2);
  for (int i = threadIdx.x; i < (tc::kABytes + C::kBBytes) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x == 0) {
    tc::mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tslot)), "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = tc::idesc_bf16(tc::kBM, NP);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int h = 0; h < tc::kKPS; ++h) {
        const uint32_t a0 = tc::smem_u32(sA + h * tc::kABlock), b0 = tc::smem_u32(sB + h * C::kBBlock);
#pragma unroll
        for (int k = 0; k < tc::kBK / 16; ++k)
          tc::mma_bf16(tmem, tc::sw128_desc(a0 + k * 32), tc::sw128_desc(b0 + k * 32), idesc, (it || h || k) ? 1u : 0u);
      }
    }
    tc::mma_commit(bar);
    const long long t1 = clock64();
    tc::mbar_wait(bar, 0);
    const long long t2 = clock64();
    out[0] = (unsigned long long)(t2 - t0);
    out[1] = (unsigned long long)(t2 - t1);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
}

}  // namespace ssd
