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

}  // namespace ssd
