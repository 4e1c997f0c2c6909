// tcgen05.mma (kind::f16, cta_group::1, M = 128, K = 16) issue/execute rate
// on one SM for N in {16, 32, 64, 128, 256}: operands in shared memory
// (SWIZZLE_128B K-major, contents irrelevant), one converged warp issuing
// back to back with one elected lane, a commit every 8 MMAs (one 32 KB
// weight unit of the GEMM) and a wait at the end. Prints cycles per MMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sw128(uint32_t a) {
  return uint64_t((a >> 4) & 0x3FFF) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) | (uint64_t(1) << 46) |
         (uint64_t(2) << 61);
}

// MODE bit 0: commit to an mbarrier after every unit; bit 1: tcgen05.fence::after_thread_sync
// per unit; bit 2: mbarrier try_wait on an already-completed phase per unit
template <int N, int MODE>
__global__ void __launch_bounds__(128, 1) rate_kernel(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = base;               // 32 KB: 2 k-blocks of 128 x 64 bf16
  uint8_t* sB = base + 32768;       // N x 128 bf16
  __shared__ uint64_t bar, ubar[8], dbar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&ubar[i])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&dbar)));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&dbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
  const uint64_t ad0 = sw128(su32(sA)), bd0 = sw128(su32(sB));
  long long t0 = 0, t1 = 0;
  if (warp == 1) {
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (MODE & 4) {
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                       : "=r"(ok)
                       : "r"(su32(&dbar))
                       : "memory");
      }
      if (MODE & 2) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint64_t ad = ad0 + uint64_t((h * 16384) >> 4), bd = bd0 + uint64_t((h * N * 128) >> 4);
        asm volatile(
            "{\n\t.reg .pred e;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
            "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, 1;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc));
      }
      if (MODE & 1)
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&ubar[it & 7]))
            : "memory");
      if (it + 1 == iters)
        asm volatile(
            "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&bar))
            : "memory");
    }
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(su32(&bar))
                   : "memory");
    t1 = clock64();
    if ((threadIdx.x & 31) == 0) out[0] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

template <int N, int MODE = 0>
static void run() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int smem = 1024 + 32768 + N * 256;
  cudaFuncSetAttribute(rate_kernel<N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int iters : {64, 1024}) {
    rate_kernel<N, MODE><<<1, 128, smem>>>(iters, d);
    unsigned long long c = 0;
    cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
    std::printf("mode %d N %3d iters %5d: %.1f cycles per MMA (%.1f per 32 KB unit) %s\n", MODE, N, iters, double(c) / (iters * 8),
                double(c) / iters, cudaGetErrorString(cudaGetLastError()));
  }
  cudaFree(d);
}

// The GEMM's MMA-only protocol: warp 0 = producer (wait empty[s], arrive
// full[s]), warp 1 = MMA issuer (wait full[s], fence, 8 MMAs, commit
// empty[s]), warps 2-5 = idle epilogue warps waiting on an unfired barrier
// (SPIN: try_wait loop; else they exit). S stages.
template <int N, int S, bool SPIN>
__global__ void __launch_bounds__(192, 1) ring_kernel(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = base;
  uint8_t* sB = base + 32768;
  __shared__ uint64_t full[S], empty[S], fin, never;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[i])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&fin)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&never)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  auto wait = [](uint64_t* b, uint32_t par) {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok)
                   : "r"(su32(b)), "r"(par)
                   : "memory");
  };
  constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
  const uint64_t ad0 = sw128(su32(sA)), bd0 = sw128(su32(sB));
  if (warp == 0) {
    for (int i = 0; i < iters; ++i) {
      const int s = i % S;
      if (i >= S) wait(&empty[s], ((i / S) - 1) & 1);
      if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&full[s])) : "memory");
    }
  } else if (warp == 1) {
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int s = i % S;
      wait(&full[s], (i / S) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint64_t ad = ad0 + uint64_t((h * 16384) >> 4), bd = bd0 + uint64_t((h * N * 128) >> 4);
        asm volatile(
            "{\n\t.reg .pred e;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
            "add.s64 b1, %2, 2;\n\tadd.s64 b2, %2, 4;\n\tadd.s64 b3, %2, 6;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, 1;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, 1;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc));
      }
      asm volatile(
          "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
          "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&empty[s]))
          : "memory");
    }
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(su32(&fin))
        : "memory");
    wait(&fin, 0);
    if ((threadIdx.x & 31) == 0) out[0] = (unsigned long long)(clock64() - t0);
    if ((threadIdx.x & 31) == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&never)) : "memory");
  } else if (SPIN) {
    wait(&never, 0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

template <int N, int S, bool SPIN>
static void run_ring() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  const int smem = 1024 + 32768 + N * 256;
  cudaFuncSetAttribute(ring_kernel<N, S, SPIN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 1024;
  ring_kernel<N, S, SPIN><<<1, 192, smem>>>(iters, d);
  unsigned long long c = 0;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  std::printf("ring S %d spin %d N %3d: %.1f cycles per 32 KB unit %s\n", S, int(SPIN), N, double(c) / iters,
              cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<16>();
  run<32>();
  run<128>();
  run<16, 1>();
  run<16, 2>();
  run<16, 4>();
  run<16, 7>();
  run<32, 7>();
  run_ring<16, 6, false>();
  run_ring<16, 6, true>();
  run_ring<32, 6, true>();
  run_ring<16, 2, true>();
  return 0;
}
