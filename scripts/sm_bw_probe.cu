// Per-SM DRAM streaming rate of 1-D bulk copies (cp.async.bulk) into a
// shared-memory ring, one CTA per SM, as a function of the SMs used, the
// ring depth and the chunk size: the ceiling of the weight-streaming GEMM
// when the colocated round gives each stream a subset of the SMs.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sm_bw_probe sm_bw_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(64, 1) stream_kernel(const uint8_t* __restrict__ src, size_t bytes_per_cta,
                                                       int chunk, int stages, unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + size_t(stages) * chunk);
  const uint8_t* base = src + size_t(blockIdx.x) * bytes_per_cta;
  const int n = int(bytes_per_cta / chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  auto issue = [&](int i) {
    const int s = i % stages;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(chunk) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            su32(sm + size_t(s) * chunk)),
        "l"(base + size_t(i) * chunk), "r"(chunk), "r"(su32(&full[s])), "l"(pol)
        : "memory");
  };
  const int pre = n < stages ? n : stages;
  for (int i = 0; i < pre; ++i) issue(i);
  unsigned long long acc = 0;
  for (int i = 0; i < n; ++i) {
    const int s = i % stages;
    const uint32_t par = (i / stages) & 1;
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(su32(&full[s])), "r"(par)
                   : "memory");
    acc += sm[size_t(s) * chunk];
    if (i + stages < n) issue(i + stages);
  }
  if (acc == 0x1234567) *sink = acc;
}

// n blocks on a green context of n SMs (the colocated round's partitions)
static cudaStream_t green_stream(int n, int* got) {
  CUdevice dev;
  cuDeviceGet(&dev, 0);
  CUdevResource all, grp, rest;
  cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM);
  unsigned k = 1;
  cuDevSmResourceSplitByCount(&grp, &k, &all, &rest, 0, unsigned(n));
  CUdevResourceDesc d;
  cuDevResourceGenerateDesc(&d, &grp, 1);
  CUgreenCtx g;
  cuGreenCtxCreate(&g, d, dev, CU_GREEN_CTX_DEFAULT_STREAM);
  CUstream s;
  cuGreenCtxStreamCreate(&s, g, CU_STREAM_NON_BLOCKING, 0);
  *got = int(grp.sm.smCount);
  return reinterpret_cast<cudaStream_t>(s);
}

// producer (warp 0) / consumer (warp 1) with full + empty barriers: the
// weight-streaming GEMM's ring without the MMA
__global__ void __launch_bounds__(192, 1) pc_kernel(const uint8_t* __restrict__ src, size_t bytes_per_cta, int chunk,
                                                    int stages, unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + size_t(stages) * chunk);
  uint64_t* empty = full + stages;
  const uint8_t* base = src + size_t(blockIdx.x) * bytes_per_cta;
  const int n = int(bytes_per_cta / chunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto wait = [](uint64_t* b, uint32_t par) {
    uint32_t done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(su32(b)), "r"(par)
                   : "memory");
  };
  if (threadIdx.x == 0) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      if (i >= stages) wait(&empty[s], ((i / stages) - 1) & 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(chunk)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], "
          "%4;" ::"r"(su32(sm + size_t(s) * chunk)),
          "l"(base + size_t(i) * chunk), "r"(chunk), "r"(su32(&full[s])), "l"(pol)
          : "memory");
    }
  } else if (threadIdx.x == 32) {
    unsigned long long acc = 0;
    for (int i = 0; i < n; ++i) {
      const int s = i % stages;
      wait(&full[s], (i / stages) & 1);
      acc += sm[size_t(s) * chunk];
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
    }
    if (acc == 0x1234567) *sink = acc;
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = size_t(4) << 30;
  uint8_t* buf;
  unsigned long long* sink;
  cudaMalloc(&buf, total);
  cudaMalloc(&sink, 8);
  cudaMemset(buf, 1, total);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int ns[] = {8, 28, 56, 92, 148};
  const int chunks[] = {32768};
  const int rings[] = {196608};
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int chunk : chunks)
    for (int ring : rings)
      for (int n : ns) {
        if (n > sms) continue;
        const int stages = ring / chunk;
        const size_t per = (total / 148) / chunk * chunk;  // ~27 MB per CTA, every n fits
        const size_t smem = size_t(ring) + 8 * stages;
        stream_kernel<<<n, 64, smem>>>(buf, per, chunk, stages, sink);
        cudaEventRecord(a);
        for (int it = 0; it < 3; ++it) stream_kernel<<<n, 64, smem>>>(buf, per, chunk, stages, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) { std::printf("error\n"); return 1; }
        const double gbs = 3.0 * per * n / (ms * 1e-3) / 1e9;
        std::printf("chunk %6d ring %7d SMs %4d: %8.1f GB/s total %6.1f GB/s per SM\n", chunk, ring, n, gbs, gbs / n);
      }
  cudaFuncSetAttribute(pc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  for (int n : {56, 92, 148}) {
    const int chunk = 32768, stages = 6;
    const size_t per = (total / 148) / chunk * chunk;
    const size_t smem = 220 * 1024;
    pc_kernel<<<n, 192, smem>>>(buf, per, chunk, stages, sink);
    cudaEventRecord(a);
    for (int it = 0; it < 3; ++it) pc_kernel<<<n, 192, smem>>>(buf, per, chunk, stages, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) { std::printf("error\n"); return 1; }
    const double gbs = 3.0 * per * n / (ms * 1e-3) / 1e9;
    std::printf("producer/consumer SMs %4d: %8.1f GB/s total %6.1f GB/s per SM\n", n, gbs, gbs / n);
  }
  // green partitions: 32 KB chunks, 192 KB ring, n blocks on n SMs
  for (int n : {28, 56, 92}) {
    int got = 0;
    cudaStream_t gs = green_stream(n, &got);
    const int chunk = 32768, stages = 6;
    const size_t per = (total / 148) / chunk * chunk;
    const size_t smem = size_t(chunk) * stages + 8 * stages;
    for (int blocks : {got, 2 * got}) {
      if (blocks > 148) continue;
      const size_t per_b = blocks > got ? per / 2 / chunk * chunk : per;
      stream_kernel<<<blocks, 64, smem, gs>>>(buf, per_b, chunk, stages, sink);
      cudaEvent_t g0, g1;
      cudaEventCreate(&g0);
      cudaEventCreate(&g1);
      cudaStream_t plain;
      cudaStreamCreateWithFlags(&plain, cudaStreamNonBlocking);
      cudaDeviceSynchronize();
      cudaEventRecord(g0, plain);
      cudaStreamWaitEvent(gs, g0, 0);
      for (int it = 0; it < 3; ++it) stream_kernel<<<blocks, 64, smem, gs>>>(buf, per_b, chunk, stages, sink);
      cudaEvent_t j;
      cudaEventCreateWithFlags(&j, cudaEventDisableTiming);
      cudaEventRecord(j, gs);
      cudaStreamWaitEvent(plain, j, 0);
      cudaEventRecord(g1, plain);
      cudaEventSynchronize(g1);
      float ms;
      if (cudaEventElapsedTime(&ms, g0, g1) != cudaSuccess) { std::printf("error\n"); return 1; }
      const double gbs = 3.0 * per_b * blocks / (ms * 1e-3) / 1e9;
      std::printf("green %3d SMs, %3d blocks: %8.1f GB/s total %6.1f GB/s per SM\n", got, blocks, gbs, gbs / got);
    }
  }
  const cudaError_t e = cudaDeviceSynchronize();
  std::printf("%s\n", cudaGetErrorString(e));
  return 0;
}
