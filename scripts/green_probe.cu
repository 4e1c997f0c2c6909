// Feasibility probe for green-context SM partitioning of the colocated SSD
// round (verifier stream vs speculator stream). Checks, on one B200:
//   1. runtime <<<>>> launches into streams made by cuGreenCtxStreamCreate,
//   2. the SM sets each stream's blocks land on (direct launch),
//   3. the same after stream capture across both streams into one graph.
// nvcc -gencode arch=compute_100a,code=sm_100a -o green_probe green_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <set>
#include <vector>

#define CU(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); \
  std::printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, s); return 1; } } while (0)
#define CR(x) do { cudaError_t r = (x); if (r != cudaSuccess) { \
  std::printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(r)); return 1; } } while (0)

__global__ void smid_kernel(int* out, int spin) {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  long long t0 = clock64();
  while (clock64() - t0 < spin) {}
  if (threadIdx.x == 0) out[blockIdx.x] = int(s);
}

static std::set<int> sms(const std::vector<int>& v) { return std::set<int>(v.begin(), v.end()); }

int main(int argc, char** argv) {
  const unsigned want = argc > 1 ? unsigned(std::atoi(argv[1])) : 48;
  CR(cudaSetDevice(0));
  CR(cudaFree(nullptr));
  CUdevice dev;
  CU(cuDeviceGet(&dev, 0));
  CUdevResource all, grp, rest;
  CU(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  unsigned n = 1;
  CU(cuDevSmResourceSplitByCount(&grp, &n, &all, &rest, 0, want));
  std::printf("device SMs %u -> group %u SMs (n=%u), remaining %u SMs\n", all.sm.smCount, grp.sm.smCount, n,
              rest.sm.smCount);
  CUdevResourceDesc da, db;
  CU(cuDevResourceGenerateDesc(&da, &grp, 1));
  CU(cuDevResourceGenerateDesc(&db, &rest, 1));
  CUgreenCtx ga, gb;
  CU(cuGreenCtxCreate(&ga, da, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CU(cuGreenCtxCreate(&gb, db, dev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream sa, sb;
  CU(cuGreenCtxStreamCreate(&sa, ga, CU_STREAM_NON_BLOCKING, 0));
  CU(cuGreenCtxStreamCreate(&sb, gb, CU_STREAM_NON_BLOCKING, 0));
  const int nb = 2 * 148;
  int *oa, *ob;
  CR(cudaMalloc(&oa, nb * sizeof(int)));
  CR(cudaMalloc(&ob, nb * sizeof(int)));
  std::vector<int> ha(nb), hb(nb);
  auto report = [&](const char* tag) -> int {
    CR(cudaMemcpy(ha.data(), oa, nb * sizeof(int), cudaMemcpyDeviceToHost));
    CR(cudaMemcpy(hb.data(), ob, nb * sizeof(int), cudaMemcpyDeviceToHost));
    auto A = sms(ha), B = sms(hb);
    int overlap = 0;
    for (int s : A) overlap += B.count(s);
    std::printf("%s: stream A on %zu SMs, stream B on %zu SMs, overlap %d\n", tag, A.size(), B.size(), overlap);
    return 0;
  };
  smid_kernel<<<nb, 128, 0, (cudaStream_t)sa>>>(oa, 200000);
  smid_kernel<<<nb, 128, 0, (cudaStream_t)sb>>>(ob, 200000);
  CR(cudaGetLastError());
  CR(cudaDeviceSynchronize());
  if (report("direct")) return 1;
  CR(cudaMemset(oa, 0xff, nb * sizeof(int)));
  CR(cudaMemset(ob, 0xff, nb * sizeof(int)));
  // capture A and B into one graph (fork/join through events)
  cudaEvent_t fork, join;
  CR(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  CR(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CR(cudaStreamBeginCapture((cudaStream_t)sa, cudaStreamCaptureModeThreadLocal));
  CR(cudaEventRecord(fork, (cudaStream_t)sa));
  CR(cudaStreamWaitEvent((cudaStream_t)sb, fork, 0));
  smid_kernel<<<nb, 128, 0, (cudaStream_t)sa>>>(oa, 200000);
  smid_kernel<<<nb, 128, 0, (cudaStream_t)sb>>>(ob, 200000);
  CR(cudaEventRecord(join, (cudaStream_t)sb));
  CR(cudaStreamWaitEvent((cudaStream_t)sa, join, 0));
  CR(cudaStreamEndCapture((cudaStream_t)sa, &g));
  CR(cudaGraphInstantiate(&ge, g, 0));
  // launch the graph on an ordinary stream and on the green stream
  cudaStream_t plain;
  CR(cudaStreamCreateWithFlags(&plain, cudaStreamNonBlocking));
  CR(cudaGraphLaunch(ge, plain));
  CR(cudaStreamSynchronize(plain));
  if (report("graph on plain stream")) return 1;
  CR(cudaMemset(oa, 0xff, nb * sizeof(int)));
  CR(cudaMemset(ob, 0xff, nb * sizeof(int)));
  CR(cudaGraphLaunch(ge, (cudaStream_t)sa));
  CR(cudaStreamSynchronize((cudaStream_t)sa));
  if (report("graph on green stream A")) return 1;
  // timing: graph with both vs A alone
  cudaEvent_t t0, t1;
  CR(cudaEventCreate(&t0));
  CR(cudaEventCreate(&t1));
  CR(cudaEventRecord(t0, plain));
  for (int i = 0; i < 10; ++i) CR(cudaGraphLaunch(ge, plain));
  CR(cudaEventRecord(t1, plain));
  CR(cudaEventSynchronize(t1));
  float ms;
  CR(cudaEventElapsedTime(&ms, t0, t1));
  std::printf("graph x10: %.3f ms\n", ms);
  // timing event nodes inside the graph (the engine's round profile): events
  // recorded on the green streams around each branch
  {
    cudaEvent_t e[4];
    for (auto& x : e) CR(cudaEventCreate(&x));
    cudaGraph_t g2;
    cudaGraphExec_t ge2;
    CR(cudaStreamBeginCapture((cudaStream_t)sa, cudaStreamCaptureModeThreadLocal));
    CR(cudaEventRecord(e[0], (cudaStream_t)sa));
    CR(cudaEventRecord(fork, (cudaStream_t)sa));
    CR(cudaStreamWaitEvent((cudaStream_t)sb, fork, 0));
    CR(cudaEventRecord(e[2], (cudaStream_t)sb));
    smid_kernel<<<nb, 128, 0, (cudaStream_t)sa>>>(oa, 200000);
    smid_kernel<<<nb, 128, 0, (cudaStream_t)sb>>>(ob, 400000);
    CR(cudaEventRecord(e[1], (cudaStream_t)sa));
    CR(cudaEventRecord(e[3], (cudaStream_t)sb));
    CR(cudaEventRecord(join, (cudaStream_t)sb));
    CR(cudaStreamWaitEvent((cudaStream_t)sa, join, 0));
    CR(cudaStreamEndCapture((cudaStream_t)sa, &g2));
    CR(cudaGraphInstantiate(&ge2, g2, 0));
    for (int it = 0; it < 3; ++it) {
      CR(cudaEventRecord(t0, plain));
      CR(cudaGraphLaunch(ge2, plain));
      CR(cudaEventRecord(t1, plain));
      CR(cudaEventSynchronize(t1));
      float tot, a, b, ab;
      CR(cudaEventElapsedTime(&tot, t0, t1));
      CR(cudaEventElapsedTime(&a, e[0], e[1]));
      CR(cudaEventElapsedTime(&b, e[2], e[3]));
      CR(cudaEventElapsedTime(&ab, e[0], e[3]));
      std::printf("timed graph: total %.3f ms, A %.3f, B %.3f, A0->B1 %.3f\n", tot, a, b, ab);
    }
    // the same with plain (non-green) streams
    cudaStream_t pa, pb;
    CR(cudaStreamCreateWithFlags(&pa, cudaStreamNonBlocking));
    CR(cudaStreamCreateWithFlags(&pb, cudaStreamNonBlocking));
    cudaGraph_t g3;
    cudaGraphExec_t ge3;
    CR(cudaStreamBeginCapture(pa, cudaStreamCaptureModeThreadLocal));
    CR(cudaEventRecord(e[0], pa));
    CR(cudaEventRecord(fork, pa));
    CR(cudaStreamWaitEvent(pb, fork, 0));
    CR(cudaEventRecord(e[2], pb));
    smid_kernel<<<nb, 128, 0, pa>>>(oa, 200000);
    smid_kernel<<<nb, 128, 0, pb>>>(ob, 400000);
    CR(cudaEventRecord(e[1], pa));
    CR(cudaEventRecord(e[3], pb));
    CR(cudaEventRecord(join, pb));
    CR(cudaStreamWaitEvent(pa, join, 0));
    CR(cudaStreamEndCapture(pa, &g3));
    CR(cudaGraphInstantiate(&ge3, g3, 0));
    for (int it = 0; it < 3; ++it) {
      CR(cudaEventRecord(t0, plain));
      CR(cudaGraphLaunch(ge3, plain));
      CR(cudaEventRecord(t1, plain));
      CR(cudaEventSynchronize(t1));
      float tot, a, b, ab;
      CR(cudaEventElapsedTime(&tot, t0, t1));
      CR(cudaEventElapsedTime(&a, e[0], e[1]));
      CR(cudaEventElapsedTime(&b, e[2], e[3]));
      CR(cudaEventElapsedTime(&ab, e[0], e[3]));
      std::printf("plain timed graph: total %.3f ms, A %.3f, B %.3f, A0->B1 %.3f\n", tot, a, b, ab);
    }
  }
  std::printf("OK\n");
  return 0;
}
