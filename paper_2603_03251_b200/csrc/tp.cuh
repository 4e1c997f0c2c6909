// Tensor-parallel verifier collectives over NVLink peer memory (
// SURVEY §8e "Megatron TP ... 2 all-reduces per layer ... vocab-parallel LM
// head"). Every TP rank owns a TpRegion in its HBM, exported by CUDA IPC and
// mapped by the other ranks; a collective is ONE kernel per rank:
//   push   this rank's block into slot [rank] of every rank's region (remote
//          stores over NVLink), system fence, release-store a sequence flag;
//   wait   for the flags of all ranks;
//   reduce / gather from the local region, summing ranks in rank order, so
//          every rank gets bit-identical results (and identical verification
//          decisions) without a further exchange.
// Sequence numbers come from a per-rank device counter (advanced by the
// kernel itself, so captured graphs replay correctly); slots are
// double-buffered by sequence parity: a rank can only push collective s + 2
// after finishing s + 1, which needs every peer's s + 1 push, which each
// peer issues only after finishing its own reduction of s.
#pragma once

#include "split.cuh"

namespace ssd {

constexpr int kTpMax = 8;

struct TpFlags {
  int ar[2][kTpMax];  // all-reduce push flags (written by peers)
  int lg[2][kTpMax];  // logits all-gather push flags
};

// Region layout: [TpFlags (4 KB)] [ar slots 2 x T x maxM x d fp32] [logits 2 x maxM x V fp32]
struct TpLayout {
  int T, maxM, d, V;
  __host__ __device__ size_t ar_off() const { return 4096; }
  __host__ __device__ size_t lg_off() const { return ar_off() + size_t(2) * T * maxM * d * 4; }
  __host__ __device__ size_t bytes() const { return lg_off() + size_t(2) * maxM * V * 4; }
  __host__ __device__ float* ar_slot(char* base, int par, int r) const {
    return reinterpret_cast<float*>(base + ar_off()) + (size_t(par) * T + r) * size_t(maxM) * d;
  }
  __host__ __device__ float* lg(char* base, int par) const {
    return reinterpret_cast<float*>(base + lg_off()) + size_t(par) * maxM * V;
  }
};

struct TpPeers {
  char* region[kTpMax];  // [r]: rank r's region (own one included)
};

struct TpCtl {
  int ar_seq, lg_seq;      // collectives completed by this rank
  int push_cnt, exit_cnt;  // CTA arrival counters of the running kernel
};

__device__ __forceinline__ void tp_wait_all(const TpFlags* f, const int (*flags)[kTpMax], int par, int T, int seq,
                                            LoopState* st) {
  for (int q = 0; q < T; ++q)
    if (!wait_seq(&flags[par][q], seq, st)) return;
}

// In-place all-reduce of buf[M][d] (fp32) over the T ranks.
__global__ void __launch_bounds__(256) tp_allreduce_kernel(float* buf, int M, TpLayout L, TpPeers peers, int rank,
                                                           TpCtl* ctl, LoopState* st) {
  __shared__ int s_seq, s_last;
  if (threadIdx.x == 0) s_seq = ctl->ar_seq + 1;
  __syncthreads();
  const int seq = s_seq, par = seq & 1, T = L.T;
  const size_t n4 = size_t(M) * L.d / 4;
  const size_t i0 = blockIdx.x * size_t(blockDim.x) + threadIdx.x, step = size_t(gridDim.x) * blockDim.x;
  // push my partial into slot [rank] of every rank (row stride d inside a slot)
  for (size_t i = i0; i < n4; i += step) {
    const float4 v = reinterpret_cast<const float4*>(buf)[i];
    for (int q = 0; q < T; ++q) reinterpret_cast<float4*>(L.ar_slot(peers.region[q], par, rank))[i] = v;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&ctl->push_cnt, 1) == int(gridDim.x) - 1;
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    ctl->push_cnt = 0;
    __threadfence_system();
    for (int q = 0; q < T; ++q)
      st_release_sys(&reinterpret_cast<TpFlags*>(peers.region[q])->ar[par][rank], seq);
  }
  // wait for every rank's block, then reduce in rank order
  if (threadIdx.x == 0) {
    const TpFlags* f = reinterpret_cast<const TpFlags*>(peers.region[rank]);
    tp_wait_all(f, f->ar, par, T, seq, st);
  }
  __syncthreads();
  for (size_t i = i0; i < n4; i += step) {
    float4 acc = __ldcv(reinterpret_cast<const float4*>(L.ar_slot(peers.region[rank], par, 0)) + i);
    for (int q = 1; q < T; ++q) {
      const float4 v = __ldcv(reinterpret_cast<const float4*>(L.ar_slot(peers.region[rank], par, q)) + i);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    reinterpret_cast<float4*>(buf)[i] = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(&ctl->exit_cnt, 1) == int(gridDim.x) - 1) {
    ctl->exit_cnt = 0;
    ctl->ar_seq = seq;
  }
}

// All-gather of the vocabulary-parallel logits: shard [M][Vl] of every rank
// into columns [r * Vl, (r + 1) * Vl) of full [M][V] = dst (on every rank).
__global__ void __launch_bounds__(256) tp_gather_logits_kernel(const float* shard, int M, int Vl, float* dst, TpLayout L,
                                                               TpPeers peers, int rank, TpCtl* ctl, LoopState* st) {
  __shared__ int s_seq, s_last;
  if (threadIdx.x == 0) s_seq = ctl->lg_seq + 1;
  __syncthreads();
  const int seq = s_seq, par = seq & 1, T = L.T, V = L.V;
  const size_t n = size_t(M) * Vl;
  const size_t i0 = blockIdx.x * size_t(blockDim.x) + threadIdx.x, step = size_t(gridDim.x) * blockDim.x;
  for (size_t i = i0; i < n; i += step) {
    const size_t mrow = i / Vl, c = i % Vl;
    const float v = shard[i];
    for (int q = 0; q < T; ++q) L.lg(peers.region[q], par)[mrow * V + size_t(rank) * Vl + c] = v;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&ctl->push_cnt, 1) == int(gridDim.x) - 1;
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    ctl->push_cnt = 0;
    __threadfence_system();
    for (int q = 0; q < T; ++q)
      st_release_sys(&reinterpret_cast<TpFlags*>(peers.region[q])->lg[par][rank], seq);
  }
  if (threadIdx.x == 0) {
    const TpFlags* f = reinterpret_cast<const TpFlags*>(peers.region[rank]);
    tp_wait_all(f, f->lg, par, T, seq, st);
  }
  __syncthreads();
  const float* full = L.lg(peers.region[rank], par);
  for (size_t i = i0; i < size_t(M) * V; i += step) dst[i] = __ldcv(full + i);
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(&ctl->exit_cnt, 1) == int(gridDim.x) - 1) {
    ctl->exit_cnt = 0;
    ctl->lg_seq = seq;
  }
}

}  // namespace ssd
