// Shared device helpers for the B200 Saguaro engine (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ssd {

constexpr int kWarp = 32;
constexpr int kMaxK = 16;        // max lookahead
constexpr int kMaxM = 256;       // max tokens per forward (branches)
constexpr int kMaxTopF = 32;     // max fan-out per position (+1 for the exclusion)

// ----------------------------------------------------------- reductions
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_maxd(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// (value desc, index asc): the total order of dist::top_indices
// (categorical.cpp:42-45). True when (va, ia) ranks before (vb, ib).
__device__ __forceinline__ bool ranks_before(float va, int ia, float vb, int ib) {
  return va > vb || (va == vb && ia < ib);
}

struct VI { float v; int i; };

__device__ __forceinline__ VI warp_best(VI a) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    VI b{__shfl_xor_sync(0xffffffffu, a.v, o), __shfl_xor_sync(0xffffffffu, a.i, o)};
    if (ranks_before(b.v, b.i, a.v, a.i)) a = b;
  }
  return a;
}

// Block-wide sum / max helpers (blockDim.x multiple of 32, <= 1024).
template <typename T>
__device__ T block_sum(T v, T* sh /* >= 32 */) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  T r = lane < nw ? sh[lane] : T(0);
  r = warp_sum(r);
  return r;  // valid in every warp
}

__device__ inline double block_maxd(double v, double* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_maxd(v);
  __syncthreads();
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double r = lane < nw ? sh[lane] : -INFINITY;
  return warp_maxd(r);
}

__device__ inline VI block_best(VI a, VI* sh) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  a = warp_best(a);
  __syncthreads();
  if (lane == 0) sh[w] = a;
  __syncthreads();
  VI r = lane < nw ? sh[lane] : VI{-INFINITY, 0x7fffffff};
  return warp_best(r);
}

// ----------------------------------------------------------- kernel timeline
// Profiling build only (-DSSD_KTL=1, scripts/ktl.py): block 0 of every
// decode-step kernel records (kind, entry, after-PDL-wait, exit) globaltimer
// stamps, to see the real (PDL-overlapped, graph-launched) step timeline.
#ifndef SSD_KTL
#define SSD_KTL 0
#endif
#if SSD_KTL
__device__ unsigned long long g_ktl[16384][4];
__device__ unsigned g_ktl_n;
__device__ __forceinline__ unsigned long long ktl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ bool ktl_lead() {
  return blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0;
}
#define KTL_ENTER(kind)                                   \
  unsigned ktl_slot_ = 0xffffffffu;                       \
  if (ktl_lead()) {                                       \
    ktl_slot_ = atomicAdd(&g_ktl_n, 1u) & 16383u;         \
    g_ktl[ktl_slot_][0] = (kind);                         \
    g_ktl[ktl_slot_][1] = ktl_now();                      \
  }
#define KTL_READY() \
  if (ktl_slot_ != 0xffffffffu) g_ktl[ktl_slot_][2] = ktl_now();
#define KTL_EXIT() \
  if (ktl_slot_ != 0xffffffffu) g_ktl[ktl_slot_][3] = ktl_now();
// sub-phase stamps of the last launch of an instrumented kernel (block 0)
__device__ unsigned long long g_ktl_sub[16];
// per-CTA (ready, MMA done, exit) stamps of the last 64 GEMM launches
__device__ unsigned long long g_ktl_cta[64][160][8];
#define KTL_SUB(i) \
  if (ktl_lead()) g_ktl_sub[i] = ktl_now();
#else
#define KTL_SUB(i)
#define KTL_ENTER(kind)
#define KTL_READY()
#define KTL_EXIT()
#endif

// ----------------------------------------------------------- mt19937_64
// std::mt19937_64 (fully specified by the C++ standard); the device copy of
// the reference's rng::Stream (rng.hpp:32-48).
struct Mt64 {
  uint64_t s[312];
  int i;
};

__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
// rng.hpp:24-26
__host__ __device__ inline uint64_t derive_seed(uint64_t root, uint64_t index) {
  return splitmix64(root + (index + 1) * 0x9E3779B97F4A7C15ull);
}

__host__ __device__ inline void mt_seed(Mt64& m, uint64_t seed) {
  m.s[0] = seed;
  for (int k = 1; k < 312; ++k) m.s[k] = 6364136223846793005ull * (m.s[k - 1] ^ (m.s[k - 1] >> 62)) + uint64_t(k);
  m.i = 312;
}

__host__ __device__ inline uint64_t mt_next(Mt64& m) {
  if (m.i >= 312) {
    const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
    for (int k = 0; k < 312; ++k) {
      const uint64_t x = (m.s[k] & UM) | (m.s[(k + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
      m.s[k] = m.s[(k + 156) % 312] ^ xa;
    }
    m.i = 0;
  }
  uint64_t y = m.s[m.i++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

// rng.hpp:39-41: one engine step per uniform, top 53 bits.
__host__ __device__ inline double mt_unit(Mt64& m) { return double(mt_next(m) >> 11) * 0x1.0p-53; }

// ----------------------------------------------------------- bf16
__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

}  // namespace ssd
