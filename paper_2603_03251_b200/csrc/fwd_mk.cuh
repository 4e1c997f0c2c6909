// Persistent forward kernel: one launch runs a whole decode / verify /
// branch step of a model.
//
// Why: at batch 1 a Llama step is ~130 dependent kernels (8B) whose fixed
// launch / ramp / drain costs (~5-10 us each) exceed the weight streaming of
// the small ones. Here every SM runs one CTA for the whole step and the
// dependent phases are separated by grid barriers, while the weight stream
// never stops: the producer warp issues the bulk copies of every GEMM of the
// step back to back into the shared-memory ring, independent of the phase
// barriers (weights do not depend on activations).
//
// Phases (ops), each ended by a grid barrier:
//   EMBED            x = E[token]                       + per-tile sum(x^2)
//   per layer:
//     QKV  GEMM      qkv = W_qkv * rmsnorm(x)          (norm fused into the B operand)
//     ATTN           RoPE + KV append + split-K flash-decoding (attn_item)
//     O    GEMM      x += W_o * attn                    + per-tile sum(x^2)
//     GU   GEMM      act = silu(g) * u, [g;u] = W_gu * rmsnorm(x) * gain
//     DN   GEMM      x += W_dn * act                    + per-tile sum(x^2)
//   HEAD GEMM        logits = W_head * rmsnorm(x) * gain_final
// RMSNorm never gets its own phase: the residual-writing epilogues (EMBED,
// O, DN) leave per-128-column sums of squares, and the B-operand producer
// of the next normed GEMM turns x into bf16(x * rsqrt(mean + eps) * gain)
// straight into the swizzled shared-memory tile (deterministic order, the
// numerics of rmsnorm_kernel up to fp32 summation order).
//
// Warp roles (256 threads): w0 weight producer (1-D bulk copies of the
// pre-tiled weights), w1 tcgen05.mma issuer (TMEM double buffer), w2-5
// epilogue + attention / embedding work, w6-7 B-operand producer (TMA for
// bf16 activations, computed tiles for normed x). The GEMM machinery is that
// of gemm_tc.cuh (swap-AB, stream-K over (tile, unit), deterministic
// last-arriver split-K reduction) with its counters continued across ops.
#pragma once

#include "gemm_tc.cuh"

namespace ssd {
namespace mk {

using tc::kABlock;
using tc::kABytes;
using tc::kBK;
using tc::kBM;
using tc::kKPS;

enum OpKind { OP_EMBED = 0, OP_QKV = 1, OP_ATTN = 2, OP_O = 3, OP_GU = 4, OP_DN = 5, OP_HEAD = 6, OP_NORM = 7 };

struct Op {
  int kind;
  int layer;
  const bf16* W;  // GEMM weights (pre-tiled), nullptr for EMBED / ATTN / NORM
  int N;          // GEMM output rows
  int KU;         // units per tile (K / (64 * KPS))
  int gain;       // NORM: 0 none, 1 layer-0 FFN gain, 2 final gain
};

struct LayerKV {
  bf16* kc;
  bf16* vc;
};

struct MkArgs {
  const Op* ops;
  int n_ops;
  int M;
  const FwdParams* P;
  int d, H, KVH, hd, ffn, V, S, nqkv, qd;
  float eps, scale;
  const bf16* embed;
  int embed_tiled;
  const float* gain_ffn0;   // layer-0 FFN norm gain
  const float* gain_final;  // final norm gain
  const float* rope_cos;
  const float* rope_sin;
  const LayerKV* kv;
  float* x;       // [maxM][d] residual stream
  float* sumsq;   // [d / 128][maxM] per-tile sums of squares of x
  int ld_sumsq;   // maxM
  float* qkv;     // [M][nqkv]
  bf16* attn;     // [maxM][qd]
  bf16* act;      // [maxM][ffn]
  float* logits;  // [M][V]
  float* ws;      // split-K partials [2 * grid][M][128]
  int* counters;  // per-tile arrival counters
  AttnWs aws;
  int nch;        // attention key chunks
  unsigned* bar;  // grid barrier: arrivals of this launch (monotonic, reset at exit)
  bf16* xb;       // [maxM][d] normalised GEMM input (NORM output)
  int pf_units;   // L2 look-ahead of the weight stream, in 32 KB units per CTA
  unsigned long long* trace;  // debug timeline [n_ops][grid][4] (globaltimer ns) or null
  unsigned long long* utrace; // debug per-unit timeline of CTA 0 [4 ops][64 units][4] or null
  int utrace_op[4];           // the ops traced per unit
};

constexpr int kThreads = 256;
constexpr int kSmemLimit = 226 * 1024;  // + static shared memory <= the 227 KB per-CTA limit

__host__ __device__ constexpr bool is_gemm(int k) { return k != OP_EMBED && k != OP_ATTN && k != OP_NORM; }

template <int NP, int G>
struct Cfg {
  static constexpr int kBBlock = NP * kBK * 2;
  static constexpr int kBBytes = kBBlock * kKPS;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kAttnNeed = attn_smem_floats(G, 128) * 4;
  static constexpr int kMisc = 2048;  // barriers, TMEM slot, row scales
  // The attention scratch aliases the B-operand ring when it fits: during an
  // ATTN phase no B tile is in flight (the previous GEMM is fully consumed
  // before its barrier; the next one loads B only after the ATTN barrier).
  static constexpr int kSA = (kSmemLimit - 1024 - kMisc) / kStageBytes;
  static constexpr int kSA2 = kSA > SSD_GEMM_MAX_STAGES ? SSD_GEMM_MAX_STAGES : kSA;
  static constexpr bool kAlias = kSA2 * kBBytes >= kAttnNeed;
  static constexpr int kAttnBytes = kAlias ? 0 : kAttnNeed;
  static constexpr int kStages0 = (kSmemLimit - 1024 - kAttnBytes - kMisc) / kStageBytes;
  static constexpr int kStages = kStages0 > SSD_GEMM_MAX_STAGES ? SSD_GEMM_MAX_STAGES : kStages0;
  static_assert(kStages >= 2, "persistent forward: shared memory");
  static_assert(!kAlias || kStages * kBBytes >= kAttnNeed, "attention alias");
  static constexpr int kAccCols = NP < 32 ? 32 : NP;
  static constexpr int kTmemCols = 2 * kAccCols <= 64 ? 64 : (2 * kAccCols <= 128 ? 128 : 256);
  static constexpr size_t kSmem = 1024 + size_t(kStages) * kStageBytes + kAttnBytes + kMisc;
};

// Watchdog: a wait that exceeds kWatchNs records (code, block, thread, aux)
// in host-mapped memory (readable after the context dies) and traps, so a
// protocol bug surfaces as an error instead of a hung GPU.
__device__ unsigned long long* g_mk_diag = nullptr;  // [8 + 8 * 256], host-mapped
__device__ int g_mk_progress = 0;  // SSD_B200_MK_PROGRESS=1 (debug)
// progress of role r of this CTA (debug: which op each role is in)
__device__ __forceinline__ void mk_progress(int role, int p) {
  unsigned long long* d = g_mk_diag;
  if (g_mk_progress && d)
    *reinterpret_cast<volatile unsigned long long*>(d + 8 + 8 * blockIdx.x + role) = (unsigned long long)(p + 1);
}
constexpr unsigned long long kWatchNs = 10000000000ull;
__device__ __noinline__ void mk_watch_fail(int code, int aux0, int aux1) {
  unsigned long long* d = g_mk_diag;
  if (d && atomicCAS(d, 0ull, 1ull) == 0ull) {
    d[1] = code;
    d[2] = blockIdx.x;
    d[3] = threadIdx.x;
    d[4] = aux0;
    d[5] = aux1;
    __threadfence_system();
  }
  __trap();
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ bool mbar_try(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(tc::smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
// mbarrier wait with the watchdog (code identifies the waiting role / barrier)
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t parity, int code, int aux0, int aux1) {
  if (mbar_try(b, parity)) return;
  const unsigned long long t0 = gtimer();
  while (!mbar_try(b, parity))
    if (gtimer() - t0 > kWatchNs) mk_watch_fail(code, aux0, aux1);
}

// timeline slot k of (op p, this CTA): 0 B operand ready (barrier passed),
// 1 first MMA issued, 2 epilogue done (arrival), 3 first weight copy issued
__device__ __forceinline__ void mk_trace(const MkArgs& a, int p, int k) {
  if (a.trace) a.trace[(size_t(p) * gridDim.x + blockIdx.x) * 4 + k] = gtimer();
}
// per-unit slot k of unit i (relative to the CTA's range) of op p, CTA 0:
// 0 weight copy issued, 1 B operand arrived, 2 MMA saw full, 3 epilogue got the tile
__device__ __forceinline__ void mk_utrace(const MkArgs& a, int p, int i, int k) {
  if (!a.utrace || blockIdx.x != 0 || i >= 64) return;
  for (int j = 0; j < 4; ++j)
    if (a.utrace_op[j] == p) a.utrace[(j * 64 + i) * 4 + k] = gtimer();
}

__device__ __forceinline__ unsigned ld_acquire_gpu_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Grid barrier: generation counter bar[1] (read at launch as g0; op p is
// complete when bar[1] reaches g0 + p + 1) and a self-resetting arrival
// count bar[0]. A CTA arrives for op p only after op p - 1 is complete.
__device__ __forceinline__ void grid_arrive(unsigned* bar) {
  __threadfence();
  if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
    atomicExch(&bar[0], 0u);
    __threadfence();
    atomicAdd(&bar[1], 1u);
  }
}
__device__ __forceinline__ void grid_wait(const unsigned* bar, unsigned target) {
  unsigned ns = 32;
  unsigned long long t0 = 0;
  while (int(ld_acquire_gpu_u32(&bar[1]) - target) < 0) {
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
    // a CTA that never arrives (not co-resident, or a fault) must not hang the GPU
    const unsigned long long t = gtimer();
    if (!t0) t0 = t;
    else if (t - t0 > kWatchNs) mk_watch_fail(9, int(target), int(ld_acquire_gpu_u32(&bar[1])));
  }
  __threadfence();  // invalidates L1 (data of other SMs)
}

// Named barrier of the 4 epilogue warps. The non-.aligned form: a warp may
// reach it divergent (e.g. lane 0 still leaving a grid wait).
struct NamedSync128 {
  __device__ __forceinline__ void operator()() const { asm volatile("barrier.sync 1, 128;" ::: "memory"); }
};

// Row scales of a normed B operand: rs[m] = 1 / sqrt(mean(x_m^2) + eps).
__device__ __forceinline__ float row_scale(const MkArgs& a, int m) {
  const int nt = a.d / kBM;
  float ss = 0.f;
  for (int t = 0; t < nt; ++t) ss += __ldcg(a.sumsq + size_t(t) * a.ld_sumsq + m);
  return 1.0f / sqrtf(ss / float(a.d) + a.eps);
}

// After the tile `t` (128 columns of the residual stream) of x is final for
// every token: sumsq[t][m] = sum of squares over those columns.
__device__ __forceinline__ void tile_sumsq(const MkArgs& a, int t, int tid) {
  asm volatile("barrier.sync 1, 128;" ::: "memory");
  if (tid < a.M) {
    const float4* r = reinterpret_cast<const float4*>(a.x + size_t(tid) * a.d + size_t(t) * kBM);
    float ss = 0.f;
#pragma unroll 8
    for (int i = 0; i < kBM / 4; ++i) {
      const float4 v = __ldcg(r + i);
      ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
    }
    a.sumsq[size_t(t) * a.ld_sumsq + tid] = ss;
  }
}

__device__ __forceinline__ void apply_out(const MkArgs& a, int kind, int N, int row, int tok, float v) {
  if (kind == OP_GU) {
    const float up = __shfl_xor_sync(0xffffffffu, v, 1);
    if ((row & 1) == 0 && row < N && tok < a.M)
      a.act[size_t(tok) * a.ffn + (row >> 1)] = __float2bfloat16_rn(v / (1.0f + expf(-v)) * up);
  } else if (row < N && tok < a.M) {
    if (kind == OP_QKV) a.qkv[size_t(tok) * a.nqkv + row] = v;
    else if (kind == OP_HEAD) a.logits[size_t(tok) * a.V + row] = v;
    else a.x[size_t(tok) * a.d + row] += v;  // O / DN: residual add
  }
}

template <int NP, int G>
__global__ void __launch_bounds__(kThreads, 1)
    fwd_kernel(const __grid_constant__ CUtensorMap map_attn, const __grid_constant__ CUtensorMap map_act,
               const __grid_constant__ CUtensorMap map_xb, MkArgs a) {
  using C = Cfg<NP, G>;
  constexpr int S = C::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * kABytes;
  float* sAttn = reinterpret_cast<float*>(C::kAlias ? sB : sB + S * C::kBBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + S * C::kBBytes + C::kAttnBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;   // [2]
  uint64_t* tempty = tfull + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  unsigned* s_g0 = tmem_slot + 1;
  int* s_last = reinterpret_cast<int*>(tmem_slot + 2);
  float* s_rs = reinterpret_cast<float*>(tmem_slot + 4);  // [NP] row scales (NORM)

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long P = gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) { tc::mbar_init(&full[s], 2); tc::mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { tc::mbar_init(&tfull[b], 1); tc::mbar_init(&tempty[b], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    *s_g0 = ld_acquire_gpu_u32(&a.bar[1]);  // stable until this CTA arrives for op 0
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tmem_slot)),
                 "r"(C::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const unsigned g0 = *s_g0;

  if (warp == 0) {
    // ---------------- weight producer: every GEMM of the step, back to back
    if (lane == 0) {
      uint64_t pol_w;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_w));
      uint32_t it = 0, pit = 0;                 // units loaded / L2-prefetched
      int pp = -1, pu = 0, pu1 = 0;             // prefetch cursor (op, unit range)
      const bf16* pw = nullptr;
      for (int p = 0; p < a.n_ops; ++p) {
        const Op op = a.ops[p];
        if (!is_gemm(op.kind)) continue;
        mk_progress(0, p);
        const long long U = (long long)((op.N + kBM - 1) / kBM) * op.KU;
        const int u0 = tc::unit_begin(blockIdx.x, U, P), u1 = tc::unit_begin(blockIdx.x + 1, U, P);
        for (int u = u0; u < u1; ++u, ++it) {
          const int s = int(it % S);
          // keep the HBM stream pf_units ahead of the ring (through the
          // latency-bound phases the ring alone cannot cover)
          while (pit < it + uint32_t(a.pf_units)) {
            if (pu >= pu1) {
              do { ++pp; } while (pp < a.n_ops && !is_gemm(a.ops[pp].kind));
              if (pp >= a.n_ops) break;
              const Op& q = a.ops[pp];
              const long long Uq = (long long)((q.N + kBM - 1) / kBM) * q.KU;
              pu = tc::unit_begin(blockIdx.x, Uq, P);
              pu1 = tc::unit_begin(blockIdx.x + 1, Uq, P);
              pw = q.W;
              continue;
            }
            if (pit >= it + uint32_t(S))  // units inside the ring are loaded directly
              asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pw + size_t(pu) * (kABytes / 2)),
                           "r"(uint32_t(kABytes))
                           : "memory");
            ++pu;
            ++pit;
          }
          if (it >= uint32_t(S)) mwait(&empty[s], ((it / S) - 1) & 1, 1, p, int(it));
          if (u == u0) mk_trace(a, p, 3);
          mk_utrace(a, p, u - u0, 0);
          tc::mbar_expect_tx(&full[s], kABytes);
          tc::bulk_load(sA + s * kABytes, op.W + size_t(u) * (kABytes / 2), kABytes, &full[s], pol_w);
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16(kBM, NP);
      uint32_t it = 0;
      int seg = -1;
      for (int p = 0; p < a.n_ops; ++p) {
        const Op op = a.ops[p];
        if (!is_gemm(op.kind)) continue;
        mk_progress(1, p);
        const long long U = (long long)((op.N + kBM - 1) / kBM) * op.KU;
        const int u0 = tc::unit_begin(blockIdx.x, U, P), u1 = tc::unit_begin(blockIdx.x + 1, U, P);
        int cur_tile = -1;
        for (int u = u0; u < u1; ++u, ++it) {
          const int t = u / op.KU, s = int(it % S);
          const bool first = t != cur_tile;
          if (first) {
            ++seg;
            cur_tile = t;
            if (seg >= 2) mwait(&tempty[seg & 1], ((seg >> 1) - 1) & 1, 2, p, seg);
          }
          mwait(&full[s], (it / S) & 1, 3, p, int(it));
          if (u == u0) mk_trace(a, p, 1);
          mk_utrace(a, p, u - u0, 2);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t dcol = tmem + uint32_t((seg & 1) * C::kAccCols);
#pragma unroll
          for (int h = 0; h < kKPS; ++h) {
            const uint32_t a0 = tc::smem_u32(sA + s * kABytes + h * kABlock);
            const uint32_t b0 = tc::smem_u32(sB + s * C::kBBytes + h * C::kBBlock);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              tc::mma_bf16(dcol, tc::sw128_desc(a0 + k * 32), tc::sw128_desc(b0 + k * 32), idesc,
                           (!first || h || k) ? 1u : 0u);
          }
          tc::mma_commit(&empty[s]);
          const bool last = (u + 1 == u1) || ((u + 1) / op.KU != t);
          if (last) tc::mma_commit(&tfull[seg & 1]);
        }
      }
    }
  } else if (warp >= 6) {
    // ---------------- B-operand producer: TMA of the op's bf16 input (warp 7 idles)
    if (warp == 6 && lane == 0) {
      uint32_t it = 0;
      for (int p = 0; p < a.n_ops; ++p) {
        const Op op = a.ops[p];
        if (!is_gemm(op.kind)) continue;
        const long long U = (long long)((op.N + kBM - 1) / kBM) * op.KU;
        const int u0 = tc::unit_begin(blockIdx.x, U, P), u1 = tc::unit_begin(blockIdx.x + 1, U, P);
        if (u0 == u1) continue;
        mk_progress(2, p);
        grid_wait(a.bar, g0 + unsigned(p));  // the op's input is complete
        mk_trace(a, p, 0);
        asm volatile("fence.proxy.async.global;" ::: "memory");
        const CUtensorMap* map = op.kind == OP_O ? &map_attn : (op.kind == OP_DN ? &map_act : &map_xb);
        for (int u = u0; u < u1; ++u, ++it) {
          const int s = int(it % S);
          if (it >= uint32_t(S)) mwait(&empty[s], ((it / S) - 1) & 1, 4, p, int(it));
          const int kb = (u % op.KU) * kKPS;
          uint8_t* dst = sB + s * C::kBBytes;
          mk_utrace(a, p, u - u0, 1);
          tc::mbar_expect_tx(&full[s], C::kBBytes);
#pragma unroll
          for (int h = 0; h < kKPS; ++h) tc::tma_load_2d(dst + h * C::kBBlock, map, &full[s], (kb + h) * kBK, 0);
        }
      }
    }
  } else {
    // ---------------- epilogue + non-GEMM phases (warps 2-5, 128 threads)
    const int tid = threadIdx.x - 64;
    const int q = warp & 3;
    const int rl = q * 32 + lane;
    int seg = -1;
    const AttnSmem asm_ = attn_smem_carve(sAttn, G, a.hd);
    for (int p = 0; p < a.n_ops; ++p) {
      const Op op = a.ops[p];
      if (lane == 0) mk_progress(3 + (warp - 2), p * 16 + 0);
      if (op.kind == OP_EMBED) {
        for (int m = blockIdx.x; m < a.M; m += gridDim.x) {
          const size_t tok = size_t(a.P->tokens[m]);
          for (int i = tid; i < a.d; i += 128) {
            const size_t at = a.embed_tiled ? tiled_at(tok, size_t(i), size_t(a.d) / 64) : tok * size_t(a.d) + size_t(i);
            a.x[size_t(m) * a.d + i] = __bfloat162float(a.embed[at]);
          }
          asm volatile("barrier.sync 1, 128;" ::: "memory");
          for (int t = tid; t < a.d / kBM; t += 128) {
            const float* r = a.x + size_t(m) * a.d + size_t(t) * kBM;
            float ss = 0.f;
            for (int i = 0; i < kBM; ++i) ss += r[i] * r[i];
            a.sumsq[size_t(t) * a.ld_sumsq + m] = ss;
          }
        }
      } else if (op.kind == OP_NORM) {
        // xb = bf16(x * rsqrt(mean(x^2) + eps) * gain): 16-byte chunks over the grid
        if (tid == 0) grid_wait(a.bar, g0 + unsigned(p));
        asm volatile("barrier.sync 1, 128;" ::: "memory");
        if (tid < a.M) s_rs[tid] = row_scale(a, tid);
        asm volatile("barrier.sync 1, 128;" ::: "memory");
        const float* gain = op.gain == 1 ? a.gain_ffn0 : (op.gain == 2 ? a.gain_final : nullptr);
        const int d8 = a.d / 8;
        for (int i = blockIdx.x * 128 + tid; i < a.M * d8; i += gridDim.x * 128) {
          const int m = i / d8, col = (i % d8) * 8;
          const float4* xs = reinterpret_cast<const float4*>(a.x + size_t(m) * a.d + col);
          const float4 v0 = __ldcg(xs), v1 = __ldcg(xs + 1);
          const float rs = s_rs[m];
          float f[8] = {v0.x * rs, v0.y * rs, v0.z * rs, v0.w * rs, v1.x * rs, v1.y * rs, v1.z * rs, v1.w * rs};
          if (gain) {
            const float4 g0v = __ldg(reinterpret_cast<const float4*>(gain + col));
            const float4 g1v = __ldg(reinterpret_cast<const float4*>(gain + col) + 1);
            f[0] *= g0v.x; f[1] *= g0v.y; f[2] *= g0v.z; f[3] *= g0v.w;
            f[4] *= g1v.x; f[5] *= g1v.y; f[6] *= g1v.z; f[7] *= g1v.w;
          }
          __nv_bfloat162 b2[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) b2[j] = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
          *reinterpret_cast<uint4*>(a.xb + size_t(m) * a.d + col) = *reinterpret_cast<uint4*>(b2);
        }
      } else if (op.kind == OP_ATTN) {
        if (tid == 0) grid_wait(a.bar, g0 + unsigned(p));
        asm volatile("barrier.sync 1, 128;" ::: "memory");
        __threadfence();  // drop L1 lines of qkv from earlier layers
        const int items = a.nch * a.KVH * a.M;
        const LayerKV kv = a.kv[op.layer];
        for (int w = blockIdx.x; w < items; w += gridDim.x) {
          const int chunk = w % a.nch, kvh = (w / a.nch) % a.KVH, m = w / (a.nch * a.KVH);
          attn_item<G>(a.qkv, a.P, a.M, a.rope_cos, a.rope_sin, kv.kc, kv.vc, a.S, a.H, a.KVH, a.hd, a.scale, a.attn,
                       a.aws, chunk, kvh, m, a.nch, tid, asm_, NamedSync128());
          asm volatile("barrier.sync 1, 128;" ::: "memory");
        }
      } else {
        // GEMM epilogue over this CTA's segments of the op
        const long long U = (long long)((op.N + kBM - 1) / kBM) * op.KU;
        const int u0 = tc::unit_begin(blockIdx.x, U, P), u1 = tc::unit_begin(blockIdx.x + 1, U, P);
        const bool resid = op.kind == OP_O || op.kind == OP_DN;
        int u = u0;
        while (u < u1) {
          const int t = u / op.KU;
          const int ku_lo = u % op.KU;
          const int seg_end = min(u1, (t + 1) * op.KU);
          const bool whole = ku_lo == 0 && seg_end == (t + 1) * op.KU;
          ++seg;
          const int b = seg & 1;
          mwait(&tfull[b], (seg >> 1) & 1, 5, p, seg);
          if (tid == 0) mk_utrace(a, p, u - u0, 3);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t taddr = tmem + (uint32_t(q * 32) << 16) + uint32_t(b * C::kAccCols);
          const int r = t * kBM + rl;
          float* part = a.ws + (size_t(2 * blockIdx.x + (u == u0 ? 0 : 1)) * a.M) * kBM;
#pragma unroll 1
          for (int c = 0; c < NP; c += 8) {
            uint32_t v[8];
            tc::tmem_ld8(taddr + c, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            if (c + 8 >= NP) {
              asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
              __syncwarp();
              if (lane == 0) tc::mbar_arrive(&tempty[b]);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float f = __uint_as_float(v[j]);
              if (whole) apply_out(a, op.kind, op.N, r, c + j, f);
              else if (c + j < a.M) part[size_t(c + j) * kBM + rl] = f;
            }
          }
          if (whole) {
            if (resid) tile_sumsq(a, t, tid);
          } else {
            // contributors: the CTAs with a non-empty range in [cf, cl] (with
            // more CTAs than units some ranges are empty)
            const int cf = tc::cta_of(t * op.KU, U, P), cl = tc::cta_of((t + 1) * op.KU - 1, U, P);
            int contrib = 0;
            for (int c2 = cf; c2 <= cl; ++c2) contrib += tc::unit_begin(c2 + 1, U, P) > tc::unit_begin(c2, U, P);
            __threadfence();
            asm volatile("barrier.sync 1, 128;" ::: "memory");
            if (tid == 0) *s_last = atomicAdd(&a.counters[t], 1) == contrib - 1;
            asm volatile("barrier.sync 1, 128;" ::: "memory");
            if (*s_last) {
              __threadfence();
              const int first_slot = 2 * cf + (tc::unit_begin(cf, U, P) >= t * op.KU ? 0 : 1);
              for (int t0 = 0; t0 < a.M; t0 += 8) {
                float acc[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[j] = 0.f;
                for (int c2 = cf; c2 <= cl; ++c2) {
                  if (tc::unit_begin(c2 + 1, U, P) == tc::unit_begin(c2, U, P)) continue;  // empty range
                  const int slot = c2 == cf ? first_slot : 2 * c2;
                  const float* src = a.ws + (size_t(slot) * a.M) * kBM + rl;
#pragma unroll
                  for (int j = 0; j < 8; ++j)
                    if (t0 + j < a.M) acc[j] += __ldcg(src + size_t(t0 + j) * kBM);
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) apply_out(a, op.kind, op.N, r, t0 + j, acc[j]);
              }
              if (tid == 0) a.counters[t] = 0;
              if (resid) tile_sumsq(a, t, tid);
            }
          }
          u = seg_end;
        }
      }
      // end of this CTA's part of op p: publish, then arrive (no barrier after the last op)
      if (lane == 0) mk_progress(3 + (warp - 2), p * 16 + 1);
      if (p + 1 < a.n_ops) {
        __threadfence();
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("barrier.sync 1, 128;" ::: "memory");
        if (lane == 0) mk_progress(3 + (warp - 2), p * 16 + 2);
        // arrivals must not run ahead of the previous barrier (a CTA with no
        // units in this op gets here early): one counter serves every phase
        if (tid == 0) {
          mk_trace(a, p, 2);
          grid_wait(a.bar, g0 + unsigned(p));
          mk_progress(3, p * 16 + 3);
          grid_arrive(a.bar);
          mk_progress(3, p * 16 + 4);
        }
      }
    }

  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::kTmemCols));
}

}  // namespace mk
}  // namespace ssd
