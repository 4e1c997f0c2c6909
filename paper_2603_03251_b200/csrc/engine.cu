// B200 Saguaro engine: host side (C++) of the C-ABI in include/ssd_b200.h.
//
// One process owns a (target, draft) pair on one GPU. The verifier runs on
// stream `sv`, the speculator on stream `ss`; a whole SSD round (verify
// forward + decision || extend + keys + K branch steps, then lookup) is one
// CUDA graph with a fork/join between the two streams, replayed per round
// with no host synchronisation for the FastRandom backup.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ssd_b200.h"
#include "gemm_tc.cuh"
#include "gemm_cl.cuh"
#include "attn_cl.cuh"
#include "attn_dec.cuh"
#include "tp.cuh"
#include "kernels.cuh"
#include "rowops.cuh"
#include "split.cuh"

namespace ssd {

// ------------------------------------------------------------------ errors
thread_local std::string g_last_error;

struct Fail : std::runtime_error {
  int code;
  Fail(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      throw Fail(SSD_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_) + " @" + std::to_string(__LINE__)); \
  } while (0)
#define KCHECK() CK(cudaGetLastError())

template <typename T>
T* dalloc(size_t n) {
  void* p = nullptr;
  CK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
  CK(cudaMemset(p, 0, std::max<size_t>(n, 1) * sizeof(T)));
  CK(cudaDeviceSynchronize());  // legacy-stream memset: done before a non-blocking stream touches p
  return static_cast<T*>(p);
}

// ------------------------------------------------------------------ TMA maps
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static void init_encode() {
  if (g_encode) return;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) throw Fail(SSD_CUDA, "cuTensorMapEncodeTiled unavailable");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

template <class Fn>
static Fn driver_fn(const char* name) {
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  CK(cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) throw Fail(SSD_CUDA, std::string(name) + " unavailable");
  return reinterpret_cast<Fn>(fn);
}

#define DRV(call) do { const CUresult r_ = (call); \
  if (r_ != CUDA_SUCCESS) throw Fail(SSD_CUDA, std::string(#call) + " failed: " + std::to_string(int(r_))); } while (0)

// Two green contexts on `device`: want_v SMs (rounded by the driver to its
// partition granularity) and the remaining SMs, one non-blocking stream in
// each. The streams take runtime launches and stream capture; the captured
// kernels keep their partition when the graph is launched on any stream
// (scripts/green_probe.cu, profiles/r02g_summary.md).
static void make_green_streams(int device, int want_v, CUgreenCtx ctx[2], cudaStream_t st[2], int sms[2]) {
  auto get_res = driver_fn<PFN_cuDeviceGetDevResource_v12040>("cuDeviceGetDevResource");
  auto split = driver_fn<PFN_cuDevSmResourceSplitByCount_v12040>("cuDevSmResourceSplitByCount");
  auto gen = driver_fn<PFN_cuDevResourceGenerateDesc_v12040>("cuDevResourceGenerateDesc");
  auto create = driver_fn<PFN_cuGreenCtxCreate_v12040>("cuGreenCtxCreate");
  auto mkstream = driver_fn<PFN_cuGreenCtxStreamCreate_v12050>("cuGreenCtxStreamCreate");
  CUdevResource all, part[2];
  DRV(get_res(CUdevice(device), &all, CU_DEV_RESOURCE_TYPE_SM));
  unsigned n = 1;
  DRV(split(&part[0], &n, &all, &part[1], 0, unsigned(want_v)));
  if (n != 1 || part[1].sm.smCount == 0) throw Fail(SSD_CONFIG, "green: SM split left no speculator SMs");
  for (int i = 0; i < 2; ++i) {
    CUdevResourceDesc d;
    DRV(gen(&d, &part[i], 1));
    DRV(create(&ctx[i], d, CUdevice(device), CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream s;
    DRV(mkstream(&s, ctx[i], CU_STREAM_NON_BLOCKING, 0));
    st[i] = reinterpret_cast<cudaStream_t>(s);
    sms[i] = int(part[i].sm.smCount);
  }
}

// 2-D bf16 [rows][cols] row-major, box = 64 (K) x box_rows, 128B swizzle.
static CUtensorMap make_map(const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows) {
  init_encode();
  CUtensorMap m;
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {cols * 2};
  const cuuint32_t box[2] = {uint32_t(tc::kBK), box_rows};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = g_encode(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Fail(SSD_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return m;
}

// ------------------------------------------------------------------ model
// Pre-tiled weight matrix (gemm_tc.cuh): rows padded to a multiple of 128.
struct WMat {
  bf16* w = nullptr;
  int N = 0, K = 0;
  long long off = 0;           // byte offset in the model's weight arena (forward order)
  long long bytes = 0;         // padded bytes streamed
  int swiglu = 0;              // gate/up (SwiGLU epilogue): may run one whole tile per CTA
};

static long long gemm_units(const WMat& W) {
  return (long long)((W.N + tc::kBM - 1) / tc::kBM) * (W.K / (tc::kBK * tc::kKPS));
}

// Launch with programmatic dependent launch (PDL): the kernel may start
// while its predecessor drains; it calls griddepcontrol.wait before reading
// the predecessor's output (weights are prefetched before that).
template <typename... KArgs, typename... Args>
static void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k, args...));
}

struct DevLayer {
  WMat qkv, o, gu, dn;
};

struct ActMap {
  const void* ptr;
  int K, np;
  CUtensorMap map;
};

struct Model {
  ssd_model_shape s{};
  int role = 0;  // 0 target, 1 draft
  int qd = 0, kvd = 0;
  bf16* embed = nullptr;
  int embed_tiled = 0;   // embed aliases the pre-tiled head (tied)
  WMat head;
  float* final_gain = nullptr;
  float* ffn_gain0 = nullptr;
  std::vector<DevLayer> layers;
  int S = 0;             // KV slots per kv-head: batch lanes x (main + branch region)
  int lane_S = 0;        // KV slots of one batch lane (lane l starts at l * lane_S)
  KvMap km{nullptr, 0, 0, 0};  // paged main cache (ssd_engine_set_block_table): slot of main key j
  bf16* kc = nullptr;    // [L][KVH][S][hd]
  bf16* vc = nullptr;
  float* rope_cos = nullptr;
  float* rope_sin = nullptr;
  int maxM = 0;
  int ctx_bound = 0;     // host-known bound on keys per query (attention grid)
  int branch_len = 0;
  float* attn_part = nullptr;
  int* attn_cnt = nullptr;
  float *x = nullptr, *qkv = nullptr, *q = nullptr, *logits = nullptr;
  float *dlt1 = nullptr, *dlt2 = nullptr;  // attention / MLP projections (residual deltas)
  float* logits_shard = nullptr;           // TP: this rank's vocabulary shard of the logits
  bf16 *xb = nullptr, *attn = nullptr, *act = nullptr;
  int64_t weight_bytes = 0;
  const char* arena = nullptr;  // every GEMM weight, contiguous in forward order (L2 prefetch stream)
  long long arena_bytes = 0;
  float* ws = nullptr;   // split-K partials
  size_t ws_floats = 0;
  int* counters = nullptr;
  std::vector<ActMap> amaps;
  std::vector<void*> owned;
  int gemm_ctas = 0;                        // cap on a GEMM's CTAs (0 = every SM)
  // tensor parallelism
  int tp_rank = 0, tp_size = 1;
  int V_full = 0;                           // unsharded vocabulary

  size_t kv_layer_elems() const { return size_t(s.n_kv_heads) * size_t(S) * size_t(s.head_dim); }
};

struct Engine {
  int dev = 0;
  Model T, D;
  int maxB = 0, maxK = 0;
  int nbmax = 1;            // batch lanes (run_protocol_harness batch_size)
  int hist_stride = 0;      // history capacity of one lane
  int* d_lanes = nullptr;   // device list of the lanes a batched draft serves
  // Round graphs of the last run_ssd call, reused while every baked-in
  // parameter is unchanged (ssd_graph_key): capturing two graphs of ~600
  // kernels each is host work paid per call otherwise.
  std::string ssd_graph_key;
  std::vector<cudaGraphExec_t> ssd_graphs;
  long long ssd_graph_launches = 0;  // kernels per round of the cached graphs
  int* ssd_log = nullptr;            // [2 * cap] outcomes + [cap] hits (baked into the graphs)
  int64_t ssd_log_cap = 0;
  int V = 0;
  cudaStream_t sv = nullptr, ss = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_verified = nullptr, ev_join = nullptr, ev_t0 = nullptr, ev_t1 = nullptr;
  cudaEvent_t ev_extended = nullptr;
  // colocated harness round: the verify forward waits for the speculator's
  // extend forward (SSD_B200_VERIFY_AFTER_EXTEND)
  int verify_after_extend = 0;
  LoopState* st = nullptr;
  int* hist = nullptr;
  FwdParams *P_t = nullptr, *P_x = nullptr, *P_b = nullptr, *P_s = nullptr, *P_pre = nullptr;
  float* tlogits = nullptr;   // [K+1][V]
  float* xrows = nullptr;     // extend rows [K+1][V]
  float* dmain = nullptr;     // drafted rows [K][lanes][V]
  float* brows[2] = {nullptr, nullptr};  // branch rows [K][lanes * B][V], double-buffered by round parity
  int *keys = nullptr, *bk = nullptr, *btok = nullptr, *bt = nullptr;
  double* bu = nullptr;
  double* ubuf = nullptr;
  int *plans = nullptr, *offs = nullptr;
  RowStat* rstat = nullptr;
  double* cum = nullptr;
  int* tok_scratch = nullptr;
  VI* cand = nullptr;       // row-op candidates [rows][chunks][T]
  RowChunk* rstat2 = nullptr;
  int nch = 1;              // vocabulary chunks of the row ops
  std::vector<void*> owned;
  long long launches = 0;
  int skip_mask = 0;  // profiling only (SSD_B200_SKIP): drop norms / attention
  // L2 prefetch look-ahead of the weight stream (SSD_B200_PF_MB). 16 MB:
  // colocated SSD round 9.53 -> 9.41 ms vs 32 MB (scripts/split_sms_sweep.py)
  long long pf_ahead = 16LL << 20;
  // SSD_B200_PF_MB_DRAFT: the draft model's look-ahead (-1: pf_ahead); measured
  // within noise of the shared 16 MB (0 / 4 / 32 MB: 9.09 / 9.11 / 9.17 ms per round)
  long long pf_ahead_draft = -1;
  int attn_cluster = 1;  // cluster/DSMEM attention (SSD_B200_ATTN_CL=0: global-merge kernel)
  int attn_dec = 1;      // one-CTA-per-(kv head, token) attention (attn_dec.cuh; SSD_B200_ATTN_DEC=0: chunked kernels)
  // ... and for forwards of >= this many tokens: the branch steps (M = 20:
  // colocated SSD round 9.71 -> 9.53 ms) and prefill chunks (the chunked
  // kernels append every token in every chunk CTA, quadratic in M: 8B M=128
  // forward 24.9 -> 12.3 ms) (SSD_B200_ATTN_DEC_WIDE_M)
  int attn_dec_wide_m = 20;
  long long cl_gemm_bytes = 72LL << 20;  // SSD_B200_CL_GEMM_MB: cluster split-K GEMM up to this size
  int cl_min_m = 17;                     // SSD_B200_CL_MIN_M: ... for forwards of at least this many tokens
  int cl_fused = 0;                      // SSD_B200_CL_FUSED=1: ... also with atomic split-K (fused mode)
  // Deterministic forwards (fixed fp32 summation order: partials + ordered
  // last-arriver reduction, residual adds in the norm kernel). Forced for the
  // split roles, whose speculators must compute bit-identical key tables in
  // separate processes, and for TP; SSD_B200_DETERMINISTIC=1 elsewhere.
  int deterministic = 0;
  long long small_gemm_bytes = 0;  // SSD_B200_SMALL_GEMM_MB: co-resident GEMM config up to this size (off: no gain measured)
  // ... inside the colocated SSD round, where the verifier and speculator
  // streams run at once: the 108 KB co-resident GEMM config lets their CTAs
  // share SMs. Measured (scripts/split_sms_sweep.py): round 9.41 -> 9.13 ms
  // for all GEMMs, while single-stream forwards (AR, SD) are faster with the
  // full config (8B step 3.62 vs 3.73 ms), so it applies to that loop only
  // (SSD_B200_CORUN_SMALL_GEMM_MB).
  long long corun_small_gemm_bytes = 2000LL << 20;
  // SSD_B200_CL_SMALL=1: the cluster GEMMs also take a co-resident (116 KB,
  // 2-stage) budget inside the co-running round. Off: measured slower
  // (round 9.47 vs 9.15 ms; too few stages in flight for the branch step).
  int cl_small = 0;
  // SSD_B200_CORUN_ATTN_KB: attention_dec smem cap inside the co-running round
  // (measured neutral: 80-140 KB give 9.13-9.16 vs 9.12-9.13 ms per round)
  int corun_attn_kb = 227;
  // colocated SSD: SMs given to the verifier's / speculator's GEMMs so that
  // both streams' GEMMs run at once (SSD_B200_SPLIT_SMS=<target>,<draft>;
  // 0 = all SMs, the default: no partition measured faster, profiles/)
  int split_t = 0, split_d = 0;
  // colocated SSD: true SM partition through two CUDA green contexts
  // (SSD_B200_GREEN=<verifier SMs>): the round graph's verifier branch runs
  // on green_v SMs, the speculator branch on the rest; 0 = shared SMs
  int green_v = 0, green_s = 0;
  CUgreenCtx green_ctx[2] = {nullptr, nullptr};
  cudaStream_t gsv = nullptr, gss = nullptr;
  // branch steps from green_tail on run on the whole device after the
  // verifier finished (SSD_B200_GREEN_TAIL; -1 = every step on the partition)
  int green_tail = -1;
  // partitioned round: the extend forward (+ keys, branch streams) first on
  // every SM, then verifier and branch steps on their partitions
  // (SSD_B200_EXTEND_FULL=0: the extend on the speculator partition beside
  // the verifier; measured 6.06 -> 5.95 ms per round, profiles/r02g_summary.md)
  int extend_full = 1;
  cudaEvent_t ev_tail = nullptr;
  // paged main cache (ssd_engine_set_block_table): prompt tokens of each lane
  // whose KV is already in its pages (prefix-cache hits): prefill starts there
  std::vector<int> prefill_skip;
  int page_tokens = 0;
  // split processes (split.cuh)
  int role = 0;                      // 0 colocated, 1 verifier, 2 speculator
  Inbox* inbox = nullptr;            // this process's mailbox (+ draft rows)
  std::vector<Inbox*> peers;         // mapped peer inboxes: [0] verifier, [1..G] speculators
  std::vector<void*> ipc_opened;     // handles to close
  Inbox** peers_dev = nullptr;       // device copy of `peers`
  int* send_counter = nullptr;
  int seq_base = 0;                  // advances by rounds + 2 per split run
  // In-graph round profile (ssd_profile_ssd_round): one-thread stamp kernels
  // of the captured round graph write %globaltimer at the segment boundaries
  // of both streams (event-record nodes cannot time streams of green
  // contexts: cudaEventElapsedTime rejects them, scripts/green_probe.cu).
  int prof_on = 0;
  unsigned long long* prof_ts = nullptr;  // [32] device
  unsigned long long prof_h[32] = {};
  // asynchronous pre-speculation session (ssd_prespec_begin / ssd_cache_*)
  cudaEvent_t ev_prespec = nullptr, ev_user = nullptr;
  int pre_active = 0, pre_count = 0, pre_kb = 0, pre_keys_valid = 0;
  std::vector<int> pre_keys;         // [2 * count] host copy after completion
  Mt64* pin_rng = nullptr;           // pinned staging of a caller stream
  // tensor-parallel verifier (tp.cuh)
  char* tp_region = nullptr;         // this rank's IPC-exported region
  TpLayout tp_L{};
  TpPeers tp_peers{};
  TpCtl* tp_ctl = nullptr;
  std::vector<void*> tp_opened;
};

// ----------------------------------------------------------------- helpers
// Host <-> device copies of the API calls: ordered on the engine stream `sv`
// (every kernel of a call runs on sv, or on ss forked from sv), and complete
// before returning. A plain cudaMemcpy would run on the legacy stream, which
// the non-blocking engine streams do not wait for, and a pageable H2D
// cudaMemcpy may return before its DMA lands: a kernel on sv could then read
// the previous contents (round 1's "corrupt first forward").
static void h2d(Engine& E, void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, E.sv));
  CK(cudaStreamSynchronize(E.sv));
}
static void d2h(Engine& E, void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, E.sv));
  CK(cudaStreamSynchronize(E.sv));
}

// Round-profile marks: 0 verifier start, 1 verify forward
// done, 2 verify decision done, 3 speculator start, 4 extend forward done,
// 5 keys + branch streams done, 6 + 2j branch step j forward done, 7 + 2j
// its token pick done (j < 8), 31 lookup done.
constexpr int kMarkRoundEnd = 31;
__global__ void stamp_kernel(unsigned long long* ts, int i) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  ts[i] = t;
}

static void mark(Engine& E, int i, cudaStream_t s) {
  if (!E.prof_on) return;
  stamp_kernel<<<1, 1, 0, s>>>(E.prof_ts, i);
  KCHECK();
}

static void rope_tables(const ssd_model_shape& s, std::vector<float>& cs, std::vector<float>& sn) {
  const int half = s.head_dim / 2;
  cs.assign(size_t(s.max_ctx) * half, 0.f);
  sn.assign(size_t(s.max_ctx) * half, 0.f);
  for (int p = 0; p < s.max_ctx; ++p)
    for (int i = 0; i < half; ++i) {
      const double inv = std::pow(s.rope_theta, -2.0 * i / double(s.head_dim));
      const double a = double(p) * inv;
      cs[size_t(p) * half + i] = float(std::cos(a));
      sn[size_t(p) * half + i] = float(std::sin(a));
    }
}

static uint64_t splitmix_h(uint64_t x) { return splitmix64(x); }
static float unit_value_h(uint64_t key, uint64_t idx) {
  const uint64_t h = derive_seed(key, idx);
  return float(int32_t(uint32_t(h >> 32)) >> 8) * 0x1.0p-23f;
}
static float sign_h(uint64_t key, size_t i) { return unit_value_h(key, i) < 0.f ? -1.f : 1.f; }

static GenShape gshape(const ssd_model_shape& s) { return GenShape{s.d_model, s.n_heads, s.n_kv_heads, s.head_dim, s.ffn}; }

static void gen_launch(bf16* dst, int rows, int cols, int stride, int off, const ssd_model_shape& self,
                       const ssd_model_shape& dr, const GenPair& gp, int role, int layer, int kind, int lr0 = 0,
                       int lc0 = 0) {
  gen_layer_kernel<<<148 * 8, 256>>>(dst, rows, cols, stride, off, gshape(self), gshape(dr), gp, role, layer, kind, lr0,
                                     lc0);
  KCHECK();
}

// Tensor-parallel shard shape (Megatron): heads, kv heads, FFN
// and vocabulary split over tp ranks; d_model replicated.
static ssd_model_shape tp_local(const ssd_model_shape& s, int tp) {
  ssd_model_shape l = s;
  l.n_heads /= tp;
  l.n_kv_heads /= tp;
  l.ffn /= tp;
  l.vocab /= tp;
  return l;
}

// sfull: the model's full shape; with tp_size > 1 this engine holds shard
// tp_rank (column-parallel QKV / gate-up, row-parallel O / down,
// vocabulary-parallel head, replicated embedding), generated as the exact
// blocks of the unsharded synthetic tensors.
// Forward capacity floor: prompts up to this length prefill in ONE forward
// (one weight pass per model; the bench's 128-token prompt).
constexpr int kPrefillChunk = 128;

static void build_model(Model& m, const ssd_model_shape& sfull, const ssd_model_shape& dr, const ssd_pair_params& pp,
                        int role, int branch_slots, int maxM, int tp_rank = 0, int tp_size = 1, int lanes = 1) {
  const ssd_model_shape s = tp_local(sfull, tp_size);
  m.s = s;
  m.role = role;
  m.tp_rank = tp_rank;
  m.tp_size = tp_size;
  m.V_full = sfull.vocab;
  const int d = s.d_model, hd = s.head_dim;
  m.qd = s.n_heads * hd;
  m.kvd = s.n_kv_heads * hd;
  const GenPair gp{pp.seed, pp.embed_scale, pp.shared_mlp_scale, pp.block_out_scale, pp.target_private_embed,
                   pp.target_private_head, pp.draft_gain_mix};
  auto own = [&](void* p) { m.owned.push_back(p); return p; };
  auto padded = [](int N) { return size_t((N + tc::kBM - 1) / tc::kBM) * tc::kBM; };
  auto wmat = [&](WMat& w, int N, int K) {
    if (K % (tc::kBK * tc::kKPS)) throw Fail(SSD_CONFIG, "engine: every GEMM K must be a multiple of 128");
    w.N = N;
    w.K = K;
    w.bytes = (long long)padded(N) * K * 2;
  };
  // Weight arena: every GEMM's pre-tiled weights back to back in the order a
  // forward streams them (qkv, o, gate/up, down per layer, then the LM head),
  // so "the next X bytes of the stream" is one address range (L2 prefetch
  // windows, forward()).
  m.layers.resize(size_t(s.n_layers));
  for (int l = 0; l < s.n_layers; ++l) {
    DevLayer& L = m.layers[size_t(l)];
    wmat(L.qkv, m.qd + 2 * m.kvd, d);
    wmat(L.o, d, m.qd);
    wmat(L.gu, 2 * s.ffn, d);
    L.gu.swiglu = 1;
    wmat(L.dn, d, s.ffn);
  }
  wmat(m.head, s.vocab, d);
  {
    long long at = 0;
    auto place = [&](WMat& w) { w.off = at; at += (w.bytes + 1023) / 1024 * 1024; };
    for (DevLayer& L : m.layers) { place(L.qkv); place(L.o); place(L.gu); place(L.dn); }
    place(m.head);
    m.arena_bytes = at;
    char* base = static_cast<char*>(own(dalloc<char>(size_t(at))));
    m.arena = base;
    for (DevLayer& L : m.layers)
      for (WMat* w : {&L.qkv, &L.o, &L.gu, &L.dn}) w->w = reinterpret_cast<bf16*>(base + w->off);
    m.head.w = reinterpret_cast<bf16*>(base + m.head.off);
  }
  // tables: the LM head is pre-tiled for the GEMM; a tied table is both
  if (s.tied && tp_size > 1) throw Fail(SSD_CONFIG, "engine: tensor parallelism needs an untied LM head");
  gen_table_kernel<<<148 * 8, 256>>>(m.head.w, s.vocab, d, dr.d_model, gp, s.tied ? 0 : 1, 1, tp_rank * s.vocab);
  KCHECK();
  if (s.tied) {
    m.embed = m.head.w;
    m.embed_tiled = 1;
  } else {
    m.embed = static_cast<bf16*>(own(dalloc<bf16>(size_t(sfull.vocab) * d)));
    gen_table_kernel<<<148 * 8, 256>>>(m.embed, sfull.vocab, d, dr.d_model, gp, 0, 0, 0);
    KCHECK();
    m.embed_tiled = 0;
  }
  // norm gains (host, float arithmetic identical to the oracle)
  std::vector<float> fg(static_cast<size_t>(d)), g0(static_cast<size_t>(d), 1.0f);
  const uint64_t kGS = derive_seed(pp.seed, 0xE0000004u), kGN = derive_seed(pp.seed, 0xE0000005u),
                 kGT = derive_seed(pp.seed, 0xE0000006u);
  const int ds = dr.d_model;
  const float comp = std::sqrt(float(ds) / float(d));
  for (int i = 0; i < d; ++i) {
    if (role == 1) {
      fg[size_t(i)] = pp.logit_scale * ((1.0f - pp.draft_gain_mix) * sign_h(kGS, size_t(i)) +
                                        pp.draft_gain_mix * sign_h(kGN, size_t(i)));
    } else {
      fg[size_t(i)] = pp.logit_scale * (i < ds ? sign_h(kGS, size_t(i)) : sign_h(kGT, size_t(i - ds)));
      if (i < ds) g0[size_t(i)] = comp;
    }
  }
  m.final_gain = static_cast<float*>(own(dalloc<float>(size_t(d))));
  m.ffn_gain0 = static_cast<float*>(own(dalloc<float>(size_t(d))));
  CK(cudaMemcpy(m.final_gain, fg.data(), fg.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(m.ffn_gain0, g0.data(), g0.size() * 4, cudaMemcpyHostToDevice));
  // layers: fused QKV [q; k; v], interleaved gate/up rows (2j gate, 2j+1 up)
  int64_t wb = 0;
  for (int l = 0; l < s.n_layers; ++l) {
    DevLayer& L = m.layers[size_t(l)];
    const int r = tp_rank;
    gen_launch(L.qkv.w, m.qd, d, 1, 0, sfull, dr, gp, role, l, 0, r * m.qd);
    gen_launch(L.qkv.w, m.kvd, d, 1, m.qd, sfull, dr, gp, role, l, 1, r * m.kvd);
    gen_launch(L.qkv.w, m.kvd, d, 1, m.qd + m.kvd, sfull, dr, gp, role, l, 2, r * m.kvd);
    gen_launch(L.o.w, d, m.qd, 1, 0, sfull, dr, gp, role, l, 3, 0, r * m.qd);
    gen_launch(L.gu.w, s.ffn, d, 2, 0, sfull, dr, gp, role, l, 4, r * s.ffn);
    gen_launch(L.gu.w, s.ffn, d, 2, 1, sfull, dr, gp, role, l, 5, r * s.ffn);
    gen_launch(L.dn.w, d, s.ffn, 1, 0, sfull, dr, gp, role, l, 6, 0, r * s.ffn);
    wb += int64_t(m.qd + 2 * m.kvd) * d + int64_t(d) * m.qd + int64_t(2 * s.ffn) * d + int64_t(d) * s.ffn;
  }
  wb += int64_t(s.vocab) * d;  // LM head
  m.weight_bytes = wb * 2;
  // KV cache
  m.lane_S = s.max_ctx + branch_slots;
  m.S = lanes * m.lane_S;
  m.km.lane_S = m.lane_S;
  m.kc = static_cast<bf16*>(own(dalloc<bf16>(m.kv_layer_elems() * size_t(s.n_layers))));
  m.vc = static_cast<bf16*>(own(dalloc<bf16>(m.kv_layer_elems() * size_t(s.n_layers))));
  std::vector<float> cs, sn;
  rope_tables(s, cs, sn);  // head_dim / max_ctx are not sharded
  m.rope_cos = static_cast<float*>(own(dalloc<float>(cs.size())));
  m.rope_sin = static_cast<float*>(own(dalloc<float>(sn.size())));
  CK(cudaMemcpy(m.rope_cos, cs.data(), cs.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(m.rope_sin, sn.data(), sn.size() * 4, cudaMemcpyHostToDevice));
  // activations
  m.maxM = maxM;
  m.x = static_cast<float*>(own(dalloc<float>(size_t(maxM) * d)));
  m.dlt1 = static_cast<float*>(own(dalloc<float>(size_t(maxM) * d)));
  m.dlt2 = static_cast<float*>(own(dalloc<float>(size_t(maxM) * d)));
  if (d > 8 * 4 * kNormThreads) throw Fail(SSD_CONFIG, "engine: d_model above 8192");
  m.xb = static_cast<bf16*>(own(dalloc<bf16>(size_t(maxM) * std::max(d, m.qd))));
  m.qkv = static_cast<float*>(own(dalloc<float>(size_t(maxM) * (m.qd + 2 * m.kvd))));
  m.q = static_cast<float*>(own(dalloc<float>(size_t(maxM) * m.qd)));
  m.attn = static_cast<bf16*>(own(dalloc<bf16>(size_t(maxM) * m.qd)));
  m.act = static_cast<bf16*>(own(dalloc<bf16>(size_t(maxM) * s.ffn)));
  m.logits = static_cast<float*>(own(dalloc<float>(size_t(maxM) * sfull.vocab)));
  if (tp_size > 1) m.logits_shard = static_cast<float*>(own(dalloc<float>(size_t(maxM) * s.vocab)));
  m.ws_floats = size_t(16) << 20;  // 64 MB of split-K partials
  m.ws = static_cast<float*>(own(dalloc<float>(m.ws_floats)));
  m.counters = static_cast<int*>(own(dalloc<int>(8192)));
  // split attention partials: [maxM][KVH][chunks][G][hd + 2]
  m.branch_len = branch_slots;
  m.ctx_bound = s.max_ctx;
  {
    const int G = s.n_heads / s.n_kv_heads;
    const int chunks = (s.max_ctx + branch_slots + kAttnChunk) / kAttnChunk + 1;
    m.attn_part = static_cast<float*>(own(dalloc<float>(size_t(maxM) * s.n_kv_heads * chunks * G * (hd + 2))));
    m.attn_cnt = static_cast<int*>(own(dalloc<int>(size_t(maxM) * s.n_kv_heads)));
  }
}

static int E_num_sms = 148;
static int g_swiglu_whole = 1;  // SSD_B200_SWIGLU_WHOLE=0: always stream-K
// SwiGLU needs complete sums: a tile split between CTAs ends in partials +
// a last-arriver reduction (~8 us after the last MMA at M = 20,
// scripts/ktl.py), worth about this many 32 KB units of streaming
// (SSD_B200_SWIGLU_REDUCE_UNITS)
static int g_swiglu_reduce_units = 10;

// Grid of a SwiGLU GEMM: w whole tiles per CTA (no partials) when that costs
// no more units per CTA than stream-K plus its reduction (1B gate/up, 128
// tiles: 1 tile per CTA on 148 SMs, 2 per CTA on a 92-SM partition), else
// stream-K over `cap` CTAs (0).
static int swiglu_whole_grid(int tiles, int KU, int cap) {
  if (!g_swiglu_whole || cap < 1) return 0;
  const int w = (tiles + cap - 1) / cap;
  const long long sk = ((long long)tiles * KU + cap - 1) / cap;
  return (long long)w * KU <= sk + g_swiglu_reduce_units ? (tiles + w - 1) / w : 0;
}

static void free_model(Model& m) {
  for (void* p : m.owned) cudaFree(p);
  m.owned.clear();
}

// ------------------------------------------------------------------ forward
static const CUtensorMap& act_map(Model& m, const void* X, int K, int np) {
  for (const ActMap& a : m.amaps)
    if (a.ptr == X && a.K == K && a.np == np) return a.map;
  m.amaps.push_back(ActMap{X, K, np, make_map(X, uint64_t(m.maxM), uint64_t(K), uint32_t(np))});
  return m.amaps.back().map;
}

template <int EPI, int NP, int BUDGET_KB = SSD_GEMM_SMEM_KB>
static void gemm_tc_launch(Model& m, const WMat& W, const bf16* X, int M, float* Y, int ldy, bf16* Yb, int ldyb,
                           cudaStream_t s, Prefetch pf, int atomic = 0) {
  using C = tc::Cfg<NP, BUDGET_KB>;
  const int tiles = (W.N + tc::kBM - 1) / tc::kBM;
  const int KU = W.K / (tc::kBK * tc::kKPS);
  const int units = tiles * KU;
#ifndef SSD_GEMM_CTAS_PER_SM
// One CTA per SM with <= ~110 KB of stages: the next GEMM's CTA fits beside
// it and prefetches its weights (PDL) while this one drains.
#define SSD_GEMM_CTAS_PER_SM 1
#endif
  const int cap = m.gemm_ctas > 0 ? std::min(m.gemm_ctas, E_num_sms) : E_num_sms * SSD_GEMM_CTAS_PER_SM;
  int grid = std::min(units, cap);
  if (EPI == EPI_SWIGLU) {
    const int gw = swiglu_whole_grid(tiles, KU, cap);
    if (gw > 0) grid = gw;
  }
  if (size_t(2) * grid * M * tc::kBM > m.ws_floats) throw Fail(SSD_TOO_LARGE, "gemm: split-K workspace");
  static int dbg_seq = 0;
  tc::GemmArgs g{W.w, W.N, KU, M, Y, ldy, Yb, ldyb, m.ws, m.counters, pf, dbg_seq++, EPI == EPI_SWIGLU ? 0 : atomic};
  launch_pdl(tc::gemm_tc_kernel<EPI, NP, BUDGET_KB>, dim3(grid), dim3(tc::kThreads), C::kSmem, s, act_map(m, X, W.K, NP),
             g);
}

// Cluster split-K GEMM (gemm_cl.cuh): NC clusters of CS CTAs.
template <int EPI, int NP, int CS, int BUDGET_KB = 224>
static void gemm_cl_launch(Model& m, const WMat& W, const bf16* X, int M, float* Y, int ldy, bf16* Yb, int ldyb,
                           cudaStream_t s, Prefetch pf) {
  using C = tc::ClCfg<NP, BUDGET_KB>;
  const int NC = E_num_sms / CS;
  const int KU = W.K / (tc::kBK * tc::kKPS);
  tc::GemmArgs g{W.w, W.N, KU, M, Y, ldy, Yb, ldyb, m.ws, m.counters, pf, 0, 0};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(NC * CS);
  cfg.blockDim = dim3(tc::kThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = CS;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  CK(cudaLaunchKernelEx(&cfg, tc::gemm_cl_kernel<EPI, NP, CS, BUDGET_KB>, act_map(m, X, W.K, NP), g));
}

// Cluster size minimising the units on a CTA's critical path (whole tiles
// per cluster x k-slice), ties to the smaller cluster.
static int pick_cluster(const WMat& W) {
  const int T = (W.N + tc::kBM - 1) / tc::kBM, KU = W.K / (tc::kBK * tc::kKPS);
  int best = 0, best_units = 1 << 30;
  for (int cs : {2, 4, 8}) {
    const int nc = E_num_sms / cs;
    const int units = ((T + nc - 1) / nc) * ((KU + cs - 1) / cs);
    if (units < best_units) { best_units = units; best = cs; }
  }
  return best;
}

// small = the co-resident budget (114 KB with its partial buffers): one such
// CTA fits beside a 108 KB GEMM CTA of the other stream (co-running loops).
constexpr int kClSmallBudgetKB = 116;
template <int EPI, int NP>
static void gemm_cl_dispatch(Model& m, const WMat& W, const bf16* X, int M, float* Y, int ldy, bf16* Yb, int ldyb,
                             cudaStream_t s, Prefetch pf, bool small) {
  const int cs = pick_cluster(W);
  if (small) {
    if (cs == 2) gemm_cl_launch<EPI, NP, 2, kClSmallBudgetKB>(m, W, X, M, Y, ldy, Yb, ldyb, s, pf);
    else if (cs == 4) gemm_cl_launch<EPI, NP, 4, kClSmallBudgetKB>(m, W, X, M, Y, ldy, Yb, ldyb, s, pf);
    else gemm_cl_launch<EPI, NP, 8, kClSmallBudgetKB>(m, W, X, M, Y, ldy, Yb, ldyb, s, pf);
    return;
  }
  switch (cs) {
    case 2: gemm_cl_launch<EPI, NP, 2>(m, W, X, M, Y, ldy, Yb, ldyb, s, pf); break;
    case 4: gemm_cl_launch<EPI, NP, 4>(m, W, X, M, Y, ldy, Yb, ldyb, s, pf); break;
    default: gemm_cl_launch<EPI, NP, 8>(m, W, X, M, Y, ldy, Yb, ldyb, s, pf); break;
  }
}

template <int EPI, int NP, int CS, int BUDGET_KB = 224>
static void configure_cl() {
  CK(cudaFuncSetAttribute(tc::gemm_cl_kernel<EPI, NP, CS, BUDGET_KB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          int(tc::ClCfg<NP, BUDGET_KB>::kSmem)));
  CK(cudaFuncSetAttribute(tc::gemm_cl_kernel<EPI, NP, CS, BUDGET_KB>, cudaFuncAttributePreferredSharedMemoryCarveout,
                          int(cudaSharedmemCarveoutMaxShared)));
}

template <int EPI, int NP, int BUDGET_KB = SSD_GEMM_SMEM_KB>
static void configure_gemm() {
  CK(cudaFuncSetAttribute(tc::gemm_tc_kernel<EPI, NP, BUDGET_KB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          int(tc::Cfg<NP, BUDGET_KB>::kSmem)));
  CK(cudaFuncSetAttribute(tc::gemm_tc_kernel<EPI, NP, BUDGET_KB>, cudaFuncAttributePreferredSharedMemoryCarveout,
                          int(cudaSharedmemCarveoutMaxShared)));
}

// Every kernel of the step asks for the same (max shared) L1/SMEM carveout,
// so consecutive kernels never force an SM carveout reconfiguration.
template <typename F>
static void carveout_max(F* f) {
  CK(cudaFuncSetAttribute(reinterpret_cast<const void*>(f), cudaFuncAttributePreferredSharedMemoryCarveout,
                          int(cudaSharedmemCarveoutMaxShared)));
}

// Kernel attributes are set once, outside any stream capture.
static void configure_kernels() {
  carveout_max(embed_kernel);
  carveout_max(rmsnorm_kernel);
  carveout_max(attention_kernel<1>);
  carveout_max(attention_kernel<2>);
  carveout_max(attention_kernel<4>);
  carveout_max(attention_kernel<8>);
  carveout_max(row_phase1_kernel);
  carveout_max(row_sample_kernel);
  carveout_max(row_keys_kernel);
  carveout_max(verify_stats_kernel);
  carveout_max(verify_decide_kernel);
  carveout_max(prep_chain_kernel);
  carveout_max(prep_draft_step_kernel);
  carveout_max(prep_prefill_kernel);
  carveout_max(prep_branch_kernel);
  carveout_max(branch_streams_kernel);
  carveout_max(lookup_kernel);
  carveout_max(set_spec_rows_kernel);
  carveout_max(commit_kernel);
  carveout_max(ar_commit_kernel);
  carveout_max(draw_uniforms_kernel);
  // Every remaining kernel is touched here too: setting an attribute loads it
  // now instead of at its first launch (CUDA lazy loading). Measured: with
  // lazy loading, the first forward of a tensor-parallel verifier pair
  // (spin-waiting peer-memory collectives) returned wrong logits in ~1 of 3
  // process pairs (scripts/tp_diag.py); eager-loaded, 0 of 15.
  carveout_max(tp_allreduce_kernel);
  carveout_max(tp_gather_logits_kernel);
  carveout_max(recv_spec_kernel);
  carveout_max(send_outcome_kernel);
  carveout_max(recv_outcome_kernel);
  carveout_max(send_spec_kernel);
  carveout_max(recv_peer_spec_kernel);
  carveout_max(scatter_spec_kernel);
  carveout_max(set_lane_spec_rows_kernel);
  carveout_max(draw_lane_uniforms_kernel);
  carveout_max(mt_init_kernel);
  carveout_max(mt_draw_kernel);
  carveout_max(keys_kernel);
  carveout_max(sample_rows_kernel);
  carveout_max(gen_layer_kernel);
  carveout_max(gen_table_kernel);
  carveout_max(rope_append_kernel);
  configure_gemm<EPI_STORE, 16>(); configure_gemm<EPI_SWIGLU, 16>();
  configure_gemm<EPI_STORE, 32>(); configure_gemm<EPI_SWIGLU, 32>();
  configure_gemm<EPI_STORE, 48>(); configure_gemm<EPI_SWIGLU, 48>();
  configure_gemm<EPI_STORE, 64>(); configure_gemm<EPI_SWIGLU, 64>();
  configure_gemm<EPI_STORE, 96>(); configure_gemm<EPI_SWIGLU, 96>();
  configure_gemm<EPI_STORE, 128>(); configure_gemm<EPI_SWIGLU, 128>();
  configure_gemm<EPI_STORE, 192>(); configure_gemm<EPI_SWIGLU, 192>();
  configure_gemm<EPI_STORE, 256>(); configure_gemm<EPI_SWIGLU, 256>();
  configure_gemm<EPI_STORE, 16, tc::kSmallBudgetKB>(); configure_gemm<EPI_SWIGLU, 16, tc::kSmallBudgetKB>();
  configure_cl<EPI_RESID, 32, 2>(); configure_cl<EPI_RESID, 32, 4>(); configure_cl<EPI_RESID, 32, 8>();
  configure_cl<EPI_RESID, 32, 2, kClSmallBudgetKB>(); configure_cl<EPI_RESID, 32, 4, kClSmallBudgetKB>();
  configure_cl<EPI_RESID, 32, 8, kClSmallBudgetKB>();
  configure_gemm<EPI_RESID, 16>(); configure_gemm<EPI_RESID, 32>(); configure_gemm<EPI_RESID, 48>();
  configure_gemm<EPI_RESID, 64>(); configure_gemm<EPI_RESID, 96>(); configure_gemm<EPI_RESID, 128>();
  configure_gemm<EPI_RESID, 192>(); configure_gemm<EPI_RESID, 256>();
  configure_gemm<EPI_RESID, 16, tc::kSmallBudgetKB>(); configure_gemm<EPI_RESID, 32, tc::kSmallBudgetKB>();
  configure_cl<EPI_STORE, 32, 2>(); configure_cl<EPI_STORE, 32, 4>(); configure_cl<EPI_STORE, 32, 8>();
  configure_cl<EPI_SWIGLU, 32, 2>(); configure_cl<EPI_SWIGLU, 32, 4>(); configure_cl<EPI_SWIGLU, 32, 8>();
  configure_cl<EPI_STORE, 32, 2, kClSmallBudgetKB>(); configure_cl<EPI_STORE, 32, 4, kClSmallBudgetKB>();
  configure_cl<EPI_STORE, 32, 8, kClSmallBudgetKB>(); configure_cl<EPI_SWIGLU, 32, 2, kClSmallBudgetKB>();
  configure_cl<EPI_SWIGLU, 32, 4, kClSmallBudgetKB>(); configure_cl<EPI_SWIGLU, 32, 8, kClSmallBudgetKB>();
  configure_gemm<EPI_STORE, 32, tc::kSmallBudgetKB>(); configure_gemm<EPI_SWIGLU, 32, tc::kSmallBudgetKB>();
  for (auto f : {attention_cl_kernel<1>, attention_cl_kernel<2>, attention_cl_kernel<4>, attention_cl_kernel<8>})
    carveout_max(f);
  CK(cudaFuncSetAttribute(attention_cl_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(attn_cl_smem(1, 128))));
  CK(cudaFuncSetAttribute(attention_cl_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(attn_cl_smem(2, 128))));
  CK(cudaFuncSetAttribute(attention_cl_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(attn_cl_smem(4, 128))));
  CK(cudaFuncSetAttribute(attention_cl_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(attn_cl_smem(8, 128))));
  {
    constexpr int kDecSmemMax = 227 * 1024 - int(kDecStaticSmem);
    auto dec = [&](const void* f) {
      CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, kDecSmemMax));
      CK(cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, int(cudaSharedmemCarveoutMaxShared)));
    };
#define SSD_DEC_CFG(GG, HH) dec((const void*)attention_dec_kernel<GG, HH, 1>); dec((const void*)attention_dec_kernel<GG, HH, 2>);
    SSD_DEC_CFG(1, 64) SSD_DEC_CFG(2, 64) SSD_DEC_CFG(4, 64) SSD_DEC_CFG(8, 64)
    SSD_DEC_CFG(1, 128) SSD_DEC_CFG(2, 128) SSD_DEC_CFG(4, 128) SSD_DEC_CFG(8, 128)
#undef SSD_DEC_CFG
  }
}

// Stream capture}

// Stream capture of one round / step into an executable graph. All kernel
// parameters (including the activation TMA maps) are baked in by value.
template <class F>
static cudaGraphExec_t capture_graph(cudaStream_t s, F&& body) {
  cudaGraph_t g = nullptr;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  try {
    body();
  } catch (...) {
    cudaStreamEndCapture(s, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  CK(cudaStreamEndCapture(s, &g));
  cudaGraphExec_t ge = nullptr;
  const cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
  cudaGraphDestroy(g);
  CK(e);
  return ge;
}

struct GraphSet {
  std::vector<cudaGraphExec_t> g;
  ~GraphSet() {
    for (auto x : g)
      if (x) cudaGraphExecDestroy(x);
  }
};

// atomic: split tiles accumulate into Y with fp32 atomics (gemm_tc.cuh
// GemmArgs::atomic; Y pre-zeroed for EPI_STORE). The cluster GEMM reduces
// over DSMEM and applies the epilogue once per element either way.
template <int EPI>
static void linear(Engine& E, Model& m, const WMat& W, const bf16* X, int M, float* Y, int ldy, bf16* Yb, int ldyb,
                   cudaStream_t s, Prefetch pf, int atomic = 0) {
  ++E.launches;
  // small weight matrices at branch widths (17..32 tokens): cluster split-K.
  // Measured: faster than stream-K for the 1B branch step (M = 20), slower at
  // M <= 16 (profiles/r01_summary.md), so decode / verify steps keep stream-K.
  // (M <= 16 measured slower with the cluster kernel too: 1B step 1.29 vs
  // 1.13 ms, r02 profiles/r02_summary.md)
  // (only with a fixed summation order: since split-K tiles accumulate with
  // fp32 atomics, stream-K is faster at these widths — 1B branch step 1.63 ->
  // 1.33 ms, colocated round 9.14 -> 8.49 ms, profiles/r02f_summary.md;
  // SSD_B200_CL_FUSED=1 restores the cluster GEMM there)
  const bool fused_mode = !E.deterministic && m.tp_size == 1;
  if ((!fused_mode || E.cl_fused) && W.bytes <= E.cl_gemm_bytes && M >= E.cl_min_m && M > 16 && M <= 32 &&
      m.gemm_ctas == 0) {
    gemm_cl_dispatch<EPI, 32>(m, W, X, M, Y, ldy, Yb, ldyb, s, pf, E.cl_small && W.bytes <= E.small_gemm_bytes);
    return;
  }
  // small weight matrices: the co-resident (small-budget) configuration
  if (W.bytes <= E.small_gemm_bytes && M <= 32) {
    if (M <= 16) gemm_tc_launch<EPI, 16, tc::kSmallBudgetKB>(m, W, X, M, Y, ldy, Yb, ldyb, s, pf, atomic);
    else gemm_tc_launch<EPI, 32, tc::kSmallBudgetKB>(m, W, X, M, Y, ldy, Yb, ldyb, s, pf, atomic);
    return;
  }
  if (M <= 16) gemm_tc_launch<EPI, 16>(m, W, X, M, Y, ldy, Yb, ldyb, s, pf, atomic);
  else if (M <= 32) gemm_tc_launch<EPI, 32>(m, W, X, M, Y, ldy, Yb, ldyb, s, pf, atomic);
  else if (M <= 48) gemm_tc_launch<EPI, 48>(m, W, X, M, Y, ldy, Yb, ldyb, s, pf, atomic);
  else if (M <= 64) gemm_tc_launch<EPI, 64>(m, W, X, M, Y, ldy, Yb, ldyb, s, pf, atomic);
  else if (M <= 96) gemm_tc_launch<EPI, 96>(m, W, X, M, Y, ldy, Yb, ldyb, s, pf, atomic);
  else if (M <= 128) gemm_tc_launch<EPI, 128>(m, W, X, M, Y, ldy, Yb, ldyb, s, pf, atomic);
  else if (M <= 192) gemm_tc_launch<EPI, 192>(m, W, X, M, Y, ldy, Yb, ldyb, s, pf, atomic);
  else gemm_tc_launch<EPI, 256>(m, W, X, M, Y, ldy, Yb, ldyb, s, pf, atomic);
}

// L2 prefetch cursor over the GEMM sequence of one forward: the stream
// position is (GEMM index, fraction of every stream-K range consumed), and
// each kernel extends the prefetched frontier to (start of the next GEMM it
// feeds + the look-ahead distance in bytes). Windows are baked into the
// kernels' arguments (and so into captured graphs).
struct PfCursor {
  std::vector<const WMat*> seq;  // GEMMs in forward order
  long long ahead;
  int gi = 0;        // frontier: GEMM index ...
  double frac = 0;   // ... and fraction of its ranges already prefetched
  PfCursor(const Model& m, long long a, bool head) : ahead(a) {
    cap = m.gemm_ctas > 0 ? std::min(m.gemm_ctas, E_num_sms) : E_num_sms * SSD_GEMM_CTAS_PER_SM;
    for (const DevLayer& L : m.layers)
      for (const WMat* w : {&L.qkv, &L.o, &L.gu, &L.dn}) seq.push_back(w);
    if (head) seq.push_back(&m.head);
  }
  int cap = 0;
  int parts(const WMat& w) const {
    const int tiles = (w.N + tc::kBM - 1) / tc::kBM;
    if (w.swiglu) {  // as gemm_tc_launch
      const int gw = swiglu_whole_grid(tiles, int(gemm_units(w) / tiles), cap);
      if (gw > 0) return gw;
    }
    return int(std::min<long long>(gemm_units(w), cap));
  }
  // Window up to `ahead` bytes past the start of GEMM `next` (index in seq).
  Prefetch upto(int next) {
    Prefetch p{};
    p.n = 0;
    if (ahead <= 0) return p;
    int tg = next;
    double tf = 0;
    long long left = ahead;
    while (tg < int(seq.size()) && left > 0) {
      const long long b = seq[size_t(tg)]->bytes;
      if (left >= b) { left -= b; ++tg; }
      else { tf = double(left) / double(b); left = 0; }
    }
    while ((gi < tg || (gi == tg && frac < tf)) && gi < int(seq.size()) && p.n < kPfSegs) {
      const WMat& w = *seq[size_t(gi)];
      const double end = gi < tg ? 1.0 : tf;
      p.seg[p.n++] = PfSeg{reinterpret_cast<const char*>(w.w), int(gemm_units(w)), parts(w), float(frac), float(end)};
      if (gi < tg) { ++gi; frac = 0; } else { frac = tf; }
    }
    return p;
  }
  // Window of GEMM g itself (issued after its own stream): g's bytes are
  // already loaded by g, so the frontier starts at GEMM g + 1 at the latest.
  Prefetch after(int g) {
    if (gi <= g) { gi = g + 1; frac = 0; }
    return upto(g + 1);
  }
};

// Key chunks of the split attention for the current context bound.
static int attn_chunks(const Model& m) {
  const int nk = std::min(m.ctx_bound, m.s.max_ctx + m.branch_len + 1);
  return std::max(1, (nk + kAttnChunk - 1) / kAttnChunk);
}

// Cluster attention (attn_cl.cuh): the nch key chunks of a (kv head, token)
// form one thread-block cluster; PDL as the other kernels of the step.
template <int G>
static void attn_cl_launch_g(Model& m, int nch, int M, const FwdParams* P, bf16* kc, bf16* vc, float scale,
                             cudaStream_t s, Prefetch pf) {
  const ssd_model_shape& sh = m.s;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(nch, sh.n_kv_heads, M);
  cfg.blockDim = dim3(kAttnThreads);
  cfg.dynamicSmemBytes = attn_cl_smem(G, sh.head_dim);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = nch;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  CK(cudaLaunchKernelEx(&cfg, attention_cl_kernel<G>, (const float*)m.qkv, P, M, (const float*)m.rope_cos,
                        (const float*)m.rope_sin, kc, vc, m.S, sh.n_heads, sh.n_kv_heads, sh.head_dim, scale, m.attn,
                        std::min(m.ctx_bound, m.S), pf));
}

static void attn_cl_launch(Model& m, int nch, int M, const FwdParams* P, bf16* kc, bf16* vc, float scale,
                           cudaStream_t s, Prefetch pf) {
  switch (m.s.n_heads / m.s.n_kv_heads) {
    case 1: attn_cl_launch_g<1>(m, nch, M, P, kc, vc, scale, s, pf); break;
    case 2: attn_cl_launch_g<2>(m, nch, M, P, kc, vc, scale, s, pf); break;
    case 4: attn_cl_launch_g<4>(m, nch, M, P, kc, vc, scale, s, pf); break;
    default: attn_cl_launch_g<8>(m, nch, M, P, kc, vc, scale, s, pf); break;
  }
}

// One-CTA-per-(kv head, token) attention (attn_dec.cuh). Returns false when
// the shape is not covered (head_dim other than 64 / 128, or the score rows
// do not fit shared memory): the caller then uses the chunked kernels.
template <int G, int HD, int MINB>
static void attn_dec_launch_g(Model& m, int M, const FwdParams* P, bf16* kc, bf16* vc, float scale, int kcap, int nst,
                              int appended, cudaStream_t s, Prefetch pf) {
  const ssd_model_shape& sh = m.s;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(sh.n_kv_heads, M);
  cfg.blockDim = dim3(kDecThreads);
  cfg.dynamicSmemBytes = attn_dec_smem(G, HD, kcap, nst);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, attention_dec_kernel<G, HD, MINB>, (const float*)m.qkv, P, M, (const float*)m.rope_cos,
                        (const float*)m.rope_sin, kc, vc, m.S, sh.n_heads, sh.n_kv_heads, scale, m.attn, kcap, nst,
                        appended, pf, m.km));
}

static int g_attn_stage = 1;  // SSD_B200_ATTN_STAGE=0: never stage KV rows in shared memory
// shared-memory cap of an attention_dec CTA (its staged rows), KB; lowered
// inside the co-running SSD round when SSD_B200_CORUN_ATTN_KB is set
static int g_attn_smem_cap_kb = 227;

template <int G, int HD>
static void attn_dec_pick(Model& m, int M, const FwdParams* P, bf16* kc, bf16* vc, float scale, int kcap,
                          cudaStream_t s, Prefetch pf) {
  constexpr size_t kSmemMax = 227 * 1024 - kDecStaticSmem;  // the kernel's static token tables
  if (size_t(M) * m.s.n_kv_heads > size_t(2 * E_num_sms)) {
    // wide forward (prefill chunk): append every row first, then attend from the cache
    launch_pdl(rope_append_kernel, dim3(M, m.s.n_kv_heads), dim3(128), 0, s, (const float*)m.qkv, P,
               (const float*)m.rope_cos, (const float*)m.rope_sin, kc, vc, m.S, m.s.n_heads, m.s.n_kv_heads, HD);
    attn_dec_launch_g<G, HD, 2>(m, M, P, kc, vc, scale, kcap, 0, 1, s, pf);
    return;
  }
  if (size_t(M) * m.s.n_kv_heads <= size_t(E_num_sms) && g_attn_stage) {
    // one CTA per SM: stage as many main KV rows as shared memory holds
    const size_t cap = std::min(kSmemMax, size_t(g_attn_smem_cap_kb) * 1024);
    const size_t base = attn_dec_smem(G, HD, kcap, 0);
    const size_t room = cap > base ? cap - base : 0;
    const int nst = int(std::min<size_t>(size_t(kcap), room / (size_t(4) * HD)));
    attn_dec_launch_g<G, HD, 1>(m, M, P, kc, vc, scale, kcap, nst, 0, s, pf);
  } else {
    attn_dec_launch_g<G, HD, 2>(m, M, P, kc, vc, scale, kcap, 0, 0, s, pf);  // two CTAs per SM, rows from L2
  }
}

static bool attn_dec_launch(Model& m, int M, const FwdParams* P, bf16* kc, bf16* vc, float scale, cudaStream_t s,
                            Prefetch pf) {
  const int hd = m.s.head_dim, G = m.s.n_heads / m.s.n_kv_heads;
  const int kcap = (std::min(m.ctx_bound, m.s.max_ctx + m.branch_len + 1) + 3) & ~3;
  if ((hd != 64 && hd != 128) || attn_dec_smem(G, hd, kcap, 0) > size_t(100 * 1024)) return false;
#define SSD_DEC(GG, HH) attn_dec_pick<GG, HH>(m, M, P, kc, vc, scale, kcap, s, pf)
  if (hd == 64) {
    if (G == 1) SSD_DEC(1, 64); else if (G == 2) SSD_DEC(2, 64); else if (G == 4) SSD_DEC(4, 64); else SSD_DEC(8, 64);
  } else {
    if (G == 1) SSD_DEC(1, 128); else if (G == 2) SSD_DEC(2, 128); else if (G == 4) SSD_DEC(4, 128); else SSD_DEC(8, 128);
  }
#undef SSD_DEC
  return true;
}

// Row-parallel projection sum over the TP ranks (tp.cuh), in place.
static void tp_allreduce(Engine& E, Model& m, float* buf, int M, cudaStream_t s) {
  if (!E.tp_peers.region[0]) throw Fail(SSD_CONFIG, "tensor parallel: peers not connected (ssd_tp_connect)");
  tp_allreduce_kernel<<<64, 256, 0, s>>>(buf, M, E.tp_L, E.tp_peers, m.tp_rank, E.tp_ctl, E.st);
  KCHECK();
  ++E.launches;
}

// Attention of layer l over this forward's M tokens (RoPE + KV append fused),
// kernel chosen by shape: attention_dec while the (kv head, token) CTAs fit
// (decode, verify, extend, branch steps), else the chunked kernels.
static void attend(Engine& E, Model& m, const FwdParams* P, int M, int l, cudaStream_t s, Prefetch pf) {
  const ssd_model_shape& sh = m.s;
  const int H = sh.n_heads, KVH = sh.n_kv_heads, hd = sh.head_dim;
  bf16* kc = m.kc + size_t(l) * m.kv_layer_elems();
  bf16* vc = m.vc + size_t(l) * m.kv_layer_elems();
  const float scale = 1.0f / std::sqrt(float(hd));
  const int nch = attn_chunks(m);
  const AttnWs aws{m.attn_part, m.attn_cnt};
  ++E.launches;
  if (m.km.tab) {  // a paged main cache: attention_dec (the kernel that reads through the block table)
    if (!attn_dec_launch(m, M, P, kc, vc, scale, s, pf))
      throw Fail(SSD_CONFIG, "paged KV: attention shape not covered by attention_dec");
    return;
  }
  if (E.attn_dec && (size_t(M) * KVH <= size_t(E_num_sms) || M >= E.attn_dec_wide_m) &&
      attn_dec_launch(m, M, P, kc, vc, scale, s, pf)) {
    // one CTA per (kv head, token) while they fit one wave (decode, verify,
    // extend) and for the branch steps / prefill chunks (measured faster:
    // profiles/r01c_summary.md)
  } else if (nch <= kAttnClMaxChunks && E.attn_cluster) {
    attn_cl_launch(m, nch, M, P, kc, vc, scale, s, pf);
  } else {
    auto k = H / KVH == 1 ? attention_kernel<1> : (H / KVH == 2 ? attention_kernel<2> : (H / KVH == 4 ? attention_kernel<4> : attention_kernel<8>));
    launch_pdl(k, dim3(nch, KVH, M), dim3(kAttnThreads), 0, s, (const float*)m.qkv, P, M, (const float*)m.rope_cos,
               (const float*)m.rope_sin, kc, vc, m.S, H, KVH, hd, scale, m.attn, aws, pf);
  }
}

// One forward step of `m` over the M tokens described by P. Logits of all M
// rows go to `logits` ([M][V]) when non-null. Every kernel is launched with
// PDL so each GEMM streams its weights while its predecessor finishes.
static void forward(Engine& E, Model& m, const FwdParams* P, int M, float* logits, cudaStream_t s) {
  if (M > m.maxM) throw Fail(SSD_CONFIG, "forward: M exceeds capacity");
  const ssd_model_shape& sh = m.s;
  const int d = sh.d_model, F = sh.ffn;
  const int nqkv = m.qd + 2 * m.kvd;
  PfCursor pf(m, (m.role == 1 && E.pf_ahead_draft >= 0) ? E.pf_ahead_draft : E.pf_ahead, logits != nullptr);
  launch_pdl(embed_kernel, dim3(M), dim3(256), 0, s, (const bf16*)m.embed, d, m.embed_tiled, P, m.x, pf.upto(0));
  ++E.launches;
  // E.skip_mask: profiling only (results are wrong): 1 = norms, 2 = attention
  const bool do_norm = !(E.skip_mask & 1), do_attn = !(E.skip_mask & 2);
  const int fused = (!E.deterministic && m.tp_size == 1) ? 1 : 0;
  for (int l = 0; l < sh.n_layers; ++l) {
    const DevLayer& L = m.layers[size_t(l)];
    // fused residual: the O / down projections add into x
    // in their epilogues (EPI_RESID); otherwise (deterministic / TP engines)
    // they store deltas that the next norm adds. xb = norm(x); the fused
    // path also clears the QKV output for its atomic split-K accumulation.
    if (do_norm)
      launch_pdl(rmsnorm_kernel, dim3(M), dim3(kNormThreads), 0, s, m.x,
                 (const float*)(l > 0 && !fused ? m.dlt2 : nullptr), d, (const float*)nullptr, sh.norm_eps, m.xb,
                 pf.upto(4 * l), fused ? m.qkv : nullptr, nqkv);
    linear<EPI_STORE>(E, m, L.qkv, m.xb, M, m.qkv, nqkv, nullptr, 0, s, pf.after(4 * l), fused);
    if (do_attn) attend(E, m, P, M, l, s, pf.upto(4 * l + 1));
    if (fused) {
      linear<EPI_RESID>(E, m, L.o, m.attn, M, m.x, d, nullptr, 0, s, pf.after(4 * l + 1), 1);
    } else {
      linear<EPI_STORE>(E, m, L.o, m.attn, M, m.dlt1, d, nullptr, 0, s, pf.after(4 * l + 1));
      if (m.tp_size > 1) tp_allreduce(E, m, m.dlt1, M, s);  // row-parallel O: sum the shards
    }
    // (x += attention projection); xb = norm(x) * g
    if (do_norm)
      launch_pdl(rmsnorm_kernel, dim3(M), dim3(kNormThreads), 0, s, m.x, (const float*)(fused ? nullptr : m.dlt1), d,
                 (const float*)(l == 0 ? m.ffn_gain0 : nullptr), sh.norm_eps, m.xb, pf.upto(4 * l + 2),
                 (float*)nullptr, 0);
    linear<EPI_SWIGLU>(E, m, L.gu, m.xb, M, nullptr, 0, m.act, F, s, pf.after(4 * l + 2));
    if (fused) {
      linear<EPI_RESID>(E, m, L.dn, m.act, M, m.x, d, nullptr, 0, s, pf.after(4 * l + 3), 1);
    } else {
      linear<EPI_STORE>(E, m, L.dn, m.act, M, m.dlt2, d, nullptr, 0, s, pf.after(4 * l + 3));
      if (m.tp_size > 1) tp_allreduce(E, m, m.dlt2, M, s);  // row-parallel down projection
    }
    E.launches += 2;
  }
  if (logits) {
    launch_pdl(rmsnorm_kernel, dim3(M), dim3(kNormThreads), 0, s, m.x, (const float*)(fused ? nullptr : m.dlt2), d,
               (const float*)m.final_gain, sh.norm_eps, m.xb, pf.upto(4 * sh.n_layers), (float*)nullptr, 0);
    if (m.tp_size > 1) {  // vocabulary-parallel head: local shard, then all-gather the rows
      linear<EPI_STORE>(E, m, m.head, m.xb, M, m.logits_shard, sh.vocab, nullptr, 0, s, pf.after(4 * sh.n_layers));
      tp_gather_logits_kernel<<<64, 256, 0, s>>>(m.logits_shard, M, sh.vocab, logits, E.tp_L, E.tp_peers, m.tp_rank,
                                                 E.tp_ctl, E.st);
      KCHECK();
      E.launches += 2;
    } else {
      linear<EPI_STORE>(E, m, m.head, m.xb, M, logits, sh.vocab, nullptr, 0, s, pf.after(4 * sh.n_layers));
      ++E.launches;
    }
  }
}

// Prefill hist[0, n) into model m (chunks of maxM). Logits of the last
// token to `last_logits` when non-null.
static void prefill(Engine& E, Model& m, int n, float* last_logits, cudaStream_t s, int lane = 0) {
  const int chunk = std::min(m.maxM, kMaxM);
  // a lane whose prompt prefix is mapped from the prefix cache (paged KV)
  // starts after it; the last token is always computed when its logits are needed
  int lo0 = 0;
  if (m.km.tab && size_t(lane) < E.prefill_skip.size())
    lo0 = std::max(0, std::min(E.prefill_skip[size_t(lane)], last_logits ? n - 1 : n));
  for (int lo = lo0; lo < n; lo += chunk) {
    const int M = std::min(chunk, n - lo);
    prep_prefill_kernel<<<1, kMaxM, 0, s>>>(E.hist + size_t(lane) * E.hist_stride, E.P_pre, lo, M, lane * m.lane_S,
                                            m.km);
    KCHECK();
    const bool last = lo + M >= n;
    forward(E, m, E.P_pre, M, (last && last_logits) ? m.logits : nullptr, s);
    if (last && last_logits)
      CK(cudaMemcpyAsync(last_logits, m.logits + size_t(M - 1) * m.V_full, size_t(m.V_full) * 4,
                         cudaMemcpyDeviceToDevice, s));
  }
}

// A split process holds only its own model.
static void need(const Model& m, const char* what) {
  if (m.layers.empty()) throw Fail(SSD_CONFIG, std::string(what) + ": model not materialised in this engine's role");
}

static DScheme dscheme(const ssd_scheme& s) {
  return DScheme{s.kind == 1 ? 1 : 0, s.fan_out, s.temperature, s.downweight};
}

static void check_scheme(const ssd_scheme& s, int V) {
  if (s.temperature < 0.0 || !std::isfinite(s.temperature)) throw Fail(SSD_ERROR, "apply_scheme: temperature must be > 0");
  if (s.kind == 1) {
    if (s.fan_out < 1 || s.fan_out > V) throw Fail(SSD_ERROR, "apply_scheme: fan_out out of range");
    if (s.fan_out > kMaxTopF) throw Fail(SSD_TOO_LARGE, "apply_scheme: fan_out above the engine's top-k capacity");
    if (!(s.downweight >= 0.0) || !(s.downweight <= 1.0)) throw Fail(SSD_ERROR, "apply_scheme: downweight must be in [0, 1]");
  }
}

// ------------------------------------------------------------------ state
static void reset_state(Engine& E, int K, int n, int64_t rounds, uint64_t dseed, uint64_t vseed, const ssd_sim_config* c,
                        cudaStream_t s, int lane = 0) {
  LoopState h;
  std::memset(&h, 0, sizeof(h));
  h.n = n;
  h.K = K;
  h.Kb = K;
  h.rounds = int(rounds);
  h.backup_kind = c ? c->backup_kind : 1;
  h.primary_time = c ? c->primary_time : 0.0;
  h.backup_time = c ? (c->backup_kind == 0 ? c->primary_time : c->backup_time) : 0.0;
  h.seq_base = E.seq_base;
  CK(cudaMemcpyAsync(E.st + lane, &h, offsetof(LoopState, vrng), cudaMemcpyHostToDevice, s));
  mt_init_kernel<<<1, 32, 0, s>>>(&E.st[lane].vrng, vseed);
  mt_init_kernel<<<1, 32, 0, s>>>(&E.st[lane].drng, dseed);
  KCHECK();
}

static LoopState read_state(Engine& E, int lane = 0) {
  LoopState h;
  d2h(E, &h, E.st + lane, offsetof(LoopState, vrng));
  return h;
}

static void raise_device_error(const LoopState& h) {
  if (h.error == 1) throw Fail(SSD_ERROR, "verify: drafted token has zero draft probability");
  if (h.error == 3) throw Fail(SSD_DEGENERATE_RESIDUAL, "residual: zero positive mass (draft equals target)");
  if (h.error == 11) throw Fail(SSD_PROTOCOL_VIOLATION, "protocol: cache missed the overlap window");
  if (h.error) throw Fail(SSD_ERROR, "device error " + std::to_string(h.error));
}

// Draw one token per row (greedy argmax or the scheme's law with the row's
// uniform u[r * u_stride]) into out[r * out_stride]: two-phase row op.
static void row_pick(Engine& E, const float* base, size_t stride, int rows, int V, const DScheme& ds, const double* u,
                     int u_stride, int* out, int out_stride, cudaStream_t s) {
  int T = 1;
  if (ds.saguaro) T = ds.tau == 0.0 ? (ds.C == 0.0 ? ds.fan_out + 1 : 1) : ds.fan_out;
  row_phase1_kernel<<<dim3(E.nch, rows), kRowThreads, 0, s>>>(base, stride, V, T, ds.tau, E.cand, E.rstat2);
  row_sample_kernel<<<rows, kRowThreads, 0, s>>>(base, stride, V, E.nch, T, ds, E.cand, E.rstat2, u, u_stride, out,
                                                 out_stride);
  KCHECK();
  E.launches += 2;
}

// Cache keys from K+1 contiguous logit rows (cache.cpp:249-270).
// Batch lanes: nl lanes of nrows rows each; lane l's branches at l * bper.
static void row_keys(Engine& E, const float* rows, int nrows, int V, int max_f, const LoopState* st, const int* excl,
                     int n_excl, cudaStream_t s, int nl = 1, int bper = 0) {
  const int T = std::min(max_f + 1, kMaxTopF + 1);
  row_phase1_kernel<<<dim3(E.nch, nrows * nl), kRowThreads, 0, s>>>(rows, size_t(V), V, T, 0.0, E.cand, E.rstat2);
  row_keys_kernel<<<nrows * nl, kRowThreads, 0, s>>>(E.nch, T, E.cand, E.plans, E.offs, st, excl, n_excl, max_f, E.keys,
                                                     E.bk, E.btok, nrows, bper);
  KCHECK();
  E.launches += 2;
}

// K sequential draft steps from the current history (specdec::draft,
// specdec.cpp:8-25): rows into dmain, tokens into st->spec.
static void draft_steps(Engine& E, int K, const ssd_scheme& sc, int origin, int src, cudaStream_t s) {
  const DScheme ds = dscheme(sc);
  for (int i = 0; i < K; ++i) {
    prep_draft_step_kernel<<<1, 32, 0, s>>>(E.st, E.hist, E.P_s, i, nullptr, 1, 0, 0, E.D.km);
    forward(E, E.D, E.P_s, 1, E.dmain + size_t(i) * E.V, s);
    draw_uniforms_kernel<<<1, 32, 0, s>>>(&E.st->drng, E.ubuf, 1);
    row_pick(E, E.dmain + size_t(i) * E.V, size_t(E.V), 1, E.V, ds, E.ubuf, 1, &E.st->spec[i], 1, s);
    KCHECK();
    E.launches += 2;
  }
  set_spec_rows_kernel<<<1, 32, 0, s>>>(E.st, E.dmain, E.V, origin, src);
  KCHECK();
  ++E.launches;
}

// specdec::draft for the nl batch lanes listed in E.d_lanes, batched: one
// M = nl draft forward per step, each lane drawing from its own stream
// (the initial drafts and the JIT backups of run_protocol_harness at batch
// size > 1, sim.cpp:524-526, 565-570). Rows: dmain[(i * nbmax + m) * V].
static void draft_lanes(Engine& E, int K, const ssd_scheme& sc, int origin, int src, int nl, cudaStream_t s) {
  const DScheme ds = dscheme(sc);
  for (int i = 0; i < K; ++i) {
    prep_draft_step_kernel<<<1, 32, 0, s>>>(E.st, E.hist, E.P_s, i, E.d_lanes, nl, E.hist_stride, E.D.lane_S, E.D.km);
    float* rows = E.dmain + size_t(i) * E.nbmax * E.V;
    forward(E, E.D, E.P_s, nl, rows, s);
    draw_lane_uniforms_kernel<<<1, 32, 0, s>>>(E.st, E.d_lanes, nl, E.ubuf);
    row_pick(E, rows, size_t(E.V), nl, E.V, ds, E.ubuf, 1, E.tok_scratch, 1, s);
    scatter_spec_kernel<<<1, 32, 0, s>>>(E.st, E.d_lanes, nl, i, E.tok_scratch);
    KCHECK();
    E.launches += 3;
  }
  set_lane_spec_rows_kernel<<<1, 32, 0, s>>>(E.st, E.d_lanes, nl, E.dmain, E.nbmax, E.V, origin, src);
  KCHECK();
  ++E.launches;
}

// Colocated SSD round on disjoint SM sets (green contexts): the verifier
// branch on `want_v` SMs, the speculator branch on the rest. The round graph
// is re-captured at the next run.
static void drop_green(Engine& E) {
  for (cudaStream_t st : {E.gsv, E.gss})
    if (st) cudaStreamDestroy(st);
  if (E.green_ctx[0] || E.green_ctx[1]) {
    auto destroy = driver_fn<PFN_cuGreenCtxDestroy_v12040>("cuGreenCtxDestroy");
    for (CUgreenCtx& g : E.green_ctx) {
      if (g) destroy(g);
      g = nullptr;
    }
  }
  E.gsv = E.gss = nullptr;
  E.green_v = E.green_s = 0;
  E.ssd_graph_key.clear();
}

static void set_green(Engine& E, int want_v) {
  drop_green(E);
  if (want_v <= 0) return;
  if (E.role != SSD_ROLE_COLOCATED || E.T.tp_size > 1)
    throw Fail(SSD_CONFIG, "sm_partition: colocated single-GPU engines only");
  if (want_v >= E_num_sms) throw Fail(SSD_CONFIG, "sm_partition: verifier SMs must leave SMs for the speculator");
  cudaStream_t st[2];
  int sms[2];
  make_green_streams(E.dev, want_v, E.green_ctx, st, sms);
  E.gsv = st[0];
  E.gss = st[1];
  E.green_v = sms[0];
  E.green_s = sms[1];
}

// Verification of st->spec against the target (verify forward M = K+1,
// then the decision kernels).
static void verify_round(Engine& E, int K, const ssd_scheme& ts, const ssd_scheme& ds, double scale, int use_draft_stream,
                         cudaStream_t s, int nl = 1) {
  prep_chain_kernel<<<nl, 32, 0, s>>>(E.st, E.hist, E.P_t, K + 1, E.hist_stride, E.T.lane_S, E.T.km);
  KCHECK();
  forward(E, E.T, E.P_t, nl * (K + 1), E.tlogits, s);
  mark(E, 1, s);
  verify_stats_kernel<<<dim3(2 * K + 1, nl), kSampleThreads, 0, s>>>(E.tlogits, E.st, E.V, dscheme(ts), dscheme(ds),
                                                                       E.rstat);
  verify_decide_kernel<<<nl, kSampleThreads, 0, s>>>(E.tlogits, E.st, E.hist, E.V, dscheme(ts), dscheme(ds), scale, E.rstat,
                                                     use_draft_stream, E.hist_stride);
  KCHECK();
  mark(E, 2, s);
  E.launches += 3;
}

// Pre-speculation for the in-flight speculation (cache::build_cache,
// cache.cpp:232-277, batched): extend over [last, s_1..s_K], candidate keys,
// per-branch streams, K branch decode steps at M = B.
// Branch sharding: every speculator computes the full key
// table and the per-branch streams, and decodes branches [lo, lo + Bl).
// Batch lanes (nl > 1, no sharding: lo = 0, Bl = B): every lane's extend
// rides one M = nl (K+1) forward, its B branches are rows [l B, (l+1) B) of
// one M = nl B branch step.
// before_streams (sequential run_ssd semantics, sim.cpp:159-204): the
// branch streams' base is drawn from the sequence stream AFTER verify's
// draws, so the branch half waits for the verifier. Kb: continuation length
// of each entry (build_cache's next_lookahead; K in the loops).
static void prespeculate(Engine& E, int K, int B, int lo, int Bl, int max_f, const ssd_scheme& sc, int parity,
                         cudaStream_t s, int nl = 1, cudaEvent_t before_streams = nullptr, int Kb = -1,
                         cudaEvent_t after_extend = nullptr, int jb = -1, int je = -1) {
  if (Kb < 0) Kb = K;
  if (je < 0) je = Kb;
  if (nl > 1) Bl = nl * B;
  const DScheme ds = dscheme(sc);
  float* rows = E.brows[parity];
  const bool sampled = sc.temperature > 0.0;
  // jb >= 0: branch steps [jb, je) only (the green tail: the last steps run
  // on the whole device once the verifier is done); else everything up to je
  auto steps = [&](int j0, int j1) {
    for (int j = j0; j < j1 && Bl > 0; ++j) {
      prep_branch_kernel<<<(Bl + 127) / 128, 128, 0, s>>>(E.st, E.bk + lo, E.btok + lo, E.bt, E.P_b, Bl, j,
                                                           E.D.s.max_ctx, nl > 1 ? B : 0, E.D.lane_S);
      float* out = rows + size_t(j) * Bl * E.V;
      forward(E, E.D, E.P_b, Bl, out, s);
      if (j < 8) mark(E, 6 + 2 * j, s);
      row_pick(E, out, size_t(E.V), Bl, E.V, ds, sampled ? E.bu + size_t(lo) * Kb + j : nullptr, Kb, E.bt + j, Kb, s);
      KCHECK();
      if (j < 8) mark(E, 7 + 2 * j, s);
      E.launches += 1;
    }
  };
  if (jb >= 0) {
    steps(jb, je);
    return;
  }
  prep_chain_kernel<<<nl, 32, 0, s>>>(E.st, E.hist, E.P_x, K + 1, E.hist_stride, E.D.lane_S, E.D.km);
  KCHECK();
  forward(E, E.D, E.P_x, nl * (K + 1), E.xrows, s);
  if (after_extend) CK(cudaEventRecord(after_extend, s));
  mark(E, 4, s);
  row_keys(E, E.xrows, K + 1, E.V, max_f, E.st, nullptr, K, s, nl, B);
  if (before_streams) CK(cudaStreamWaitEvent(s, before_streams, 0));
  branch_streams_kernel<<<nl, 128, 0, s>>>(E.st, B, E.bu, sampled ? 1 : 0);
  KCHECK();
  mark(E, 5, s);
  E.launches += 2;
  steps(0, je);
}

static void upload_plans(Engine& E, const ssd_plan& p, const ssd_plan& b, int K, int& B, int& max_f) {
  std::vector<int> fan(size_t(2 * (K + 1))), off(size_t(2 * (K + 1)));
  B = 0;
  max_f = 1;
  for (int r = 0; r < 2; ++r) {
    const ssd_plan& pl = r == 0 ? p : b;
    if (pl.lookahead != K) throw Fail(SSD_ERROR, "build_cache: plan length does not match speculation");
    int tot = 0;
    for (int k = 0; k <= K; ++k) {
      const int f = pl.fan_out[k];
      if (f < 0) throw Fail(SSD_ERROR, "plan: negative fan-out");
      if (f > kMaxTopF - 1) throw Fail(SSD_TOO_LARGE, "plan: fan-out above the engine's top-k capacity");
      if (f > (k < K ? E.V - 1 : E.V)) throw Fail(SSD_ERROR, "plan: fan-out exceeds candidate count");
      fan[size_t(r * (K + 1) + k)] = f;
      off[size_t(r * (K + 1) + k)] = tot;
      tot += f;
      max_f = std::max(max_f, f);
    }
    B = std::max(B, tot);
  }
  if (B > E.maxB) throw Fail(SSD_TOO_LARGE, "plan: budget exceeds the engine's branch capacity");
  B = std::max(B, 1);
  h2d(E, E.plans, fan.data(), fan.size() * 4);
  h2d(E, E.offs, off.data(), off.size() * 4);
}

static void set_history(Engine& E, const int32_t* prompt, int n, int max_ctx_needed, int lanes = 1) {
  if (n < 1) throw Fail(SSD_ERROR, "prompt must hold at least one token");
  const int cap = std::min(E.T.s.max_ctx, E.D.s.max_ctx);
  if (max_ctx_needed > cap) throw Fail(SSD_TOO_LARGE, "context exceeds max_ctx");
  E.T.ctx_bound = E.D.ctx_bound = max_ctx_needed + 2 * E.maxK + 2;
  for (int i = 0; i < n; ++i)
    if (prompt[i] < 0 || prompt[i] >= E.V) throw Fail(SSD_ERROR, "context_index: token out of range");
  for (int l = 0; l < lanes; ++l)
    h2d(E, E.hist + size_t(l) * E.hist_stride, prompt, size_t(n) * 4);
}

// RunStats counters summed over batch lanes (sim.cpp:548-586 counts every
// sequence); the virtual clock is shared.
static LoopState sum_lanes(const std::vector<LoopState>& v) {
  LoopState h = v[0];
  for (size_t l = 1; l < v.size(); ++l) {
    const LoopState& o = v[l];
    h.tokens += o.tokens; h.p_lookups += o.p_lookups; h.p_hits += o.p_hits; h.b_lookups += o.b_lookups;
    h.b_hits += o.b_hits; h.hit_rounds += o.hit_rounds; h.miss_rounds += o.miss_rounds;
    h.initial_rounds += o.initial_rounds; h.hit_round_tokens += o.hit_round_tokens;
    h.miss_round_tokens += o.miss_round_tokens; h.accepted_sum += o.accepted_sum;
    if (o.error && !h.error) h.error = o.error;
  }
  return h;
}

static void fill_stats(const LoopState& h, int64_t rounds, float ms, long long launches, ssd_run_stats* out) {
  if (!out) return;
  out->rounds = rounds;
  out->tokens = h.tokens;
  out->virtual_time = h.clock;
  out->primary_origin_lookups = h.p_lookups;
  out->primary_origin_hits = h.p_hits;
  out->backup_origin_lookups = h.b_lookups;
  out->backup_origin_hits = h.b_hits;
  out->hit_rounds = h.hit_rounds;
  out->miss_rounds = h.miss_rounds;
  out->initial_rounds = h.initial_rounds;
  out->hit_round_tokens = h.hit_round_tokens;
  out->miss_round_tokens = h.miss_round_tokens;
  out->accepted_sum = h.accepted_sum;
  out->device_ms = ms;
  out->kernel_launches = launches;
}

static void copy_out(Engine& E, int n0, int n, int32_t* out, int64_t cap, int64_t* out_len, int lane = 0) {
  const int64_t len = n - n0;
  if (out_len) *out_len = len;
  if (out && len > 0)
    d2h(E, out, E.hist + size_t(lane) * E.hist_stride + n0, size_t(std::min<int64_t>(len, cap)) * 4);
}

static void validate_cfg(Engine& E, const ssd_sim_config* c) {
  if (!c) throw Fail(SSD_CONFIG, "sim: config required");
  if (c->lookahead < 1) throw Fail(SSD_ERROR, "sim: lookahead must be >= 1");
  if (c->lookahead > E.maxK) throw Fail(SSD_TOO_LARGE, "sim: lookahead exceeds the engine's capacity");
  if (c->rounds < 1) throw Fail(SSD_ERROR, "sim: rounds must be >= 1");
  check_scheme(c->scheme, E.V);
  check_scheme(c->target_scheme, E.V);
}

}  // namespace ssd

using namespace ssd;

struct ssd_engine {
  Engine e;
};

#define API_BEGIN try {
#define API_END                                      \
  }                                                  \
  catch (const Fail& f) {                            \
    g_last_error = f.what();                         \
    return ssd_status(f.code);                       \
  }                                                  \
  catch (const std::exception& x) {                  \
    g_last_error = x.what();                         \
    return SSD_ERROR;                                \
  }                                                  \
  return SSD_OK;

extern "C" {

const char* ssd_last_error(void) { return g_last_error.c_str(); }
int ssd_abi_version(void) { return SSD_B200_ABI_VERSION; }

ssd_status ssd_engine_create(const ssd_model_shape* target, const ssd_model_shape* draft, const ssd_pair_params* pair,
                             int32_t device, int32_t max_branches, int32_t max_lookahead, ssd_engine** out) {
  return ssd_engine_create_role(target, draft, pair, device, SSD_ROLE_COLOCATED, max_branches, max_lookahead, out);
}

ssd_status ssd_engine_create_role(const ssd_model_shape* target, const ssd_model_shape* draft,
                                  const ssd_pair_params* pair, int32_t device, int32_t role, int32_t max_branches,
                                  int32_t max_lookahead, ssd_engine** out) {
  return ssd_engine_create_tp(target, draft, pair, device, role, 0, 1, max_branches, max_lookahead, out);
}

static ssd_status engine_create(const ssd_model_shape* target, const ssd_model_shape* draft,
                                const ssd_pair_params* pair, int32_t device, int32_t role, int32_t tp_rank,
                                int32_t tp_size, int32_t max_batch, int32_t max_branches, int32_t max_lookahead,
                                ssd_engine** out) {
  API_BEGIN
  if (max_batch < 1) throw Fail(SSD_ERROR, "sim: batch_size must be >= 1");
  if (max_batch > 1 && (role != SSD_ROLE_COLOCATED || tp_size > 1))
    throw Fail(SSD_CONFIG, "engine: batch lanes are for the colocated engine");
  if (!target || !draft || !pair || !out) throw Fail(SSD_CONFIG, "engine: null argument");
  if (role < SSD_ROLE_COLOCATED || role > SSD_ROLE_SPECULATOR) throw Fail(SSD_CONFIG, "engine: unknown role");
  if (tp_size < 1 || tp_size > kTpMax || tp_rank < 0 || tp_rank >= tp_size) throw Fail(SSD_CONFIG, "engine: bad TP rank");
  if (tp_size > 1) {
    // a TP verifier of the split run, or a colocated TP engine (target
    // sharded, draft replicated on every rank) for the same-box AR / SD
    // baselines of a TP configuration (BASELINE configs[3])
    if (role == SSD_ROLE_SPECULATOR) throw Fail(SSD_CONFIG, "engine: tensor parallelism is for the target's ranks");
    const int T = tp_size;
    if (target->n_kv_heads % T || target->n_heads % T || target->ffn % T || target->vocab % T ||
        (target->ffn / T) % 128 || (target->n_heads / T * target->head_dim) % 128 || target->tied)
      throw Fail(SSD_CONFIG, "engine: target shape does not shard over this TP size");
  }
  if (target->vocab != draft->vocab) throw Fail(SSD_ERROR, "sim: target and draft shapes differ");
  if (draft->d_model > target->d_model || draft->ffn > target->ffn || !draft->tied)
    throw Fail(SSD_CONFIG, "engine: the draft must be tied and no wider than the target");
  for (const ssd_model_shape* s : {target, draft}) {
    if (s->head_dim < 16 || s->head_dim > 128 || (s->head_dim & (s->head_dim - 1)) || s->n_heads % s->n_kv_heads ||
        s->d_model % 8 || s->ffn % 8)
      throw Fail(SSD_CONFIG, "engine: unsupported shape");
  }
  if (max_lookahead < 1 || max_lookahead > kMaxK) throw Fail(SSD_TOO_LARGE, "engine: lookahead capacity");
  if (max_branches < 1 || max_branches > kMaxM) throw Fail(SSD_TOO_LARGE, "engine: branch capacity");
  for (const ssd_model_shape* s : {target, draft})
    if (s->n_heads / s->n_kv_heads > kMaxGroup || (kMaxGroup % (s->n_heads / s->n_kv_heads)))
      throw Fail(SSD_CONFIG, "engine: GQA group must divide 8");
  if (max_batch * std::max(max_branches, max_lookahead + 1) > kMaxM)
    throw Fail(SSD_TOO_LARGE, "engine: batch x branches above the forward capacity");
  CK(cudaSetDevice(device));
  // every validation is above; a failure below frees what was built so far
  std::unique_ptr<ssd_engine, ssd_status (*)(ssd_engine*)> holder(new ssd_engine(), ssd_engine_destroy);
  ssd_engine* h = holder.get();
  Engine& E = h->e;
  E.dev = device;
  E.nbmax = max_batch;
  E.maxB = max_branches;
  E.maxK = max_lookahead;
  E.V = target->vocab;
  E.role = role;
  if (const char* sk = std::getenv("SSD_B200_SKIP")) E.skip_mask = std::atoi(sk);
  if (const char* pf = std::getenv("SSD_B200_PF_MB")) E.pf_ahead = std::max(0LL, std::atoll(pf)) << 20;
  if (const char* pfd = std::getenv("SSD_B200_PF_MB_DRAFT")) E.pf_ahead_draft = std::max(0LL, std::atoll(pfd)) << 20;
  if (const char* acl = std::getenv("SSD_B200_ATTN_CL")) E.attn_cluster = std::atoi(acl) != 0;
  if (const char* adc = std::getenv("SSD_B200_ATTN_DEC")) E.attn_dec = std::atoi(adc) != 0;
  if (const char* ast = std::getenv("SSD_B200_ATTN_STAGE")) g_attn_stage = std::atoi(ast) != 0;
  if (const char* aw = std::getenv("SSD_B200_ATTN_DEC_WIDE_M")) E.attn_dec_wide_m = std::max(1, std::atoi(aw));
  if (const char* sg = std::getenv("SSD_B200_SMALL_GEMM_MB")) E.small_gemm_bytes = std::atoll(sg) << 20;
  if (const char* cg = std::getenv("SSD_B200_CL_GEMM_MB")) E.cl_gemm_bytes = std::atoll(cg) << 20;
  if (const char* cm = std::getenv("SSD_B200_CL_MIN_M")) E.cl_min_m = std::max(1, std::atoi(cm));
  if (const char* cf = std::getenv("SSD_B200_CL_FUSED")) E.cl_fused = std::atoi(cf) != 0;
  if (const char* sw = std::getenv("SSD_B200_SWIGLU_WHOLE")) g_swiglu_whole = std::atoi(sw) != 0;
  if (const char* swr = std::getenv("SSD_B200_SWIGLU_REDUCE_UNITS")) g_swiglu_reduce_units = std::max(0, std::atoi(swr));
  E.deterministic = role != SSD_ROLE_COLOCATED || tp_size > 1;
  if (const char* dt = std::getenv("SSD_B200_DETERMINISTIC")) E.deterministic = E.deterministic || std::atoi(dt) != 0;
  if (const char* cs = std::getenv("SSD_B200_CORUN_SMALL_GEMM_MB")) E.corun_small_gemm_bytes = std::atoll(cs) << 20;
  if (const char* cls = std::getenv("SSD_B200_CL_SMALL")) E.cl_small = std::atoi(cls) != 0;
  if (const char* ca = std::getenv("SSD_B200_CORUN_ATTN_KB")) E.corun_attn_kb = std::max(8, std::min(227, std::atoi(ca)));
  if (const char* vae = std::getenv("SSD_B200_VERIFY_AFTER_EXTEND")) E.verify_after_extend = std::atoi(vae) != 0;
  if (const char* sp = std::getenv("SSD_B200_SPLIT_SMS")) std::sscanf(sp, "%d,%d", &E.split_t, &E.split_d);
  {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    E_num_sms = sms;
  }
  const int nb = max_batch;
  const int maxM = nb * std::max(max_branches, max_lookahead + 1);
  if (maxM > kMaxM) throw Fail(SSD_TOO_LARGE, "engine: batch x branches above the forward capacity");
  // a split process materialises only its own model
  if (role != SSD_ROLE_SPECULATOR)
    build_model(E.T, *target, *draft, *pair, 0, 0, std::max(maxM, kPrefillChunk), tp_rank, tp_size, nb);
  else E.T.s = *target;
  if (role != SSD_ROLE_VERIFIER)
    build_model(E.D, *draft, *draft, *pair, 1, max_branches * max_lookahead, std::max(maxM, kPrefillChunk), 0, 1, nb);
  else E.D.s = *draft;
  configure_kernels();
  {
    // colocated SSD: optionally give the speculator (the longer chain of
    // dependent steps per round) the higher stream priority
    // (SSD_B200_SPEC_PRIO=1; measured neutral, profiles/r01_summary.md)
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    const char* sp = std::getenv("SSD_B200_SPEC_PRIO");
    const bool prio = sp && std::atoi(sp) != 0;
    CK(cudaStreamCreateWithPriority(&E.sv, cudaStreamNonBlocking, lo));
    CK(cudaStreamCreateWithPriority(&E.ss, cudaStreamNonBlocking, prio ? hi : lo));
  }
  if (role == SSD_ROLE_COLOCATED && tp_size == 1) {
    // default: 3/8 of the SMs for the verifier (bench workload sweep,
    // profiles/r02g_summary.md); SSD_B200_GREEN=<SMs> overrides, 0 = shared
    int want = E_num_sms * 3 / 8;
    if (const char* gv = std::getenv("SSD_B200_GREEN")) want = std::atoi(gv);
    if (const char* gt = std::getenv("SSD_B200_GREEN_TAIL")) E.green_tail = std::atoi(gt);
    if (const char* ef = std::getenv("SSD_B200_EXTEND_FULL")) E.extend_full = std::atoi(ef) != 0;
    CK(cudaEventCreateWithFlags(&E.ev_tail, cudaEventDisableTiming));
    try {
      set_green(E, want);
    } catch (const Fail&) {
      // no green-context support (driver, MIG, MPS limits): the round runs
      // on shared SMs; ssd_engine_sm_partition reports the error explicitly
      drop_green(E);
      cudaGetLastError();
    }
  }
  CK(cudaEventCreateWithFlags(&E.ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&E.ev_verified, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&E.ev_join, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&E.ev_extended, cudaEventDisableTiming));
  CK(cudaEventCreate(&E.ev_t0));
  CK(cudaEventCreate(&E.ev_t1));
  CK(cudaEventCreateWithFlags(&E.ev_prespec, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&E.ev_user, cudaEventDisableTiming));
  CK(cudaHostAlloc(reinterpret_cast<void**>(&E.pin_rng), sizeof(Mt64), cudaHostAllocDefault));
  auto own = [&](void* p) { E.owned.push_back(p); return p; };
  const int K = max_lookahead, B = max_branches, V = E.V;
  E.st = static_cast<LoopState*>(own(dalloc<LoopState>(size_t(nb))));
  E.hist_stride = std::max(target->max_ctx, draft->max_ctx) + K + 2;
  E.hist = static_cast<int*>(own(dalloc<int>(size_t(nb) * E.hist_stride)));
  E.d_lanes = static_cast<int*>(own(dalloc<int>(size_t(nb))));
  E.P_t = static_cast<FwdParams*>(own(dalloc<FwdParams>(1)));
  E.P_x = static_cast<FwdParams*>(own(dalloc<FwdParams>(1)));
  E.P_b = static_cast<FwdParams*>(own(dalloc<FwdParams>(1)));
  E.P_s = static_cast<FwdParams*>(own(dalloc<FwdParams>(1)));
  E.P_pre = static_cast<FwdParams*>(own(dalloc<FwdParams>(1)));
  E.tlogits = static_cast<float*>(own(dalloc<float>(size_t(nb) * (K + 1) * V)));
  E.xrows = static_cast<float*>(own(dalloc<float>(size_t(nb) * (K + 1) * V)));
  E.dmain = static_cast<float*>(own(dalloc<float>(size_t(K) * nb * V)));
  E.brows[0] = static_cast<float*>(own(dalloc<float>(size_t(K) * nb * B * V)));
  E.brows[1] = static_cast<float*>(own(dalloc<float>(size_t(K) * nb * B * V)));
  E.keys = static_cast<int*>(own(dalloc<int>(size_t(nb) * (K + 1) * kMaxTopF)));
  E.bk = static_cast<int*>(own(dalloc<int>(size_t(nb) * B)));
  E.btok = static_cast<int*>(own(dalloc<int>(size_t(nb) * B)));
  E.bt = static_cast<int*>(own(dalloc<int>(size_t(nb) * B * K)));
  E.bu = static_cast<double*>(own(dalloc<double>(size_t(nb) * B * K)));
  E.ubuf = static_cast<double*>(own(dalloc<double>(64)));
  E.plans = static_cast<int*>(own(dalloc<int>(size_t(2 * (K + 1)))));
  E.offs = static_cast<int*>(own(dalloc<int>(size_t(2 * (K + 1)))));
  E.rstat = static_cast<RowStat*>(own(dalloc<RowStat>(size_t(nb) * (2 * K + 1))));
  E.tok_scratch = static_cast<int*>(own(dalloc<int>(64)));
  E.nch = std::max(1, std::min(kMaxChunks, (V + 1023) / 1024));
  {
    const int rows = nb * std::max(B, K + 1);
    E.cand = static_cast<VI*>(own(dalloc<VI>(size_t(rows) * E.nch * (kMaxTopF + 1))));
    E.rstat2 = static_cast<RowChunk*>(own(dalloc<RowChunk>(size_t(rows) * E.nch)));
  }
  // exact sequential cumulative of the uniform law (FastRandom tokens)
  std::vector<double> cum(static_cast<size_t>(V));
  double c = 0.0;
  for (int i = 0; i < V; ++i) { c += 1.0 / V; cum[size_t(i)] = c; }
  E.cum = static_cast<double*>(own(dalloc<double>(size_t(V))));
  h2d(E, E.cum, cum.data(), size_t(V) * 8);
  // mailbox (own allocation so it can be exported alone by CUDA IPC)
  {
    void* p = nullptr;
    CK(cudaMalloc(&p, kInboxRows + size_t(2) * K * V * 4));
    CK(cudaMemset(p, 0, kInboxRows + size_t(2) * K * V * 4));
    E.inbox = static_cast<Inbox*>(p);
    E.send_counter = static_cast<int*>(own(dalloc<int>(1)));
  }
  if (tp_size > 1) {  // TP collective region (own allocation: exported alone)
    E.tp_L = TpLayout{tp_size, E.T.maxM, target->d_model, target->vocab};
    void* p = nullptr;
    CK(cudaMalloc(&p, E.tp_L.bytes()));
    CK(cudaMemset(p, 0, E.tp_L.bytes()));
    if (std::getenv("SSD_B200_TP_POISON"))  // debug: slots start as NaN (flags stay 0)
      CK(cudaMemset(static_cast<char*>(p) + E.tp_L.ar_off(), 0xFF, E.tp_L.bytes() - E.tp_L.ar_off()));
    E.tp_region = static_cast<char*>(p);
    E.tp_ctl = static_cast<TpCtl*>(own(dalloc<TpCtl>(1)));
  }
  CK(cudaDeviceSynchronize());
  *out = holder.release();
  API_END
}

ssd_status ssd_engine_create_tp(const ssd_model_shape* target, const ssd_model_shape* draft,
                                const ssd_pair_params* pair, int32_t device, int32_t role, int32_t tp_rank,
                                int32_t tp_size, int32_t max_branches, int32_t max_lookahead, ssd_engine** out) {
  return engine_create(target, draft, pair, device, role, tp_rank, tp_size, 1, max_branches, max_lookahead, out);
}

ssd_status ssd_engine_create_batch(const ssd_model_shape* target, const ssd_model_shape* draft,
                                   const ssd_pair_params* pair, int32_t device, int32_t max_batch, int32_t max_branches,
                                   int32_t max_lookahead, ssd_engine** out) {
  return engine_create(target, draft, pair, device, SSD_ROLE_COLOCATED, 0, 1, max_batch, max_branches, max_lookahead,
                       out);
}

ssd_status ssd_engine_destroy(ssd_engine* h) {
  API_BEGIN
  if (!h) return SSD_OK;
  Engine& E = h->e;
  cudaSetDevice(E.dev);
  cudaDeviceSynchronize();
  free_model(E.T);
  free_model(E.D);
  for (void* p : E.ipc_opened) cudaIpcCloseMemHandle(p);
  for (void* p : E.tp_opened) cudaIpcCloseMemHandle(p);
  if (E.tp_region) cudaFree(E.tp_region);
  if (E.inbox) cudaFree(E.inbox);
  if (E.peers_dev) cudaFree(E.peers_dev);
  for (auto g : E.ssd_graphs)
    if (g) cudaGraphExecDestroy(g);
  if (E.ssd_log) cudaFree(E.ssd_log);
  for (void* p : E.owned) cudaFree(p);
  for (cudaStream_t st : {E.sv, E.ss})
    if (st) cudaStreamDestroy(st);
  drop_green(E);
  for (cudaEvent_t ev : {E.ev_fork, E.ev_verified, E.ev_join, E.ev_t0, E.ev_t1, E.ev_prespec, E.ev_user, E.ev_extended, E.ev_tail})
    if (ev) cudaEventDestroy(ev);
  if (E.pin_rng) cudaFreeHost(E.pin_rng);
  if (E.prof_ts) cudaFree(E.prof_ts);
  cudaGetLastError();  // teardown errors must not surface in a later call
  delete h;
  API_END
}

int64_t ssd_engine_weight_bytes(const ssd_engine* h, int32_t which) {
  if (!h) return 0;
  return which == 0 ? h->e.T.weight_bytes : h->e.D.weight_bytes;
}

ssd_status ssd_run_ar(ssd_engine* h, const int32_t* prompt, int32_t n0, const ssd_scheme* ts, int64_t tokens,
                      uint64_t seed, int32_t* out, int64_t cap, ssd_run_stats* stats) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  need(E.T, "run_ar");
  if (tokens < 1) throw Fail(SSD_ERROR, "run_ar: tokens must be >= 1");
  if (!ts) throw Fail(SSD_CONFIG, "run_ar: scheme required");
  check_scheme(*ts, E.V);
  set_history(E, prompt, n0, int(n0 + tokens + 1));
  cudaStream_t s = E.sv;
  reset_state(E, 1, n0, tokens, derive_seed(seed, 0), 0, nullptr, s);
  if (n0 > 1) prefill(E, E.T, n0 - 1, nullptr, s);
  const DScheme d = dscheme(*ts);
  // one decode step = one graph (device-resident state: no host round trip)
  E.launches = 0;
  GraphSet gs;
  gs.g.push_back(capture_graph(s, [&] {
    prep_chain_kernel<<<1, 32, 0, s>>>(E.st, E.hist, E.P_t, 1, E.hist_stride, E.T.lane_S, E.T.km);
    forward(E, E.T, E.P_t, 1, E.tlogits, s);
    draw_uniforms_kernel<<<1, 32, 0, s>>>(&E.st->drng, E.ubuf, 1);
    row_pick(E, E.tlogits, size_t(E.V), 1, E.V, d, E.ubuf, 1, E.tok_scratch, 1, s);
    ar_commit_kernel<<<1, 32, 0, s>>>(E.st, E.hist, E.tok_scratch);
    KCHECK();
    E.launches += 3;
  }));
  const long long per_step = E.launches;
  CK(cudaEventRecord(E.ev_t0, s));
  for (int64_t i = 0; i < tokens; ++i) CK(cudaGraphLaunch(gs.g[0], s));
  E.launches = per_step * tokens;
  CK(cudaEventRecord(E.ev_t1, s));
  CK(cudaStreamSynchronize(s));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, E.ev_t0, E.ev_t1));
  LoopState st = read_state(E);
  raise_device_error(st);
  st.clock = double(tokens);
  fill_stats(st, tokens, ms, E.launches, stats);
  copy_out(E, n0, st.n, out, cap, nullptr);
  API_END
}

ssd_status ssd_run_sd(ssd_engine* h, const int32_t* prompt, int32_t n0, const ssd_sim_config* c, int32_t* out,
                      int64_t cap, int64_t* out_len, ssd_run_stats* stats) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  validate_cfg(E, c);
  need(E.T, "run_sd");
  need(E.D, "run_sd");
  const int K = c->lookahead;
  set_history(E, prompt, n0, int(n0 + c->rounds * (K + 1) + K + 2));
  cudaStream_t s = E.sv;
  reset_state(E, K, n0, c->rounds, derive_seed(c->seed, 0), 0, c, s);
  if (n0 > 1) prefill(E, E.D, n0 - 1, nullptr, s);
  if (n0 > 1) prefill(E, E.T, n0 - 1, nullptr, s);
  // one round (K draft steps, verify forward, decision, commit) = one graph
  E.launches = 0;
  GraphSet gs;
  gs.g.push_back(capture_graph(s, [&] {
    draft_steps(E, K, c->scheme, 0, 0, s);
    verify_round(E, K, c->target_scheme, c->scheme, c->accept_scale, /*single stream*/ 1, s);
    commit_kernel<<<1, 32, 0, s>>>(E.st);
    KCHECK();
    ++E.launches;
  }));
  const long long per_round = E.launches;
  CK(cudaEventRecord(E.ev_t0, s));
  for (int64_t r = 0; r < c->rounds; ++r) CK(cudaGraphLaunch(gs.g[0], s));
  E.launches = per_round * c->rounds;
  CK(cudaEventRecord(E.ev_t1, s));
  CK(cudaStreamSynchronize(s));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, E.ev_t0, E.ev_t1));
  LoopState st = read_state(E);
  raise_device_error(st);
  st.clock = double(c->rounds) * (1.0 + c->primary_time);
  fill_stats(st, c->rounds, ms, E.launches, stats);
  copy_out(E, n0, st.n, out, cap, out_len);
  API_END
}

}  // extern "C"

namespace ssd {

// run_protocol_harness (sim.cpp:502-601) over `nb` batch lanes: lane l is
// sequence j = l with draft stream derive_seed(seed, l) and verifier stream
// derive_seed(derive_seed(seed, 0x5EED), l) (sim.cpp:379-380, 516-518); all
// lanes share the prompt, their forwards are batched (verify M = nb (K+1),
// branch steps M = nb B), and a miss in any lane stalls the round's clock
// for the backup (sim.cpp:570-577).
// mode 1: run_ssd_batch semantics (sim.cpp:128-250) — one stream per
// sequence (verify, then the cache base, then the backup), cache built after
// verify, clock += previous all hit ? max(1, T_p) : 1 + T_b. tr: optional
// per-round transcript log (sim.cpp:271-317).
static void run_ssd_impl(Engine& E, const int32_t* prompt, int32_t n0, const ssd_sim_config* c, int nb, int32_t* out,
                         int64_t cap, int64_t* out_lens, int32_t* out_outcomes, int32_t* out_hits, ssd_run_stats* stats,
                         double* prof = nullptr, int mode = 0, std::vector<int>* tr_i = nullptr,
                         std::vector<double>* tr_d = nullptr, std::vector<int>* tr_init = nullptr) {
  CK(cudaSetDevice(E.dev));
  validate_cfg(E, c);
  need(E.T, "run_ssd");
  need(E.D, "run_ssd");
  if (nb < 1) throw Fail(SSD_ERROR, "sim: batch_size must be >= 1");
  if (nb > E.nbmax) throw Fail(SSD_TOO_LARGE, "sim: batch_size exceeds the engine's batch capacity");
  if (E.T.tp_size > 1) throw Fail(SSD_CONFIG, "run_ssd: a tensor-parallel target runs SSD in the split mode (ssd_run_ssd_verifier)");
  const int K = c->lookahead;
  int B = 0, max_f = 0;
  upload_plans(E, c->primary_plan, c->backup_plan, K, B, max_f);
  if (nb * B > E.D.maxM || nb * (K + 1) > E.T.maxM) throw Fail(SSD_TOO_LARGE, "sim: batch x branches exceeds capacity");
  set_history(E, prompt, n0, int(n0 + c->rounds * (K + 1) + 2 * K + 2), nb);
  const int64_t R = c->rounds;
  // per-round logs (their address is baked into the graphs): [2 cap]
  // outcomes + [cap] hits, then the transcript log [cap][maxB lanes][kTrInts]
  // ints and [cap][2] doubles
  const size_t tr_ints = size_t(E.nbmax) * kTrInts;
  if (R > E.ssd_log_cap) {
    if (E.ssd_log) cudaFree(E.ssd_log);
    E.ssd_log = nullptr;
    E.ssd_log_cap = 0;
    E.ssd_log = dalloc<int>(size_t(R) * (3 + tr_ints + 4));
    E.ssd_log_cap = R;
  }
  int* const d_out = E.ssd_log;
  int* const d_hit = E.ssd_log + 2 * E.ssd_log_cap;
  TrLog tr{nullptr, nullptr, n0};
  if (tr_i) {
    tr.i = E.ssd_log + 3 * E.ssd_log_cap;
    tr.d = reinterpret_cast<double*>(tr.i + ((size_t(E.ssd_log_cap) * tr_ints + 1) & ~size_t(1)));
  }
  cudaStream_t sv = E.sv, ss = E.ss;
  for (int l = 0; l < nb; ++l) {
    // harness: draft stream derive_seed(seed, j), verifier derive_seed(derive_seed(seed, 0x5EED), j)
    // (sim.cpp:379-380, 516-518); run_ssd_batch: the single stream derive_seed(seed, j) (sim.cpp:142)
    reset_state(E, K, n0, R, derive_seed(c->seed, uint64_t(l)), derive_seed(derive_seed(c->seed, 0x5EED), uint64_t(l)),
                c, sv, l);
    if (n0 > 1) prefill(E, E.D, n0 - 1, nullptr, sv, l);
    if (n0 > 1) prefill(E, E.T, n0 - 1, nullptr, sv, l);
  }
  // initial synchronous drafts; clock starts at T_p (sim.cpp:524-526)
  std::vector<int> lanes(static_cast<size_t>(nb));
  for (int l = 0; l < nb; ++l) lanes[size_t(l)] = l;
  CK(cudaMemcpyAsync(E.d_lanes, lanes.data(), size_t(nb) * 4, cudaMemcpyHostToDevice, sv));
  draft_lanes(E, K, c->scheme, 0, 0, nb, sv);
  for (int l = 0; l < nb; ++l) {
    const double clock0 = mode == 1 ? 1.0 + c->primary_time : c->primary_time;
    CK(cudaMemcpyAsync(reinterpret_cast<char*>(E.st + l) + offsetof(LoopState, clock), &clock0, sizeof(double),
                       cudaMemcpyHostToDevice, sv));
    CK(cudaStreamSynchronize(sv));
  }
  if (tr_init) {  // the initial speculations (the transcript's first d2v message)
    tr_init->clear();
    for (int l = 0; l < nb; ++l) {
      const LoopState h0 = read_state(E, l);
      tr_init->insert(tr_init->end(), h0.spec, h0.spec + K);
    }
  }
  const bool jit = c->backup_kind == 0;
  // One SSD round = one graph: the verifier branch (verify forward +
  // decision) and the speculator branch (extend, keys, K branch steps) fork
  // from the verifier stream and join at the lookup. Two graphs alternate the
  // branch-row buffers (the next round's verifier reads this round's rows).
  E.launches = 0;
  // verifier and speculator GEMMs on disjoint SM sets so both streams run at once
  E.T.gemm_ctas = E.green_v ? E.green_v : E.split_t;
  E.D.gemm_ctas = E.green_v ? E.green_s : E.split_d;
  const long long small_saved = E.small_gemm_bytes;
  // co-running streams on shared SMs: the co-resident (small-budget) GEMM
  // configuration; on disjoint partitions each stream keeps the full one
  if (!E.gsv) E.small_gemm_bytes = std::max(E.small_gemm_bytes, E.corun_small_gemm_bytes);
  g_attn_smem_cap_kb = E.corun_attn_kb;
  struct Uncap {
    Engine& e;
    long long small;
    ~Uncap() { e.T.gemm_ctas = e.D.gemm_ctas = 0; e.small_gemm_bytes = small; g_attn_smem_cap_kb = 227; }
  } uncap{E, small_saved};
  // every value the capture bakes into kernel parameters or launch shapes
  char keybuf[512];
  std::snprintf(keybuf, sizeof keybuf, "%d %d %d %d | %d %d %.17g %.17g | %d %d %.17g %.17g | %.17g | %d %d | %d %d | %p %lld %d",
                K, B, max_f, nb, c->scheme.kind, c->scheme.fan_out, c->scheme.temperature, c->scheme.downweight,
                c->target_scheme.kind, c->target_scheme.fan_out, c->target_scheme.temperature,
                c->target_scheme.downweight, c->accept_scale, E.T.ctx_bound, E.D.ctx_bound, E.T.gemm_ctas, E.D.gemm_ctas,
                static_cast<void*>(E.ssd_log), E.small_gemm_bytes, g_attn_smem_cap_kb);
  const std::string key = std::string(keybuf) + (E.prof_on ? " prof" : "") + " mode" + std::to_string(mode) +
                          " vae" + std::to_string(E.verify_after_extend) + " tail" + std::to_string(E.green_tail) + " xf" + std::to_string(E.extend_full) +
                          (tr.i ? " tr" : "") + " n0 " + std::to_string(n0);
  if (key != E.ssd_graph_key || E.ssd_graphs.size() != 2) {
    for (auto g : E.ssd_graphs)
      if (g) cudaGraphExecDestroy(g);
    E.ssd_graphs.clear();
    E.ssd_graph_key.clear();
    GraphSet gs;
    // green partition: the round's two branches are captured on the green streams
    cudaStream_t cv = E.gsv ? E.gsv : sv, cs = E.gss ? E.gss : ss;
  for (int parity = 0; parity < 2; ++parity) {
    gs.g.push_back(capture_graph(cv, [&] {
      mark(E, 0, cv);
      CK(cudaEventRecord(E.ev_fork, cv));
      CK(cudaStreamWaitEvent(cs, E.ev_fork, 0));
      mark(E, 3, cs);
      cudaStream_t cend = cs;  // the speculator's last stream (lookup, join)
      if (mode == 1) {
        // verify first on the sequence stream; extend + keys overlap it, the
        // branch streams / steps follow it (their base is drawn after verify)
        verify_round(E, K, c->target_scheme, c->scheme, c->accept_scale, 1, cv, nb);
        CK(cudaEventRecord(E.ev_verified, cv));
        prespeculate(E, K, B, 0, B, max_f, c->scheme, parity, cs, nb, E.ev_verified);
      } else {
        // verify_after_extend: the verify forward starts when the extend
        // forward has finished, so the speculator's first (critical-path)
        // forward does not share HBM with the verifier's heaviest GEMMs
        const int tail = E.gsv && E.green_tail >= 0 && E.green_tail < K ? E.green_tail : -1;
        if (E.gsv && E.extend_full) {
          // the extend forward (+ keys, branch streams) first, on every SM;
          // then the verifier and the branch steps on their partitions
          CK(cudaStreamWaitEvent(ss, E.ev_fork, 0));
          const int dcap = E.D.gemm_ctas;
          E.D.gemm_ctas = 0;
          prespeculate(E, K, B, 0, B, max_f, c->scheme, parity, ss, nb, nullptr, -1, nullptr, -1, 0);
          E.D.gemm_ctas = dcap;
          CK(cudaEventRecord(E.ev_extended, ss));
          CK(cudaStreamWaitEvent(cs, E.ev_extended, 0));
          CK(cudaStreamWaitEvent(cv, E.ev_extended, 0));
          prespeculate(E, K, B, 0, B, max_f, c->scheme, parity, cs, nb, nullptr, -1, nullptr, 0, tail >= 0 ? tail : K);
        } else {
          prespeculate(E, K, B, 0, B, max_f, c->scheme, parity, cs, nb, nullptr, -1,
                       E.verify_after_extend ? E.ev_extended : nullptr, -1, tail);
          if (E.verify_after_extend) CK(cudaStreamWaitEvent(cv, E.ev_extended, 0));
        }
        verify_round(E, K, c->target_scheme, c->scheme, c->accept_scale, 0, cv, nb);
        CK(cudaEventRecord(E.ev_verified, cv));
        CK(cudaStreamWaitEvent(cs, E.ev_verified, 0));
        if (tail >= 0) {
          // the verifier is done: the remaining branch steps on every SM
          // (ordinary stream, uncapped GEMM grids, the full-budget configs)
          CK(cudaEventRecord(E.ev_tail, cs));
          CK(cudaStreamWaitEvent(ss, E.ev_tail, 0));
          const int dcap = E.D.gemm_ctas;
          const long long small = E.small_gemm_bytes;
          E.D.gemm_ctas = 0;
          E.small_gemm_bytes = small_saved;
          prespeculate(E, K, B, 0, B, max_f, c->scheme, parity, ss, nb, nullptr, -1, nullptr, tail, K);
          E.D.gemm_ctas = dcap;
          E.small_gemm_bytes = small;
          cend = ss;
        }
      }
      lookup_kernel<<<1, 32, 0, cend>>>(E.st, nb, E.keys, max_f, E.offs, E.bt, E.brows[parity], 0, nb * B, B, E.V,
                                        E.cum, d_out, d_hit, mode, tr);
      KCHECK();
      mark(E, kMarkRoundEnd, cend);
      ++E.launches;
      CK(cudaEventRecord(E.ev_join, cend));
      CK(cudaStreamWaitEvent(cv, E.ev_join, 0));
    }));
  }
    E.ssd_graphs = gs.g;
    gs.g.clear();
    E.ssd_graph_key = key;
    E.ssd_graph_launches = E.launches / 2;
  }
  const long long per_round = E.ssd_graph_launches;
  E.launches = 0;
  E.small_gemm_bytes = small_saved;  // JIT re-drafts below run alone on one stream
  g_attn_smem_cap_kb = 227;
  long long jit_launches = 0;
  std::vector<int> hits(static_cast<size_t>(nb));
  CK(cudaEventRecord(E.ev_t0, sv));
  for (int64_t r = 0; r < R; ++r) {
    CK(cudaGraphLaunch(E.ssd_graphs[size_t(r & 1)], sv));
    if (E.prof_on && prof) {  // in-graph segment times of this round (one host sync per round)
      CK(cudaMemcpyAsync(E.prof_h, E.prof_ts, sizeof E.prof_h, cudaMemcpyDeviceToHost, sv));
      CK(cudaStreamSynchronize(sv));
      auto el = [&](int a, int b) { return 1e-6 * double(static_cast<long long>(E.prof_h[b] - E.prof_h[a])); };
      prof[0] += el(0, kMarkRoundEnd);
      prof[1] += el(0, 1);
      prof[2] += el(1, 2);
      prof[3] += el(3, 4);
      prof[4] += el(4, 5);
      int prev = 5;
      for (int j = 0; j < std::min(K, 8); ++j) {
        prof[5] += el(prev, 6 + 2 * j);
        prof[6] += el(6 + 2 * j, 7 + 2 * j);
        prev = 7 + 2 * j;
      }
      prof[7] += el(prev, kMarkRoundEnd);
      prof[8] += el(0, 3);
      prof[9] += 1.0;
    }
    if (jit && r + 1 < R) {
      // SamePrimaryJIT: the lanes that missed re-draft from their new
      // history, batched (the one host round trip of the JIT backup)
      CK(cudaStreamSynchronize(sv));
      CK(cudaMemcpy2DAsync(hits.data(), sizeof(int), reinterpret_cast<char*>(E.st) + offsetof(LoopState, hit),
                           sizeof(LoopState), sizeof(int), size_t(nb), cudaMemcpyDeviceToHost, sv));
      CK(cudaStreamSynchronize(sv));
      int nm = 0;
      for (int l = 0; l < nb; ++l)
        if (!hits[size_t(l)]) lanes[size_t(nm++)] = l;
      if (nm > 0) {
        const long long before = E.launches;
        CK(cudaMemcpyAsync(E.d_lanes, lanes.data(), size_t(nm) * 4, cudaMemcpyHostToDevice, sv));
        draft_lanes(E, K, c->scheme, 1, 2, nm, sv);
        if (tr.i) tr_log_spec_kernel<<<1, 32, 0, sv>>>(E.st, E.d_lanes, nm, nb, tr);
        jit_launches += E.launches - before;
      }
    }
  }
  E.launches = per_round * R + jit_launches;
  CK(cudaEventRecord(E.ev_t1, sv));
  CK(cudaStreamSynchronize(sv));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, E.ev_t0, E.ev_t1));
  std::vector<LoopState> sts;
  for (int l = 0; l < nb; ++l) sts.push_back(read_state(E, l));
  if (out_outcomes) d2h(E, out_outcomes, d_out, size_t(2 * R) * 4);
  if (out_hits) d2h(E, out_hits, d_hit, size_t(R) * 4);
  if (tr.i) {
    tr_i->resize(size_t(R) * nb * kTrInts);
    tr_d->resize(size_t(2 * R));
    for (int64_t r = 0; r < R; ++r)
      d2h(E, tr_i->data() + size_t(r) * nb * kTrInts, tr.i + size_t(r) * nb * kTrInts, size_t(nb) * kTrInts * 4);
    d2h(E, tr_d->data(), tr.d, size_t(2 * R) * 8);
  }
  const LoopState st = sum_lanes(sts);
  raise_device_error(st);
  fill_stats(st, R, ms, E.launches, stats);
  for (int l = 0; l < nb; ++l)
    copy_out(E, n0, sts[size_t(l)].n, out ? out + size_t(l) * cap : nullptr, cap, out_lens ? out_lens + l : nullptr, l);
}

}  // namespace ssd

using namespace ssd;

extern "C" {

ssd_status ssd_run_ssd(ssd_engine* h, const int32_t* prompt, int32_t n0, const ssd_sim_config* c, int32_t* out,
                       int64_t cap, int64_t* out_len, int32_t* out_outcomes, int32_t* out_hits, ssd_run_stats* stats) {
  API_BEGIN
  run_ssd_impl(h->e, prompt, n0, c, 1, out, cap, out_len, out_outcomes, out_hits, stats);
  API_END
}

ssd_status ssd_run_ssd_batch(ssd_engine* h, const int32_t* prompt, int32_t n0, const ssd_sim_config* c, int32_t batch,
                             int32_t* out, int64_t cap, int64_t* out_lens, int32_t* out_outcomes, int32_t* out_hits,
                             ssd_run_stats* stats) {
  API_BEGIN
  run_ssd_impl(h->e, prompt, n0, c, batch, out, cap, out_lens, out_outcomes, out_hits, stats);
  API_END
}

// JSONL transcript (reference Transcript::to_jsonl, sim.cpp:489-500): one
// line per message, keys as the reference's Channel writes them.
static std::string transcript_jsonl(const std::vector<int>& ti, const std::vector<double>& td,
                                    const std::vector<int>& init, int nb, int K, int V, int64_t R, double t0) {
  std::string out;
  char buf[64];
  auto num = [&](double v) { std::snprintf(buf, sizeof buf, "%.17g", v); return std::string(buf); };
  auto d2v = [&](int64_t round, const int* hits, const std::vector<std::vector<int>>& toks, double vclock) {
    std::string h = "[", t = "[";
    for (int l = 0; l < nb; ++l) {
      h += (l ? "," : "") + std::to_string(hits ? hits[l] : 0);
      t += l ? ",[" : "[";
      for (int i = 0; i < K; ++i) t += (i ? "," : "") + std::to_string(toks[size_t(l)][size_t(i)]);
      t += "]";
    }
    out += "{\"dir\":\"d2v\",\"payload_summary\":{\"dists_shape\":[" + std::to_string(K) + "," + std::to_string(V) +
           "],\"hits\":" + h + "],\"tokens\":" + t + "]},\"round\":" + std::to_string(round) + ",\"vclock\":" + num(vclock) + "}\n";
  };
  std::vector<std::vector<int>> toks(static_cast<size_t>(nb), std::vector<int>(static_cast<size_t>(K)));
  for (int l = 0; l < nb; ++l)
    for (int i = 0; i < K; ++i) toks[size_t(l)][size_t(i)] = init[size_t(l) * K + i];
  d2v(1, nullptr, toks, t0);
  for (int64_t r = 0; r < R; ++r) {
    std::string o = "[", sl = "[";
    std::vector<int> hits(static_cast<size_t>(nb));
    for (int l = 0; l < nb; ++l) {
      const int* e = ti.data() + (size_t(r) * nb + l) * kTrInts;
      o += (l ? ",[" : "[") + std::to_string(e[0]) + "," + std::to_string(e[1]) + "]";
      sl += (l ? "," : "") + std::to_string(e[3]);
      hits[size_t(l)] = e[2];
      for (int i = 0; i < K; ++i) toks[size_t(l)][size_t(i)] = e[4 + i];
    }
    out += "{\"dir\":\"v2d\",\"payload_summary\":{\"outcomes\":" + o + "],\"seq_lens\":" + sl + "]},\"round\":" +
           std::to_string(r + 1) + ",\"vclock\":" + num(td[size_t(2 * r)]) + "}\n";
    if (r + 1 < R) d2v(r + 2, hits.data(), toks, td[size_t(2 * r + 1)]);
  }
  return out;
}

ssd_status ssd_run_ssd_ex(ssd_engine* h, const int32_t* prompt, int32_t n0, const ssd_sim_config* c, int32_t batch,
                          const ssd_run_options* opt, int32_t* out, int64_t cap, int64_t* out_lens, int32_t* out_outcomes,
                          int32_t* out_hits, ssd_run_stats* stats) {
  API_BEGIN
  Engine& E = h->e;
  const int mode = opt ? opt->semantics : SSD_SEMANTICS_HARNESS;
  if (mode != SSD_SEMANTICS_HARNESS && mode != SSD_SEMANTICS_SEQUENTIAL) throw Fail(SSD_CONFIG, "run_ssd: unknown semantics");
  const bool want_tr = opt && (opt->transcript || opt->transcript_len);
  if (want_tr && mode != SSD_SEMANTICS_HARNESS) throw Fail(SSD_CONFIG, "transcript: harness semantics only");
  std::vector<int> ti, init;
  std::vector<double> td;
  run_ssd_impl(E, prompt, n0, c, batch, out, cap, out_lens, out_outcomes, out_hits, stats, nullptr, mode,
               want_tr ? &ti : nullptr, want_tr ? &td : nullptr, want_tr ? &init : nullptr);
  if (want_tr) {
    const std::string j = transcript_jsonl(ti, td, init, batch, c->lookahead, E.V, c->rounds, c->primary_time);
    if (opt->transcript_len) *opt->transcript_len = int64_t(j.size());
    if (opt->transcript && opt->transcript_cap > 0) {
      const size_t n = std::min<size_t>(j.size(), size_t(opt->transcript_cap - 1));
      std::memcpy(opt->transcript, j.data(), n);
      opt->transcript[n] = 0;
    }
  }
  API_END
}

ssd_status ssd_profile_ssd_round(ssd_engine* h, const int32_t* prompt, int32_t n0, const ssd_sim_config* c,
                                 double* out_ms, ssd_run_stats* stats) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  if (!out_ms) throw Fail(SSD_CONFIG, "profile_ssd_round: null output");
  if (!E.prof_ts) E.prof_ts = dalloc<unsigned long long>(32);
  double acc[10] = {0};
  E.prof_on = 1;
  struct Off {
    Engine& e;
    ~Off() { e.prof_on = 0; }
  } off{E};
  run_ssd_impl(E, prompt, n0, c, 1, nullptr, 0, nullptr, nullptr, nullptr, stats, acc);
  const double n = acc[9] > 0 ? acc[9] : 1.0;
  for (int i = 0; i < 9; ++i) out_ms[i] = acc[i] / n;
  API_END
}

// ------------------------------------------------- split processes (§6)

ssd_status ssd_mailbox_export(ssd_engine* h, uint8_t* handle64) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  if (!handle64) throw Fail(SSD_CONFIG, "mailbox: null handle buffer");
  cudaIpcMemHandle_t mh;
  CK(cudaIpcGetMemHandle(&mh, E.inbox));
  static_assert(sizeof(mh) == SSD_MAILBOX_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle64, &mh, sizeof(mh));
  API_END
}

ssd_status ssd_mailbox_connect(ssd_engine* h, int32_t n_peers, const uint8_t* handles, int32_t self) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  if (n_peers < 2 || !handles || self < 0 || self >= n_peers) throw Fail(SSD_CONFIG, "mailbox: bad peer table");
  for (void* p : E.ipc_opened) cudaIpcCloseMemHandle(p);
  E.ipc_opened.clear();
  E.peers.assign(size_t(n_peers), nullptr);
  for (int i = 0; i < n_peers; ++i) {
    if (i == self) {
      E.peers[size_t(i)] = E.inbox;
      continue;
    }
    cudaIpcMemHandle_t mh;
    std::memcpy(&mh, handles + size_t(i) * SSD_MAILBOX_HANDLE_BYTES, sizeof(mh));
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, mh, cudaIpcMemLazyEnablePeerAccess));
    E.ipc_opened.push_back(p);
    E.peers[size_t(i)] = static_cast<Inbox*>(p);
  }
  if (E.peers_dev) cudaFree(E.peers_dev);
  E.peers_dev = dalloc<Inbox*>(size_t(n_peers));
  h2d(E, E.peers_dev, E.peers.data(), size_t(n_peers) * sizeof(Inbox*));
  // a fresh connection starts from a clean inbox and sequence 0
  CK(cudaMemset(E.inbox, 0, kInboxRows));
  E.seq_base = 0;
  CK(cudaDeviceSynchronize());
  API_END
}

ssd_status ssd_tp_export(ssd_engine* h, uint8_t* handle64) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  if (!E.tp_region) throw Fail(SSD_CONFIG, "tensor parallel: engine created with tp_size 1");
  if (!handle64) throw Fail(SSD_CONFIG, "tensor parallel: null handle buffer");
  cudaIpcMemHandle_t mh;
  CK(cudaIpcGetMemHandle(&mh, E.tp_region));
  std::memcpy(handle64, &mh, sizeof(mh));
  API_END
}

ssd_status ssd_tp_connect(ssd_engine* h, const uint8_t* handles) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  if (!E.tp_region || !handles) throw Fail(SSD_CONFIG, "tensor parallel: not a TP engine");
  for (void* p : E.tp_opened) cudaIpcCloseMemHandle(p);
  E.tp_opened.clear();
  for (int r = 0; r < E.tp_L.T; ++r) {
    if (r == E.T.tp_rank) {
      E.tp_peers.region[r] = E.tp_region;
      continue;
    }
    cudaIpcMemHandle_t mh;
    std::memcpy(&mh, handles + size_t(r) * SSD_MAILBOX_HANDLE_BYTES, sizeof(mh));
    void* p = nullptr;
    CK(cudaIpcOpenMemHandle(&p, mh, cudaIpcMemLazyEnablePeerAccess));
    E.tp_opened.push_back(p);
    E.tp_peers.region[r] = static_cast<char*>(p);
  }
  CK(cudaMemset(E.tp_region, 0, 4096));
  CK(cudaMemset(E.tp_ctl, 0, sizeof(TpCtl)));
  CK(cudaDeviceSynchronize());
  API_END
}

// Branch block of speculator `rank` out of G (contiguous, sizes differ by <= 1).
static void branch_block(int B, int rank, int G, int& lo, int& Bl) {
  lo = int((long long)B * rank / G);
  Bl = int((long long)B * (rank + 1) / G) - lo;
}

static void split_common_checks(Engine& E, const ssd_sim_config* c, int T, int G) {
  validate_cfg(E, c);
  if (G < 1) throw Fail(SSD_CONFIG, "split: at least one speculator");
  if (T < 1 || T > kTpMax) throw Fail(SSD_CONFIG, "split: verifier ranks");
  if (int(E.peers.size()) != T + G)
    throw Fail(SSD_CONFIG, "split: mailbox not connected to T verifier ranks + G speculators");
  if (E.V % 4) throw Fail(SSD_CONFIG, "split: vocabulary must be a multiple of 4");
}

ssd_status ssd_run_ssd_verifier(ssd_engine* h, const int32_t* prompt, int32_t n0, const ssd_sim_config* c,
                                int32_t n_spec, int32_t* out, int64_t cap, int64_t* out_len, int32_t* out_outcomes,
                                ssd_run_stats* stats) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  if (E.role != SSD_ROLE_VERIFIER) throw Fail(SSD_CONFIG, "run_ssd_verifier: engine role is not verifier");
  need(E.T, "run_ssd_verifier");
  const int T = E.T.tp_size;  // a tensor-parallel verifier: every rank verifies, rank 0 answers
  split_common_checks(E, c, T, n_spec);
  const int K = c->lookahead;
  const int64_t R = c->rounds;
  set_history(E, prompt, n0, int(n0 + R * (K + 1) + 2 * K + 2));
  cudaStream_t s = E.sv;
  // VerifierProcess streams: derive_seed(derive_seed(seed, 0x5EED), j) (sim.cpp:323-331)
  reset_state(E, K, n0, R, 0, derive_seed(derive_seed(c->seed, 0x5EED), 0), c, s);
  E.seq_base += int(R) + 2;
  if (n0 > 1) prefill(E, E.T, n0 - 1, nullptr, s);
  int* d_out = dalloc<int>(size_t(2 * R));
  const float* rows = reinterpret_cast<const float*>(reinterpret_cast<const char*>(E.inbox) + kInboxRows);
  E.launches = 0;
  GraphSet gs;
  gs.g.push_back(capture_graph(s, [&] {
    recv_spec_kernel<<<1, 32, 0, s>>>(E.st, E.inbox, rows, E.V);
    verify_round(E, K, c->target_scheme, c->scheme, c->accept_scale, 0, s);
    send_outcome_kernel<<<1, 32, 0, s>>>(E.st, E.peers_dev + T, E.T.tp_rank == 0 ? n_spec : 0, d_out);
    commit_kernel<<<1, 32, 0, s>>>(E.st);
    KCHECK();
    E.launches += 3;
  }));
  const long long per_round = E.launches;
  CK(cudaStreamSynchronize(s));
  CK(cudaEventRecord(E.ev_t0, s));
  for (int64_t r = 0; r < R; ++r) CK(cudaGraphLaunch(gs.g[0], s));
  CK(cudaEventRecord(E.ev_t1, s));
  CK(cudaStreamSynchronize(s));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, E.ev_t0, E.ev_t1));
  LoopState st = read_state(E);
  if (out_outcomes) d2h(E, out_outcomes, d_out, size_t(2 * R) * 4);
  cudaFree(d_out);
  if (st.error == 10) {
    Inbox ib;
    d2h(E, &ib, E.inbox, sizeof(Inbox));
    throw Fail(SSD_PROTOCOL_VIOLATION, "verifier: speculation message missing or out of order at round " +
                                           std::to_string(st.round) + " (want seq " +
                                           std::to_string(st.seq_base + st.round + 1) + ", inbox seq " +
                                           std::to_string(ib.d2v.seq) + ")");
  }
  raise_device_error(st);
  fill_stats(st, R, ms, per_round * R, stats);
  copy_out(E, n0, st.n, out, cap, out_len);
  API_END
}

ssd_status ssd_run_ssd_speculator(ssd_engine* h, const int32_t* prompt, int32_t n0, const ssd_sim_config* c,
                                  int32_t rank, int32_t n_spec, int32_t n_verifiers, int32_t* out_hits,
                                  ssd_run_stats* stats) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  if (E.role != SSD_ROLE_SPECULATOR) throw Fail(SSD_CONFIG, "run_ssd_speculator: engine role is not speculator");
  need(E.D, "run_ssd_speculator");
  const int T = n_verifiers;
  split_common_checks(E, c, T, n_spec);
  if (rank < 0 || rank >= n_spec) throw Fail(SSD_CONFIG, "run_ssd_speculator: rank out of range");
  const int K = c->lookahead;
  int B = 0, max_f = 0;
  upload_plans(E, c->primary_plan, c->backup_plan, K, B, max_f);
  int lo = 0, Bl = 0;
  branch_block(B, rank, n_spec, lo, Bl);
  const int64_t R = c->rounds;
  set_history(E, prompt, n0, int(n0 + R * (K + 1) + 2 * K + 2));
  int* d_hit = dalloc<int>(size_t(R));
  cudaStream_t s = E.sv;
  // DraftProcess streams: derive_seed(seed, j) (sim.cpp:376-386); identical on every speculator
  reset_state(E, K, n0, R, derive_seed(c->seed, 0), 0, c, s);
  {  // every message of earlier runs counts as consumed (credit flow control, split.cuh)
    const int run_base = E.seq_base;
    CK(cudaMemcpyAsync(&E.inbox->credit.done, &run_base, sizeof(int), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  }
  E.seq_base += int(R) + 2;
  if (n0 > 1) prefill(E, E.D, n0 - 1, nullptr, s);
  Inbox** vpeers = E.peers_dev;  // [0..T) verifier ranks, [T..T+G) speculators
  // (the verification's sanity checks read the draft rows in every mode, so
  // the message always carries them)
  const int with_rows = 1;
  const int send_blocks = 2 * E_num_sms;
  // initial synchronous draft, clock starts at T_p (sim.cpp:524-526)
  draft_steps(E, K, c->scheme, 0, 0, s);
  {
    LoopState tmp;
    tmp.clock = c->primary_time;
    CK(cudaMemcpyAsync(reinterpret_cast<char*>(E.st) + offsetof(LoopState, clock), &tmp.clock, sizeof(double),
                       cudaMemcpyHostToDevice, s));
  }
  send_spec_kernel<<<send_blocks, 256, 0, s>>>(E.st, vpeers, T, n_spec, rank, E.V, 1, E.send_counter, with_rows);
  KCHECK();
  const bool jit = c->backup_kind == 0;
  E.launches = 0;
  GraphSet gs;
  for (int parity = 0; parity < 2; ++parity) {
    gs.g.push_back(capture_graph(s, [&] {
      prespeculate(E, K, B, lo, Bl, max_f, c->scheme, parity, s);
      recv_outcome_kernel<<<1, 32, 0, s>>>(E.st, E.inbox, E.hist);
      lookup_kernel<<<1, 32, 0, s>>>(E.st, 1, E.keys, max_f, E.offs, E.bt, E.brows[parity], lo, Bl, 0, E.V, E.cum, nullptr,
                                     d_hit, 0, TrLog{nullptr, nullptr, 0});
      send_spec_kernel<<<send_blocks, 256, 0, s>>>(E.st, vpeers, T, n_spec, rank, E.V, 0, E.send_counter, with_rows);
      recv_peer_spec_kernel<<<1, 32, 0, s>>>(E.st, E.inbox);
      KCHECK();
      E.launches += 4;
    }));
  }
  const long long per_round = E.launches / 2;
  long long jit_launches = 0;
  CK(cudaStreamSynchronize(s));
  CK(cudaEventRecord(E.ev_t0, s));
  for (int64_t r = 0; r < R; ++r) {
    CK(cudaGraphLaunch(gs.g[size_t(r & 1)], s));
    if (jit && r + 1 < R) {
      CK(cudaStreamSynchronize(s));
      int hit = 0;
      d2h(E, &hit, reinterpret_cast<char*>(E.st) + offsetof(LoopState, hit), sizeof(int));
      if (!hit) {  // SamePrimaryJIT re-draft (sim.cpp:229-232), identical on every speculator; rank 0 sends
        const long long before = E.launches;
        draft_steps(E, K, c->scheme, 1, 2, s);
        send_spec_kernel<<<send_blocks, 256, 0, s>>>(E.st, vpeers, T, n_spec, rank, E.V, 1, E.send_counter, with_rows);
        KCHECK();
        jit_launches += E.launches - before + 1;
      }
    }
  }
  CK(cudaEventRecord(E.ev_t1, s));
  CK(cudaStreamSynchronize(s));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, E.ev_t0, E.ev_t1));
  LoopState st = read_state(E);
  if (out_hits) d2h(E, out_hits, d_hit, size_t(R) * 4);
  cudaFree(d_hit);
  if (st.error == 10) {
    Inbox ib;
    d2h(E, &ib, E.inbox, sizeof(Inbox));
    throw Fail(SSD_PROTOCOL_VIOLATION,
               "speculator " + std::to_string(rank) + ": message missing or out of order at round " +
                   std::to_string(st.round) + " (base " + std::to_string(st.seq_base) + ", hit " +
                   std::to_string(st.hit) + ", own " + std::to_string(st.own) + ", v2d seq " +
                   std::to_string(ib.v2d[0].seq) + "/" + std::to_string(ib.v2d[1].seq) + ", peer seq " +
                   std::to_string(ib.peer[0].seq) + "/" + std::to_string(ib.peer[1].seq) + ")");
  }
  raise_device_error(st);
  fill_stats(st, R, ms, per_round * R + jit_launches, stats);
  API_END
}

ssd_status ssd_logits(ssd_engine* h, int32_t which, const int32_t* ctx, int32_t n, float* out) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  Model& m = which == 0 ? E.T : E.D;
  need(m, "logits");
  set_history(E, ctx, n, n + 1);
  prefill(E, m, n, E.tlogits, E.sv);
  CK(cudaStreamSynchronize(E.sv));
  d2h(E, out, E.tlogits, size_t(E.V) * 4);
  API_END
}

ssd_status ssd_draft(ssd_engine* h, const int32_t* ctx, int32_t n, int32_t K, const ssd_scheme* sc, uint64_t seed,
                     int32_t* out_tokens, float* out_rows) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  need(E.D, "draft");
  if (K < 1) throw Fail(SSD_ERROR, "draft: lookahead must be >= 1");
  if (K > E.maxK) throw Fail(SSD_TOO_LARGE, "draft: lookahead exceeds the engine's capacity");
  if (!sc) throw Fail(SSD_CONFIG, "draft: scheme required");
  check_scheme(*sc, E.V);
  set_history(E, ctx, n, n + K + 1);
  cudaStream_t s = E.sv;
  reset_state(E, K, n, 1, seed, 0, nullptr, s);
  if (n > 1) prefill(E, E.D, n - 1, nullptr, s);
  draft_steps(E, K, *sc, 0, 0, s);
  CK(cudaStreamSynchronize(s));
  LoopState st = read_state(E);
  std::memcpy(out_tokens, st.spec, size_t(K) * 4);
  if (out_rows) d2h(E, out_rows, E.dmain, size_t(K) * E.V * 4);
  API_END
}

ssd_status ssd_build_cache(ssd_engine* h, const int32_t* ctx, int32_t n, const int32_t* spec, int32_t K,
                           const ssd_plan* plan, const ssd_scheme* sc, int32_t next_K, uint64_t seed, int32_t* out_keys,
                           int32_t* out_entry_tokens, int32_t* out_count) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  need(E.D, "build_cache");
  if (!plan || !sc) throw Fail(SSD_CONFIG, "build_cache: plan and scheme required");
  if (plan->lookahead != K) throw Fail(SSD_ERROR, "build_cache: plan length does not match speculation");
  if (next_K != K) throw Fail(SSD_CONFIG, "build_cache: the engine drafts continuations of the same lookahead");
  if (K < 1 || K > E.maxK) throw Fail(SSD_TOO_LARGE, "build_cache: lookahead exceeds the engine's capacity");
  check_scheme(*sc, E.V);
  int B = 0, max_f = 0;
  upload_plans(E, *plan, *plan, K, B, max_f);
  int total = 0;
  for (int k = 0; k <= K; ++k) total += plan->fan_out[k];
  set_history(E, ctx, n, n + 2 * K + 2);
  for (int i = 0; i < K; ++i)
    if (spec[i] < 0 || spec[i] >= E.V) throw Fail(SSD_ERROR, "context_index: token out of range");
  cudaStream_t s = E.sv;
  reset_state(E, K, n, 1, seed, 0, nullptr, s);
  {
    int tmp[kMaxK + 1];
    std::memcpy(tmp, spec, size_t(K) * 4);
    CK(cudaMemcpyAsync(reinterpret_cast<char*>(E.st) + offsetof(LoopState, spec), tmp, size_t(K) * 4,
                       cudaMemcpyHostToDevice, s));
    const int origin = plan->role;
    CK(cudaMemcpyAsync(reinterpret_cast<char*>(E.st) + offsetof(LoopState, spec_origin), &origin, 4,
                       cudaMemcpyHostToDevice, s));
  }
  if (n > 1) prefill(E, E.D, n - 1, nullptr, s);
  if (total > 0) prespeculate(E, K, B, 0, B, max_f, *sc, 0, s);
  else branch_streams_kernel<<<1, 32, 0, s>>>(E.st, 0, E.bu, 0);
  CK(cudaStreamSynchronize(s));
  std::vector<int> bkh(static_cast<size_t>(B)), bth(static_cast<size_t>(B)), tt(static_cast<size_t>(B) * K);
  d2h(E, bkh.data(), E.bk, size_t(B) * 4);
  d2h(E, bth.data(), E.btok, size_t(B) * 4);
  d2h(E, tt.data(), E.bt, size_t(B) * K * 4);
  for (int i = 0; i < total; ++i) {
    if (out_keys) { out_keys[2 * i] = bkh[size_t(i)]; out_keys[2 * i + 1] = bth[size_t(i)]; }
    if (out_entry_tokens) std::memcpy(out_entry_tokens + size_t(i) * K, &tt[size_t(i) * K], size_t(K) * 4);
  }
  if (out_count) *out_count = total;
  API_END
}

static_assert(sizeof(ssd_rng_stream) == sizeof(Mt64), "ssd_rng_stream mirrors the device stream");

void ssd_rng_stream_seed(ssd_rng_stream* s, uint64_t seed) { mt_seed(*reinterpret_cast<Mt64*>(s), seed); }
uint64_t ssd_rng_stream_next_u64(ssd_rng_stream* s) { return mt_next(*reinterpret_cast<Mt64*>(s)); }
double ssd_rng_stream_next_uniform(ssd_rng_stream* s) { return mt_unit(*reinterpret_cast<Mt64*>(s)); }
uint64_t ssd_derive_seed(uint64_t root, uint64_t index) { return derive_seed(root, index); }

// The caller's stream into / out of lane 0's draft stream (the single stream
// of draft / verify / build_cache calls).
static void put_stream(Engine& E, const ssd_rng_stream* r) {
  if (!r) throw Fail(SSD_CONFIG, "rng stream required");
  h2d(E, &E.st->drng, r, sizeof(Mt64));
}
static void get_stream(Engine& E, ssd_rng_stream* r) { d2h(E, r, &E.st->drng, sizeof(Mt64)); }

static void check_tokens(const int32_t* t, int n, int V, const char* what) {
  if (n > 0 && !t) throw Fail(SSD_CONFIG, std::string(what) + ": null tokens");
  for (int i = 0; i < n; ++i)
    if (t[i] < 0 || t[i] >= V) throw Fail(SSD_ERROR, "context_index: token out of range");
}

ssd_status ssd_draft_stream(ssd_engine* h, const int32_t* ctx, int32_t n, int32_t K, const ssd_scheme* sc,
                            ssd_rng_stream* rng, int32_t* out_tokens, float* out_rows) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  need(E.D, "draft");
  if (K < 1) throw Fail(SSD_ERROR, "draft: lookahead must be >= 1");
  if (K > E.maxK) throw Fail(SSD_TOO_LARGE, "draft: lookahead exceeds the engine's capacity");
  if (!sc || !out_tokens) throw Fail(SSD_CONFIG, "draft: scheme and output required");
  check_scheme(*sc, E.V);
  set_history(E, ctx, n, n + K + 1);
  cudaStream_t s = E.sv;
  reset_state(E, K, n, 1, 0, 0, nullptr, s);
  put_stream(E, rng);
  if (n > 1) prefill(E, E.D, n - 1, nullptr, s);
  draft_steps(E, K, *sc, 0, 0, s);
  CK(cudaStreamSynchronize(s));
  const LoopState st = read_state(E);
  std::memcpy(out_tokens, st.spec, size_t(K) * 4);
  if (out_rows) d2h(E, out_rows, E.dmain, size_t(K) * E.V * 4);
  get_stream(E, rng);
  API_END
}

ssd_status ssd_verify(ssd_engine* h, const int32_t* ctx, int32_t n, const int32_t* spec, int32_t K,
                      const float* spec_rows, const ssd_scheme* ds, const ssd_scheme* ts, double scale,
                      ssd_rng_stream* rng, int32_t* accepted, int32_t* bonus, int32_t* emitted) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  need(E.T, "verify");
  if (K < 1) throw Fail(SSD_ERROR, "verify: empty speculation");
  if (K > E.maxK) throw Fail(SSD_TOO_LARGE, "verify: lookahead exceeds the engine's capacity");
  if (!ds || !ts || !accepted || !bonus) throw Fail(SSD_CONFIG, "verify: schemes and outputs required");
  if (!(scale > 0.0) || scale > 1.0) throw Fail(SSD_ERROR, "verify: accept_scale must be in (0, 1]");
  check_scheme(*ds, E.V);
  check_scheme(*ts, E.V);
  check_tokens(spec, K, E.V, "verify");
  set_history(E, ctx, n, n + K + 2);
  cudaStream_t s = E.sv;
  reset_state(E, K, n, 1, 0, 0, nullptr, s);
  put_stream(E, rng);
  {
    int tmp[kMaxK];
    std::memcpy(tmp, spec, size_t(K) * 4);
    h2d(E, reinterpret_cast<char*>(E.st) + offsetof(LoopState, spec), tmp, size_t(K) * 4);
  }
  if (spec_rows) {
    h2d(E, E.dmain, spec_rows, size_t(K) * E.V * 4);
    set_spec_rows_kernel<<<1, 32, 0, s>>>(E.st, E.dmain, E.V, 0, 0);
    KCHECK();
  } else {
    const int one = 1;
    h2d(E, reinterpret_cast<char*>(E.st) + offsetof(LoopState, spec_uniform), &one, 4);
  }
  if (n > 1) prefill(E, E.T, n - 1, nullptr, s);
  verify_round(E, K, *ts, *ds, scale, /*the caller's stream*/ 1, s);
  CK(cudaStreamSynchronize(s));
  const LoopState st = read_state(E);
  raise_device_error(st);
  *accepted = st.out_k;
  *bonus = st.out_t;
  if (emitted) d2h(E, emitted, E.hist + n, size_t(st.out_k + 1) * 4);
  get_stream(E, rng);
  API_END
}

// Shared by the synchronous and asynchronous build_cache: plan upload and
// capacity checks; returns the entry count.
static int prespec_setup(Engine& E, const ssd_plan* plan, const ssd_scheme* sc, int K, int next_K, int& B,
                         int& max_f) {
  need(E.D, "build_cache");
  if (!plan || !sc) throw Fail(SSD_CONFIG, "build_cache: plan and scheme required");
  if (plan->lookahead != K) throw Fail(SSD_ERROR, "build_cache: plan length does not match speculation");
  if (K < 1 || K > E.maxK) throw Fail(SSD_TOO_LARGE, "build_cache: lookahead exceeds the engine's capacity");
  if (next_K < 1) throw Fail(SSD_ERROR, "build_cache: next_lookahead must be >= 1");
  if (next_K > E.maxK) throw Fail(SSD_TOO_LARGE, "build_cache: next_lookahead exceeds the engine's capacity");
  check_scheme(*sc, E.V);
  upload_plans(E, *plan, *plan, K, B, max_f);
  int total = 0;
  for (int k = 0; k <= K; ++k) total += plan->fan_out[k];
  return total;
}

ssd_status ssd_build_cache_stream(ssd_engine* h, const int32_t* ctx, int32_t n, const int32_t* spec, int32_t K,
                                  const ssd_plan* plan, const ssd_scheme* sc, int32_t next_K, ssd_rng_stream* rng,
                                  int32_t* out_keys, int32_t* out_entry_tokens, float* out_entry_rows,
                                  int32_t* out_count) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  int B = 0, max_f = 0;
  const int total = prespec_setup(E, plan, sc, K, next_K, B, max_f);
  check_tokens(spec, K, E.V, "build_cache");
  set_history(E, ctx, n, n + K + next_K + 2);
  cudaStream_t s = E.sv;
  reset_state(E, K, n, 1, 0, 0, nullptr, s);
  put_stream(E, rng);
  {
    int tmp[kMaxK + 1];
    std::memcpy(tmp, spec, size_t(K) * 4);
    h2d(E, reinterpret_cast<char*>(E.st) + offsetof(LoopState, spec), tmp, size_t(K) * 4);
    const int origin = plan->role;
    h2d(E, reinterpret_cast<char*>(E.st) + offsetof(LoopState, spec_origin), &origin, 4);
    h2d(E, reinterpret_cast<char*>(E.st) + offsetof(LoopState, Kb), &next_K, 4);
  }
  if (n > 1) prefill(E, E.D, n - 1, nullptr, s);
  if (total > 0) prespeculate(E, K, B, 0, B, max_f, *sc, 0, s, 1, nullptr, next_K);
  else branch_streams_kernel<<<1, 32, 0, s>>>(E.st, 0, E.bu, 0);  // the one next_u64 (cache.cpp:245)
  KCHECK();
  CK(cudaStreamSynchronize(s));
  std::vector<int> bkh(static_cast<size_t>(B)), bth(static_cast<size_t>(B)), tt(static_cast<size_t>(B) * next_K);
  d2h(E, bkh.data(), E.bk, size_t(B) * 4);
  d2h(E, bth.data(), E.btok, size_t(B) * 4);
  d2h(E, tt.data(), E.bt, size_t(B) * next_K * 4);
  for (int i = 0; i < total; ++i) {
    if (out_keys) { out_keys[2 * i] = bkh[size_t(i)]; out_keys[2 * i + 1] = bth[size_t(i)]; }
    if (out_entry_tokens) std::memcpy(out_entry_tokens + size_t(i) * next_K, &tt[size_t(i) * next_K], size_t(next_K) * 4);
    if (out_entry_rows)
      for (int j = 0; j < next_K; ++j)  // branch rows are [j][B][V]
        d2h(E, out_entry_rows + (size_t(i) * next_K + j) * E.V, E.brows[0] + (size_t(j) * B + i) * E.V,
            size_t(E.V) * 4);
  }
  if (out_count) *out_count = total;
  get_stream(E, rng);
  API_END
}

ssd_status ssd_prespec_begin(ssd_engine* h, const int32_t* d_ctx, int32_t n, const int32_t* d_spec, int32_t K,
                             const ssd_plan* plan, const ssd_scheme* sc, int32_t next_K, ssd_rng_stream* rng,
                             void* cuda_stream) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  if (!d_ctx || !d_spec || n < 1) throw Fail(SSD_ERROR, "prespec_begin: context and speculation required");
  if (!rng) throw Fail(SSD_CONFIG, "rng stream required");
  if (E.pre_active) CK(cudaEventSynchronize(E.ev_prespec));  // the previous session's buffers are reused
  int B = 0, max_f = 0;
  const int total = prespec_setup(E, plan, sc, K, next_K, B, max_f);
  const int cap = std::min(E.T.s.max_ctx, E.D.s.max_ctx);
  if (n + K + next_K + 2 > cap) throw Fail(SSD_TOO_LARGE, "context exceeds max_ctx");
  E.D.ctx_bound = n + K + next_K + 2 + 2 * E.maxK;
  cudaStream_t s = E.sv;
  if (cuda_stream) {  // ordered after the caller's producer of d_ctx / d_spec
    CK(cudaEventRecord(E.ev_user, static_cast<cudaStream_t>(cuda_stream)));
    CK(cudaStreamWaitEvent(s, E.ev_user, 0));
  }
  // the device stream starts from the caller's state; the host copy takes the
  // same one draw (cache.cpp:245), so both stay in step without a sync
  std::memcpy(E.pin_rng, rng, sizeof(Mt64));
  ssd_rng_stream_next_u64(rng);
  reset_state(E, K, n, 1, 0, 0, nullptr, s);
  CK(cudaMemcpyAsync(&E.st->drng, E.pin_rng, sizeof(Mt64), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(E.hist, d_ctx, size_t(n) * 4, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(reinterpret_cast<char*>(E.st) + offsetof(LoopState, spec), d_spec, size_t(K) * 4,
                     cudaMemcpyDeviceToDevice, s));
  set_spec_origin_kernel<<<1, 32, 0, s>>>(E.st, plan->role, next_K);
  KCHECK();
  if (n > 1) prefill(E, E.D, n - 1, nullptr, s);
  if (total > 0) prespeculate(E, K, B, 0, B, max_f, *sc, 0, s, 1, nullptr, next_K);
  CK(cudaEventRecord(E.ev_prespec, s));
  E.pre_active = 1;
  E.pre_count = total;
  E.pre_kb = next_K;
  E.pre_keys_valid = 0;
  API_END
}

static void prespec_wait(Engine& E) {
  if (!E.pre_active) throw Fail(SSD_CONFIG, "cache: no pre-speculation started (ssd_prespec_begin)");
  CK(cudaEventSynchronize(E.ev_prespec));
  if (E.pre_keys_valid) return;
  const int n = E.pre_count;
  std::vector<int> bk(static_cast<size_t>(std::max(n, 1))), bt(static_cast<size_t>(std::max(n, 1)));
  d2h(E, bk.data(), E.bk, size_t(n) * 4);
  d2h(E, bt.data(), E.btok, size_t(n) * 4);
  E.pre_keys.assign(size_t(2 * n), 0);
  for (int i = 0; i < n; ++i) { E.pre_keys[size_t(2 * i)] = bk[size_t(i)]; E.pre_keys[size_t(2 * i + 1)] = bt[size_t(i)]; }
  LoopState st = read_state(E);
  raise_device_error(st);
  E.pre_keys_valid = 1;
}

ssd_status ssd_cache_lookup(ssd_engine* h, int32_t k, int32_t t, int32_t* slot) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  if (!slot) throw Fail(SSD_CONFIG, "cache_lookup: null output");
  prespec_wait(E);
  *slot = -1;
  for (int i = 0; i < E.pre_count; ++i)
    if (E.pre_keys[size_t(2 * i)] == k && E.pre_keys[size_t(2 * i + 1)] == t) { *slot = i; break; }
  API_END
}

ssd_status ssd_cache_keys(ssd_engine* h, int32_t* out_keys, int32_t* out_count) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  prespec_wait(E);
  if (out_keys) std::memcpy(out_keys, E.pre_keys.data(), E.pre_keys.size() * 4);
  if (out_count) *out_count = E.pre_count;
  API_END
}

ssd_status ssd_cache_entry(ssd_engine* h, int32_t slot, int32_t* out_tokens, float* out_rows) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  prespec_wait(E);
  if (slot < 0 || slot >= E.pre_count) throw Fail(SSD_ERROR, "cache_entry: slot out of range");
  const int Kb = E.pre_kb, B = E.pre_count;
  if (out_tokens) d2h(E, out_tokens, E.bt + size_t(slot) * Kb, size_t(Kb) * 4);
  if (out_rows)
    for (int j = 0; j < Kb; ++j) d2h(E, out_rows + size_t(j) * E.V, E.brows[0] + (size_t(j) * B + slot) * E.V, size_t(E.V) * 4);
  API_END
}

ssd_status ssd_topk_keys(ssd_engine* h, const float* rows, int32_t n_rows, int32_t V, const int32_t* fan,
                         const int32_t* excluded, int32_t max_f, int32_t* keys) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  if (n_rows < 1 || n_rows > E.maxK + 1 || V > E.V || V < 1) throw Fail(SSD_TOO_LARGE, "topk_keys: shape exceeds capacity");
  if (max_f > kMaxTopF) throw Fail(SSD_TOO_LARGE, "topk_keys: fan-out above capacity");
  std::vector<int> fan2(size_t(2 * n_rows)), off2(size_t(2 * n_rows));
  int tot = 0;
  for (int k = 0; k < n_rows; ++k) {
    if (fan[k] > max_f || fan[k] >= kMaxTopF) throw Fail(SSD_TOO_LARGE, "topk_keys: fan-out above capacity");
    fan2[size_t(k)] = fan2[size_t(n_rows + k)] = fan[k];
    off2[size_t(k)] = off2[size_t(n_rows + k)] = tot;
    tot += fan[k];
  }
  if (tot > E.maxB) throw Fail(SSD_TOO_LARGE, "topk_keys: too many candidates");
  h2d(E, E.plans, fan2.data(), fan2.size() * 4);
  h2d(E, E.offs, off2.data(), off2.size() * 4);
  h2d(E, E.xrows, rows, size_t(n_rows) * V * 4);
  h2d(E, E.tok_scratch, excluded, size_t(n_rows) * 4);
  row_keys(E, E.xrows, n_rows, V, max_f, nullptr, E.tok_scratch, n_rows, E.sv);
  CK(cudaStreamSynchronize(E.sv));
  d2h(E, keys, E.keys, size_t(n_rows) * max_f * 4);
  API_END
}

ssd_status ssd_verify_rows(ssd_engine* h, const float* trows, const float* drows, const int32_t* tokens, int32_t K,
                           int32_t V, const ssd_scheme* ds, const ssd_scheme* ts, double scale, uint64_t seed,
                           int32_t* accepted, int32_t* bonus) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  if (K < 1) throw Fail(SSD_ERROR, "verify: empty speculation");
  if (K > E.maxK || V != E.V) throw Fail(SSD_TOO_LARGE, "verify_rows: shape exceeds capacity");
  check_scheme(*ds, V);
  check_scheme(*ts, V);
  for (int i = 0; i < K; ++i)
    if (tokens[i] < 0 || tokens[i] >= V) throw Fail(SSD_ERROR, "verify: token out of range");
  cudaStream_t s = E.sv;
  h2d(E, E.tlogits, trows, size_t(K + 1) * V * 4);
  if (drows) h2d(E, E.dmain, drows, size_t(K) * V * 4);
  std::vector<int> hist0(1, 0);
  h2d(E, E.hist, hist0.data(), 4);
  reset_state(E, K, 1, 1, 0, seed, nullptr, s);
  {
    int tmp[kMaxK];
    std::memcpy(tmp, tokens, size_t(K) * 4);
    CK(cudaMemcpyAsync(reinterpret_cast<char*>(E.st) + offsetof(LoopState, spec), tmp, size_t(K) * 4,
                       cudaMemcpyHostToDevice, s));
  }
  if (drows) set_spec_rows_kernel<<<1, 32, 0, s>>>(E.st, E.dmain, V, 0, 0);
  else {
    const int one = 1;
    CK(cudaMemcpyAsync(reinterpret_cast<char*>(E.st) + offsetof(LoopState, spec_uniform), &one, 4,
                       cudaMemcpyHostToDevice, s));
  }
  verify_stats_kernel<<<2 * K + 1, kSampleThreads, 0, s>>>(E.tlogits, E.st, V, dscheme(*ts), dscheme(*ds), E.rstat);
  verify_decide_kernel<<<1, kSampleThreads, 0, s>>>(E.tlogits, E.st, E.hist, V, dscheme(*ts), dscheme(*ds), scale, E.rstat, 0,
                                                    E.hist_stride);
  KCHECK();
  CK(cudaStreamSynchronize(s));
  LoopState st = read_state(E);
  raise_device_error(st);
  *accepted = st.out_k;
  *bonus = st.out_t;
  API_END
}

ssd_status ssd_profile_forward(ssd_engine* h, int32_t which, int32_t M, int32_t pos, int32_t iters, double* ms_forward,
                               double* ms_gemm, int64_t* gemm_bytes, int32_t* gemm_launches) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  Model& m = which == 0 ? E.T : E.D;
  need(m, "profile_forward");
  if (M < 1 || M > m.maxM || pos + M > m.s.max_ctx || iters < 1) throw Fail(SSD_TOO_LARGE, "profile: bad shape");
  // SSD_B200_PROFILE_PART=v|s: on the verifier / speculator partition of
  // the colocated round (its green stream and GEMM grid cap); the timing
  // events stay on the ordinary stream (joined through events)
  cudaStream_t s = E.sv;
  if (const char* pp = std::getenv("SSD_B200_PROFILE_PART"); pp && E.gsv && (pp[0] == 'v' || pp[0] == 's')) {
    s = pp[0] == 'v' ? E.gsv : E.gss;
    m.gemm_ctas = pp[0] == 'v' ? E.green_v : E.green_s;
  }
  struct Uncap {
    Model& m;
    ~Uncap() { m.gemm_ctas = 0; }
  } uncap{m};
  auto t_begin = [&] {
    CK(cudaEventRecord(E.ev_t0, E.sv));
    CK(cudaStreamWaitEvent(s, E.ev_t0, 0));
  };
  auto t_end = [&] {
    CK(cudaEventRecord(E.ev_join, s));
    CK(cudaStreamWaitEvent(E.sv, E.ev_join, 0));
    CK(cudaEventRecord(E.ev_t1, E.sv));
    CK(cudaEventSynchronize(E.ev_t1));
  };
  m.ctx_bound = pos + M + 1;
  prep_prefill_kernel<<<1, kMaxM, 0, s>>>(E.hist, E.P_pre, pos, M, 0, m.km);
  KCHECK();
  const ssd_model_shape& sh = m.s;
  const int d = sh.d_model, F = sh.ffn, nqkv = m.qd + 2 * m.kvd;
  const int fused = (!E.deterministic && m.tp_size == 1) ? 1 : 0;
  auto gemms = [&]() {  // (QKV accumulates into whatever qkv holds: timing only)
    PfCursor pf(m, E.pf_ahead, true);
    for (int l = 0; l < sh.n_layers; ++l) {
      const DevLayer& L = m.layers[size_t(l)];
      linear<EPI_STORE>(E, m, L.qkv, m.xb, M, m.qkv, nqkv, nullptr, 0, s, pf.after(4 * l), fused);
      if (fused) linear<EPI_RESID>(E, m, L.o, m.attn, M, m.x, d, nullptr, 0, s, pf.after(4 * l + 1), 1);
      else linear<EPI_STORE>(E, m, L.o, m.attn, M, m.dlt1, d, nullptr, 0, s, pf.after(4 * l + 1));
      linear<EPI_SWIGLU>(E, m, L.gu, m.xb, M, nullptr, 0, m.act, F, s, pf.after(4 * l + 2));
      if (fused) linear<EPI_RESID>(E, m, L.dn, m.act, M, m.x, d, nullptr, 0, s, pf.after(4 * l + 3), 1);
      else linear<EPI_STORE>(E, m, L.dn, m.act, M, m.dlt2, d, nullptr, 0, s, pf.after(4 * l + 3));
    }
    linear<EPI_STORE>(E, m, m.head, m.xb, M, m.logits, sh.vocab, nullptr, 0, s, pf.after(4 * sh.n_layers));
  };
  forward(E, m, E.P_pre, M, m.logits, s);  // warm
  gemms();
  t_begin();
  for (int i = 0; i < iters; ++i) forward(E, m, E.P_pre, M, m.logits, s);
  t_end();
  float f_ms = 0.f;
  CK(cudaEventElapsedTime(&f_ms, E.ev_t0, E.ev_t1));
  t_begin();
  for (int i = 0; i < iters; ++i) gemms();
  t_end();
  float g_ms = 0.f;
  CK(cudaEventElapsedTime(&g_ms, E.ev_t0, E.ev_t1));
  *ms_forward = f_ms / iters;
  *ms_gemm = g_ms / iters;
  // algorithmic bytes: every weight once + bf16 activations in + fp32 out
  const int64_t act = int64_t(M) * (int64_t(sh.n_layers) * (2LL * d + 2LL * m.qd + 2LL * d + 2LL * F +
                                                              4LL * nqkv + 8LL * d + 2LL * F + 8LL * d) +
                                    2LL * d + 4LL * sh.vocab);
  *gemm_bytes = m.weight_bytes + act;
  *gemm_launches = 4 * sh.n_layers + 1;
  API_END
}

ssd_status ssd_bench_read_bw(ssd_engine* h, int64_t bytes, int32_t iters, double* gbs) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  const size_t n = size_t(bytes) / 16;
  uint4* buf = dalloc<uint4>(n);
  uint4* sink = dalloc<uint4>(1);
  int sms = E_num_sms;
  read_bw_kernel<<<sms * 8, 512, 0, E.sv>>>(buf, n, sink);
  CK(cudaEventRecord(E.ev_t0, E.sv));
  for (int i = 0; i < iters; ++i) read_bw_kernel<<<sms * 8, 512, 0, E.sv>>>(buf, n, sink);
  CK(cudaEventRecord(E.ev_t1, E.sv));
  CK(cudaEventSynchronize(E.ev_t1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, E.ev_t0, E.ev_t1));
  *gbs = double(n) * 16.0 * iters / (ms * 1e-3) / 1e9;
  cudaFree(buf);
  cudaFree(sink);
  API_END
}


// ------------------------------------------------------------- paged KV
// the engine's main caches as pages of page_tokens slots
// (page p = page p % ppl of lane p / ppl's main region, ppl = max_ctx /
// page_tokens, the same page index in the target and the draft arena). A
// lane's block table maps its logical pages to these; csrc/paged.cpp's pool
// decides them (ssd_kv_seq_admit / reserve / commit).
static int kv_ppl(const Engine& E, int pt) {
  int ctx = 1 << 30;
  for (const Model* m : {&E.T, &E.D})
    if (m->kc) ctx = std::min(ctx, m->s.max_ctx);
  if (pt < 1 || (pt & (pt - 1)) || ctx % pt) throw Fail(SSD_CONFIG, "paged KV: page_tokens must be a power of two dividing max_ctx");
  return ctx / pt;
}

ssd_status ssd_engine_kv_pages(ssd_engine* h, int32_t page_tokens, int32_t* n_pages) {
  API_BEGIN
  Engine& E = h->e;
  if (!n_pages) throw Fail(SSD_CONFIG, "kv pages: null output");
  *n_pages = E.nbmax * kv_ppl(E, page_tokens);
  API_END
}

ssd_status ssd_engine_set_block_table(ssd_engine* h, int32_t lane, const int32_t* pages, int32_t n, int32_t page_tokens,
                                      int32_t cached_tokens) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  const int ppl = kv_ppl(E, page_tokens);
  if (lane < 0 || lane >= E.nbmax) throw Fail(SSD_CONFIG, "block table: lane out of range");
  if (n < 0 || n > ppl || (n > 0 && !pages)) throw Fail(SSD_TOO_LARGE, "block table: more pages than a lane's main cache");
  if (E.page_tokens && E.page_tokens != page_tokens) throw Fail(SSD_CONFIG, "block table: page_tokens differs from the tables set");
  for (int i = 0; i < n; ++i)
    if (pages[i] < 0 || pages[i] >= E.nbmax * ppl) throw Fail(SSD_CONFIG, "block table: page out of range");
  if (cached_tokens < 0 || cached_tokens > n * page_tokens) throw Fail(SSD_CONFIG, "block table: cached tokens beyond the pages");
  int shift = 0;
  while ((1 << shift) < page_tokens) ++shift;
  for (Model* m : {&E.T, &E.D}) {
    if (!m->kc) continue;
    if (!m->km.tab) {  // identity for every lane
      int* tab = static_cast<int*>(dalloc<int>(size_t(E.nbmax) * ppl));
      m->owned.push_back(tab);
      std::vector<int> id(static_cast<size_t>(E.nbmax) * static_cast<size_t>(ppl));
      for (int l = 0; l < E.nbmax; ++l)
        for (int i = 0; i < ppl; ++i) id[size_t(l) * ppl + i] = l * m->lane_S + i * page_tokens;
      h2d(E, tab, id.data(), id.size() * 4);
      m->km.tab = tab;
    }
    std::vector<int> row(static_cast<size_t>(ppl));
    for (int i = 0; i < ppl; ++i) {
      const int p = i < n ? pages[i] : lane * ppl + i;
      row[size_t(i)] = (p / ppl) * m->lane_S + (p % ppl) * page_tokens;
    }
    h2d(E, const_cast<int*>(m->km.tab) + size_t(lane) * ppl, row.data(), row.size() * 4);
    m->km.shift = shift;
    m->km.lane_S = m->lane_S;
    m->km.ppl = ppl;
  }
  E.page_tokens = page_tokens;
  E.prefill_skip.resize(size_t(E.nbmax), 0);
  E.prefill_skip[size_t(lane)] = cached_tokens;
  E.ssd_graph_key.clear();  // captured graphs bake the (un)paged layout
  API_END
}

ssd_status ssd_engine_clear_block_tables(ssd_engine* h) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  for (Model* m : {&E.T, &E.D}) m->km.tab = nullptr;  // the table allocation stays owned by the model
  E.page_tokens = 0;
  E.prefill_skip.clear();
  E.ssd_graph_key.clear();
  API_END
}

ssd_status ssd_engine_sm_partition(ssd_engine* h, int32_t verifier_sms, int32_t* out_v, int32_t* out_s) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  if (verifier_sms >= 0) {
    CK(cudaDeviceSynchronize());  // no round graph of this engine in flight
    set_green(E, verifier_sms);
  }
  if (out_v) *out_v = E.green_v;
  if (out_s) *out_s = E.green_s;
  API_END
}

#if SSD_GEMM_TRACE
extern "C" int ssd_debug_gemm_trace(unsigned long long* out /* 5 x 512 */) {
  return int(cudaMemcpyFromSymbol(out, tc::g_trace, sizeof(unsigned long long) * 5 * 512));
}
#endif

// Kernel timeline (profiling build -DSSD_KTL=1): copies up to n records
// (kind, entry, ready, exit) and resets the ring; returns the count.
int ssd_debug_ktl(unsigned long long* out, int n) {
#if SSD_KTL
  unsigned cnt = 0;
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  cudaMemcpyFromSymbol(&cnt, g_ktl_n, sizeof(cnt));
  const int m = std::min<int>(n, std::min<unsigned>(cnt, 16384u));
  cudaMemcpyFromSymbol(out, g_ktl, size_t(m) * 4 * sizeof(unsigned long long));
  const unsigned zero = 0;
  cudaMemcpyToSymbol(g_ktl_n, &zero, sizeof(zero));
  if (n >= m + 4) cudaMemcpyFromSymbol(out + size_t(m) * 4, g_ktl_sub, 16 * sizeof(unsigned long long));
  if (n >= m + 4 + 64 * 160 * 8)
    cudaMemcpyFromSymbol(out + size_t(m) * 4 + 16, g_ktl_cta, size_t(64) * 160 * 8 * sizeof(unsigned long long));
  return m;
#else
  (void)out;
  (void)n;
  return -1;
#endif
}

ssd_status ssd_rng_u64(ssd_engine* h, uint64_t seed, int32_t n, uint64_t* out) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  uint64_t* d = dalloc<uint64_t>(size_t(n));
  Mt64* m = dalloc<Mt64>(1);
  mt_init_kernel<<<1, 32, 0, E.sv>>>(m, seed);
  mt_draw_kernel<<<1, 32, 0, E.sv>>>(m, n, d);
  KCHECK();
  d2h(E, out, d, size_t(n) * 8);
  cudaFree(d);
  cudaFree(m);
  API_END
}

ssd_status ssd_weight_bits(ssd_engine* h, int32_t which, int32_t layer, int32_t kind, const int64_t* rows,
                           const int64_t* cols, int32_t n, uint16_t* out) {
  API_BEGIN
  Engine& E = h->e;
  CK(cudaSetDevice(E.dev));
  Model& m = which == 0 ? E.T : E.D;
  const size_t d = size_t(m.s.d_model);
  for (int i = 0; i < n; ++i) {
    const size_t r = size_t(rows[i]), c = size_t(cols[i]);
    const bf16* p = nullptr;
    const size_t kd = d / 64, kq = size_t(m.qd) / 64, kf = size_t(m.s.ffn) / 64;
    if (kind == 100) p = m.embed + (m.embed_tiled ? tiled_at(r, c, kd) : r * d + c);
    else if (kind == 101) p = m.head.w + tiled_at(r, c, kd);
    else {
      if (layer < 0 || layer >= m.s.n_layers) throw Fail(SSD_ERROR, "weight_bits: bad layer");
      const DevLayer& L = m.layers[size_t(layer)];
      switch (kind) {
        case 0: p = L.qkv.w + tiled_at(r, c, kd); break;
        case 1: p = L.qkv.w + tiled_at(size_t(m.qd) + r, c, kd); break;
        case 2: p = L.qkv.w + tiled_at(size_t(m.qd + m.kvd) + r, c, kd); break;
        case 3: p = L.o.w + tiled_at(r, c, kq); break;
        case 4: p = L.gu.w + tiled_at(2 * r, c, kd); break;
        case 5: p = L.gu.w + tiled_at(2 * r + 1, c, kd); break;
        case 6: p = L.dn.w + tiled_at(r, c, kf); break;
        default: throw Fail(SSD_ERROR, "weight_bits: bad kind");
      }
    }
    d2h(E, &out[i], p, 2);
  }
  API_END
}

}  // extern "C"
