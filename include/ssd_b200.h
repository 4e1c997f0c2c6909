/*
 * ssd_b200.h — C-ABI of the B200-native Saguaro (speculative speculative
 * decoding) hot path.
 *
 * This is the drop-in boundary for the reference's speculator / verifier /
 * speculation-cache interfaces (ssd-lab, proj/include/ssdlab). Every entry
 * point names the reference interface it replaces. Plain C types only: no
 * torch, no C++ in the signatures. All device work runs on the engine's own
 * CUDA streams; results are copied back to caller-owned HOST buffers.
 *
 * Errors: every call returns an ssd_status; the codes map one-to-one onto
 * the reference exception hierarchy (errors.hpp:9-61), and ssd_last_error()
 * returns the message of the last failure on the calling thread. The C++
 * shim (include/ssdlab_b200.hpp) re-throws the matching ssdlab:: type.
 *
 * Randomness: the engine reproduces the reference's stream discipline on the
 * device — mt19937_64 streams seeded through derive_seed (rng.hpp:24-48),
 * one uniform per draw, the same consumption order as run_ar / run_sd /
 * run_protocol_harness (sim.cpp:64-121, 502-601) — so outputs can be
 * compared with the CPU oracle stream for stream.
 */
#ifndef SSD_B200_H_
#define SSD_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSD_B200_ABI_VERSION 1
#define SSD_MAX_LOOKAHEAD 16

/* errors.hpp:9-61 (ssdlab::Error and subclasses) */
typedef enum ssd_status {
  SSD_OK = 0,
  SSD_ERROR = 1,                /* ssdlab::Error */
  SSD_ALL_ZERO = 2,             /* AllZeroError */
  SSD_DEGENERATE_RESIDUAL = 3,  /* DegenerateResidualError */
  SSD_TOO_LARGE = 4,            /* TooLargeError */
  SSD_BUDGET_TOO_SMALL = 5,     /* BudgetTooSmallError */
  SSD_DIVERGENT = 6,            /* DivergentError */
  SSD_INSUFFICIENT_DATA = 7,    /* InsufficientDataError */
  SSD_UNREACHABLE = 8,          /* UnreachableError */
  SSD_NO_CROSSOVER = 9,         /* NoCrossoverError */
  SSD_PROTOCOL_VIOLATION = 10,  /* ProtocolViolationError */
  SSD_CONFIG = 11,              /* ConfigError */
  SSD_CUDA = 100                /* CUDA runtime failure (no reference analogue) */
} ssd_status;

const char* ssd_last_error(void);
int ssd_abi_version(void);

/* ---------------------------------------------------------------- types */

/* Llama-style decoder shape. Replaces the reference's model parameter
 * (lm::SyntheticLM, lm.hpp:12-47) with a transformer resident on the GPU. */
typedef struct ssd_model_shape {
  int32_t vocab, d_model, n_layers, n_heads, n_kv_heads, head_dim, ffn;
  int32_t tied;    /* embedding doubles as LM head */
  int32_t max_ctx; /* KV capacity in tokens */
  double rope_theta;
  float norm_eps;
} ssd_model_shape;

/* Correlated random pair; the analogue of
 * lm::derive_draft / calibrate_pair (lm.hpp:55-90). */
typedef struct ssd_pair_params {
  uint64_t seed;
  float embed_scale, shared_mlp_scale, block_out_scale;
  float target_private_embed, target_private_head, draft_gain_mix;
  float logit_scale; /* magnitude of the final RMSNorm gains */
} ssd_pair_params;

/* dist::SamplingScheme (categorical.hpp:43-60). temperature == 0 selects
 * greedy decoding (the tau -> 0 limit; argmax with lowest-index ties). */
typedef struct ssd_scheme {
  int32_t kind; /* 0 = Standard, 1 = Saguaro */
  int32_t fan_out;
  double temperature;
  double downweight;
} ssd_scheme;

/* cache::FanOutPlan (cache.hpp:18-25) */
typedef struct ssd_plan {
  int32_t lookahead;
  int32_t role; /* 0 = Primary, 1 = Backup */
  int32_t budget;
  int32_t fan_out[SSD_MAX_LOOKAHEAD + 1];
} ssd_plan;

/* sim::SimConfig (sim.hpp:28-53), minus the models (owned by the engine). */
typedef struct ssd_sim_config {
  int32_t lookahead;
  ssd_scheme scheme;
  ssd_scheme target_scheme;
  ssd_plan primary_plan;
  ssd_plan backup_plan;
  int32_t backup_kind;  /* 0 = SamePrimaryJIT, 1 = FastRandom (sim.hpp:17-20) */
  double primary_time, backup_time;
  int64_t rounds;
  uint64_t seed;
  double accept_scale;
} ssd_sim_config;

/* sim::RunStats (sim.hpp:55-104) plus measured device time. */
typedef struct ssd_run_stats {
  int64_t rounds, tokens;
  double virtual_time;
  int64_t primary_origin_lookups, primary_origin_hits;
  int64_t backup_origin_lookups, backup_origin_hits;
  int64_t hit_rounds, miss_rounds, initial_rounds;
  int64_t hit_round_tokens, miss_round_tokens;
  double accepted_sum;
  double device_ms;     /* CUDA-event time of the decode loop (prefill excluded) */
  int64_t kernel_launches; /* engine kernels launched inside the timed loop */
} ssd_run_stats;

typedef struct ssd_engine ssd_engine;

/* Process roles of a split run: the reference's
 * VerifierProcess / DraftProcess (sim.cpp:321-485) as separate OS processes
 * on separate GPUs. A verifier materialises only the target, a speculator
 * only the draft. */
typedef enum ssd_role {
  SSD_ROLE_COLOCATED = 0,
  SSD_ROLE_VERIFIER = 1,
  SSD_ROLE_SPECULATOR = 2
} ssd_role;

#define SSD_MAILBOX_HANDLE_BYTES 64

/* ------------------------------------------------- plans (host-only) */

/* cache::geometric_fanout (cache.hpp:57-60, cache.cpp:39-113). */
ssd_status ssd_geometric_fanout(double acceptance, double exponent, int32_t lookahead, int32_t budget,
                                int32_t role, ssd_plan* out);
/* cache::uniform_fanout (cache.hpp:62-64, cache.cpp:115-127). */
ssd_status ssd_uniform_fanout(int32_t lookahead, int32_t budget, int32_t role, ssd_plan* out);
/* cache::conditional_hit_rate (cache.hpp:79-85, cache.cpp:150-169). */
double ssd_conditional_hit_rate(const ssd_plan* plan, double acceptance, double exponent);

/* hitmodel::fit_powerlaw (hitmodel.hpp:39-50, hitmodel.cpp:65-106): fit
 * miss = A F^-r to n measured (fan-out, miss rate) samples by log-log least
 * squares; the exponent r calibrates ssd_geometric_fanout.
 * SSD_INSUFFICIENT_DATA with fewer than two distinct fan-outs. */
ssd_status ssd_fit_powerlaw(const double* fan_out, const double* miss_rate, int32_t n, double* exponent,
                            double* log_amplitude, double* r_squared);
/* perf::speedup_batch (perf.hpp:54-59, perf.cpp:44-55): per-sequence
 * speedup of a batch whose rounds stall for the backup when any sequence
 * misses (all-hit probability hit_rate^batch). Times in verify passes. */
ssd_status ssd_speedup_batch(double hit_rate, double hit_tokens, double miss_tokens, double primary_time,
                             double backup_time, double batch, double* out);
/* perf::critical_batch (perf.hpp:61-72, perf.cpp:57-73): the batch size b*
 * at which the free (FastRandom) backup overtakes the JIT re-draft; the
 * Saguaro fallback policy uses JIT below b*. SSD_NO_CROSSOVER when one
 * strategy dominates at every batch size. */
ssd_status ssd_critical_batch(double hit_rate, double hit_tokens, double miss_tokens, double primary_time,
                              double* out);
/* --------------------------------------------------------------- engine */

/* Materialise the (target, draft) pair on `device` with synthetic weights
 * (bit-identical to the CPU oracle's generator) and allocate KV caches for
 * up to `max_branches` pre-speculation branches. */
ssd_status ssd_engine_create(const ssd_model_shape* target, const ssd_model_shape* draft,
                             const ssd_pair_params* pair, int32_t device, int32_t max_branches,
                             int32_t max_lookahead, ssd_engine** out);
/* Same, for one role of a split run (ssd_role). */
ssd_status ssd_engine_create_role(const ssd_model_shape* target, const ssd_model_shape* draft,
                                  const ssd_pair_params* pair, int32_t device, int32_t role, int32_t max_branches,
                                  int32_t max_lookahead, ssd_engine** out);
/* Same, for rank tp_rank of a tensor-parallel target of tp_size ranks
 * (Megatron sharding: column-parallel QKV / gate-up, row-parallel O / down,
 * vocabulary-parallel head, replicated embedding). Role SSD_ROLE_VERIFIER:
 * the split run's verifier; SSD_ROLE_COLOCATED: the target sharded and the
 * draft replicated on every rank, for the same-box AR / SD baselines
 * (ssd_run_ar / ssd_run_sd). Connect the ranks with ssd_tp_export /
 * ssd_tp_connect; every rank then makes the same calls and computes
 * identical results. */
ssd_status ssd_engine_create_tp(const ssd_model_shape* target, const ssd_model_shape* draft,
                                const ssd_pair_params* pair, int32_t device, int32_t role, int32_t tp_rank,
                                int32_t tp_size, int32_t max_branches, int32_t max_lookahead, ssd_engine** out);
/* Same, colocated, with `max_batch` batch lanes (SimConfig::batch_size,
 * sim.hpp:40): each lane has its own KV region, history and streams. */
ssd_status ssd_engine_create_batch(const ssd_model_shape* target, const ssd_model_shape* draft,
                                   const ssd_pair_params* pair, int32_t device, int32_t max_batch,
                                   int32_t max_branches, int32_t max_lookahead, ssd_engine** out);
ssd_status ssd_engine_destroy(ssd_engine* e);
/* Bytes of weights streamed per forward step of model `which` (0 target,
 * 1 draft): the algorithmic bytes of one decode step. */
int64_t ssd_engine_weight_bytes(const ssd_engine* e, int32_t which);

/* ------------------------------------------------- decode loops (sim.hpp) */

/* sim::run_ar (sim.cpp:64-86): `tokens` autoregressive target samples. */
ssd_status ssd_run_ar(ssd_engine* e, const int32_t* prompt, int32_t prompt_len,
                      const ssd_scheme* target_scheme, int64_t tokens, uint64_t seed,
                      int32_t* out_tokens, int64_t out_capacity, ssd_run_stats* stats);

/* sim::run_sd (sim.cpp:88-121): draft K, verify, repeat. */
ssd_status ssd_run_sd(ssd_engine* e, const int32_t* prompt, int32_t prompt_len,
                      const ssd_sim_config* cfg, int32_t* out_tokens, int64_t out_capacity,
                      int64_t* out_len, ssd_run_stats* stats);

/* sim::run_protocol_harness (sim.cpp:502-601): the Saguaro loop. The
 * speculator pre-speculates every predicted outcome while the verifier
 * verifies; one message pair per round (v2d outcome, d2v speculation).
 * Per-round outcomes (k, t*) and hit bits of the sequence are written to
 * out_outcomes[2*r..2*r+1] / out_hits[r] when non-NULL. */
ssd_status ssd_run_ssd(ssd_engine* e, const int32_t* prompt, int32_t prompt_len,
                       const ssd_sim_config* cfg, int32_t* out_tokens, int64_t out_capacity,
                       int64_t* out_len, int32_t* out_outcomes, int32_t* out_hits,
                       ssd_run_stats* stats);

/* run_protocol_harness with SimConfig::batch_size = `batch` (sim.cpp:502-601,
 * sim.hpp:121-126): every sequence shares the prompt, sequence j drafts from
 * Stream(derive_seed(seed, j)) and verifies from
 * Stream(derive_seed(derive_seed(seed, 0x5EED), j)); the batch's forwards run
 * batched on the GPU (verify M = batch (K+1), branch steps M = batch B), and a
 * miss in any sequence stalls the round's virtual clock for the backup
 * (whole-batch stall). Streams go to out_tokens[j * out_capacity ..] with
 * lengths out_lens[j]; outcomes / hits are sequence 0's; stats sum over the
 * batch (RunStats semantics). batch == 1 is ssd_run_ssd. */
ssd_status ssd_run_ssd_batch(ssd_engine* e, const int32_t* prompt, int32_t prompt_len,
                             const ssd_sim_config* cfg, int32_t batch, int32_t* out_tokens,
                             int64_t out_capacity, int64_t* out_lens, int32_t* out_outcomes,
                             int32_t* out_hits, ssd_run_stats* stats);
/* Loop semantics and the round transcript (ssd_run_ssd_ex). */
enum { SSD_SEMANTICS_HARNESS = 0,    /* sim::run_protocol_harness (sim.cpp:502-601): verifier and
                                        draft streams, cache built while verifying */
       SSD_SEMANTICS_SEQUENTIAL = 1  /* sim::run_ssd / run_ssd_batch (sim.cpp:123-250): one stream per
                                        sequence; verify, then build_cache, then the backup */ };
typedef struct ssd_run_options {
  int32_t semantics;        /* SSD_SEMANTICS_* */
  char* transcript;         /* optional JSONL round transcript (Transcript::to_jsonl, sim.cpp:489-500),
                               NUL-terminated, harness semantics only */
  int64_t transcript_cap;   /* bytes available at transcript */
  int64_t* transcript_len;  /* optional: bytes the full transcript needs (without the NUL) */
} ssd_run_options;

/* ssd_run_ssd_batch with a choice of semantics and an optional transcript.
 * Raises SSD_PROTOCOL_VIOLATION when the harness' overlap invariant fails
 * (sim.cpp:534-537). */
ssd_status ssd_run_ssd_ex(ssd_engine* e, const int32_t* prompt, int32_t prompt_len, const ssd_sim_config* cfg,
                          int32_t batch, const ssd_run_options* opt, int32_t* out_tokens, int64_t out_capacity,
                          int64_t* out_lens, int32_t* out_outcomes, int32_t* out_hits, ssd_run_stats* stats);

/* ------------------------------------------ split processes (sim.cpp:258-601)
 * The reference's Channel between VerifierProcess and DraftProcess becomes
 * device mailboxes in HBM, mapped across processes/GPUs by CUDA IPC (NVLink
 * peer memory); messages are written by the sender's kernels inside the
 * round graph. Peer table order: [0..T) verifier ranks (T = tensor-parallel
 * size, 1 without TP), [T..T+G) speculators. */

/* Export this engine's mailbox (SSD_MAILBOX_HANDLE_BYTES bytes). */
ssd_status ssd_mailbox_export(ssd_engine* e, uint8_t* handle);
/* Map the peers' mailboxes: handles[i * SSD_MAILBOX_HANDLE_BYTES ..] for
 * i in [0, n_peers); entry `self` is this engine's own. */
ssd_status ssd_mailbox_connect(ssd_engine* e, int32_t n_peers, const uint8_t* handles, int32_t self);

/* Tensor-parallel verifier: export this rank's collective region (CUDA IPC,
 * SSD_MAILBOX_HANDLE_BYTES bytes) and map all ranks' regions
 * (handles[r * SSD_MAILBOX_HANDLE_BYTES ..] for r in [0, tp_size)). The two
 * all-reduces per layer and the logits all-gather then run as peer-memory
 * kernels inside every forward. */
ssd_status ssd_tp_export(ssd_engine* e, uint8_t* handle);
ssd_status ssd_tp_connect(ssd_engine* e, const uint8_t* handles);

/* VerifierProcess side of run_protocol_harness (sim.cpp:321-351, 502-601):
 * per round wait for the speculation, verify (M = K+1 target forward +
 * fused verification), send (k*, t*) to the n_spec speculators (TP rank 0
 * of a tensor-parallel verifier; every rank verifies identically). Writes
 * the emitted tokens and per-round outcomes. */
ssd_status ssd_run_ssd_verifier(ssd_engine* e, const int32_t* prompt, int32_t prompt_len, const ssd_sim_config* cfg,
                                int32_t n_spec, int32_t* out_tokens, int64_t out_capacity, int64_t* out_len,
                                int32_t* out_outcomes, ssd_run_stats* stats);

/* DraftProcess side (sim.cpp:376-485) for speculator `rank` of n_spec:
 * pre-speculates its block of branches while the verifier verifies, rebuilds
 * the history from (k*, t*), looks up, backs up, and sends the next
 * speculation when it owns the hit (or, rank 0, for a backup). Stats hold
 * the full RunStats counters (identical on every speculator). */
ssd_status ssd_run_ssd_speculator(ssd_engine* e, const int32_t* prompt, int32_t prompt_len, const ssd_sim_config* cfg,
                                  int32_t rank, int32_t n_spec, int32_t n_verifiers, int32_t* out_hits,
                                  ssd_run_stats* stats);

/* ------------------------------------------ single operations (specdec.hpp,
 * cache.hpp). Each starts from `context` (prefilled into the model's KV). */

/* lm::SyntheticLM::logits_at (lm.cpp:82-84): fp32 logits after `context`. */
ssd_status ssd_logits(ssd_engine* e, int32_t which, const int32_t* context, int32_t n,
                      float* out_logits);

/* specdec::draft (specdec.hpp:59-61): K tokens drawn from the draft under
 * `scheme` with stream Stream(seed); fp32 draft logit rows [K][V] copied out
 * when out_rows != NULL. */
ssd_status ssd_draft(ssd_engine* e, const int32_t* context, int32_t n, int32_t lookahead,
                     const ssd_scheme* scheme, uint64_t seed, int32_t* out_tokens, float* out_rows);

/* cache::build_cache + SpeculationCache::lookup key set (cache.hpp:149-154,
 * 123-126): the pre-speculation of the in-flight `spec_tokens` drafted from
 * `context`. Writes the Σ F_k keys (k, t) in ordinal order to out_keys[2i..]
 * and each entry's next_lookahead tokens to out_entry_tokens[i*next_K ..].
 * `base_seed` stands for the one draw the reference takes from the caller's
 * stream (cache.cpp:245). */
ssd_status ssd_build_cache(ssd_engine* e, const int32_t* context, int32_t n,
                           const int32_t* spec_tokens, int32_t lookahead, const ssd_plan* plan,
                           const ssd_scheme* scheme, int32_t next_lookahead, uint64_t base_seed,
                           int32_t* out_keys, int32_t* out_entry_tokens, int32_t* out_count);

/* ------------------------------------------------ caller-owned streams
 * rng::Stream (rng.hpp:29-48) as a plain C value: the mt19937_64 state of
 * std::mt19937_64(seed), advanced in place by every call that takes an
 * ssd_rng_stream* exactly as the reference advances the Stream& it is given
 * (one uniform per draw, one next_u64 per build_cache). Layout-compatible
 * with the engine's device streams, so state moves between host and GPU. */
typedef struct ssd_rng_stream {
  uint64_t state[312];
  int32_t index;
  int32_t reserved_;
} ssd_rng_stream;
void ssd_rng_stream_seed(ssd_rng_stream* s, uint64_t seed);  /* Stream(seed) */
uint64_t ssd_rng_stream_next_u64(ssd_rng_stream* s);          /* Stream::next_u64 */
double ssd_rng_stream_next_uniform(ssd_rng_stream* s);        /* Stream::next_uniform, (x >> 11) * 2^-53 */
uint64_t ssd_derive_seed(uint64_t root, uint64_t index);      /* rng::derive_seed (rng.hpp:24-26) */

/* specdec::draft (specdec.hpp:59-61) with the caller's stream: K uniforms
 * drawn from *rng (greedy draws none); tokens and the fp32 draft logit rows
 * [K][V] they were drawn from (the Speculation's dists = scheme(rows)). */
ssd_status ssd_draft_stream(ssd_engine* e, const int32_t* context, int32_t n, int32_t lookahead,
                            const ssd_scheme* scheme, ssd_rng_stream* rng, int32_t* out_tokens, float* out_rows);

/* specdec::verify (specdec.hpp:81-83, specdec.cpp:27-69): the target's
 * verify forward over context || spec (K+1 logit rows, M = K+1) and the
 * fused decision, drawing coins / the bonus from *rng. spec_rows: the draft
 * logit rows [K][V] the speculation was drawn from under draft_scheme, NULL
 * for a speculation with uniform dists (the FastRandom backup, sim.cpp:35-48).
 * Writes the outcome (k, t*) and emitted[0..k] (the accepted prefix plus the
 * bonus; capacity K+1). VerifyOptions = (target_scheme, accept_scale). */
ssd_status ssd_verify(ssd_engine* e, const int32_t* context, int32_t n, const int32_t* spec_tokens,
                      int32_t lookahead, const float* spec_rows, const ssd_scheme* draft_scheme,
                      const ssd_scheme* target_scheme, double accept_scale, ssd_rng_stream* rng,
                      int32_t* accepted, int32_t* bonus, int32_t* emitted);

/* cache::build_cache (cache.hpp:149-154, cache.cpp:232-277) with the
 * caller's stream: exactly one next_u64 taken from *rng as the entries'
 * base (cache.cpp:245); entry i continues for next_lookahead (1 .. engine
 * capacity, may differ from the speculation's K) tokens drawn from
 * Stream(derive_seed(base, i)). Writes the keys (k, t) in ordinal order,
 * each entry's tokens [count][next_K] and, when out_entry_rows != NULL, the
 * draft logit rows they were drawn from [count][next_K][V]. */
ssd_status ssd_build_cache_stream(ssd_engine* e, const int32_t* context, int32_t n, const int32_t* spec_tokens,
                                  int32_t lookahead, const ssd_plan* plan, const ssd_scheme* scheme,
                                  int32_t next_lookahead, ssd_rng_stream* rng, int32_t* out_keys,
                                  int32_t* out_entry_tokens, float* out_entry_rows, int32_t* out_count);

/* ------------------------------------- asynchronous pre-speculation
 * the speculator's build_cache as a device-side session call.
 * ssd_prespec_begin enqueues the pre-speculation of DEVICE buffers
 * d_context[n] / d_spec_tokens[K] on the engine's speculator stream, ordered
 * after the work already queued on `cuda_stream` (a cudaStream_t, NULL = no
 * ordering), and returns without waiting; it takes one next_u64 from *rng
 * on the host (cache.cpp:245). The cache stays valid until the next
 * ssd_prespec_begin. ssd_cache_lookup / _keys / _entry wait for it. */
ssd_status ssd_prespec_begin(ssd_engine* e, const int32_t* d_context, int32_t n, const int32_t* d_spec_tokens,
                             int32_t lookahead, const ssd_plan* plan, const ssd_scheme* scheme,
                             int32_t next_lookahead, ssd_rng_stream* rng, void* cuda_stream);
/* SpeculationCache::lookup (cache.hpp:123-126): *slot = entry ordinal of
 * key (accepted, bonus), or -1 on a miss. */
ssd_status ssd_cache_lookup(ssd_engine* e, int32_t accepted, int32_t bonus, int32_t* slot);
/* Every key (k, t) in ordinal order (out_keys[2 * count]) — the parity hook. */
ssd_status ssd_cache_keys(ssd_engine* e, int32_t* out_keys, int32_t* out_count);
/* Entry `slot`: tokens [next_K] and (optional) draft logit rows [next_K][V], host buffers. */
ssd_status ssd_cache_entry(ssd_engine* e, int32_t slot, int32_t* out_tokens, float* out_rows);

/* ------------------------------------------- kernel-level parity hooks
 * (host buffers in, host buffers out; used by tests/). */

/* Candidate keys from draft logit rows (cache.cpp:249-270): for each row k,
 * the first fan_out[k] tokens of the (value desc, index asc) order that are
 * not excluded[k] (-1 = no exclusion). Writes keys[k*max_f + j]. */
ssd_status ssd_topk_keys(ssd_engine* e, const float* rows, int32_t n_rows, int32_t vocab,
                         const int32_t* fan_out, const int32_t* excluded, int32_t max_f,
                         int32_t* keys);

/* specdec::verify decision (specdec.cpp:27-69) on given logits: target rows
 * [K+1][V], draft rows [K][V] (NULL = uniform dists, the FastRandom backup),
 * drafted tokens [K], verifier stream Stream(seed). Writes (accepted, bonus). */
ssd_status ssd_verify_rows(ssd_engine* e, const float* target_rows, const float* draft_rows,
                           const int32_t* tokens, int32_t lookahead, int32_t vocab,
                           const ssd_scheme* draft_scheme, const ssd_scheme* target_scheme,
                           double accept_scale, uint64_t seed, int32_t* accepted, int32_t* bonus);

/* Roofline hook (bench.py): times `iters` forward steps of model `which`
 * over M tokens at context position `pos` with CUDA events on the engine
 * stream, and separately the step's weight-streaming GEMM launches alone.
 * Outputs average ms per step / per step's GEMM launches and the GEMM
 * launches' algorithmic bytes (weights + activations) per step. */
ssd_status ssd_profile_forward(ssd_engine* e, int32_t which, int32_t M, int32_t pos, int32_t iters,
                               double* ms_forward, double* ms_gemm, int64_t* gemm_bytes, int32_t* gemm_launches);

/* In-graph profile of the colocated SSD round: runs the same
 * round graphs as ssd_run_ssd, captured with event-record nodes at the
 * segment boundaries of both streams, one host sync per round. out_ms[9]
 * (averages over cfg->rounds rounds): [0] round, [1] verify forward (8B,
 * M = K+1, co-running), [2] verify decision, [3] extend forward (draft,
 * M = K+1), [4] cache keys + branch streams, [5] K branch-step forwards
 * (M = B, summed), [6] their token picks, [7] join + lookup, [8] fork lag. */
ssd_status ssd_profile_ssd_round(ssd_engine* e, const int32_t* prompt, int32_t prompt_len,
                                 const ssd_sim_config* cfg, double* out_ms, ssd_run_stats* stats);

/* Read-only HBM streaming probe: achievable read bandwidth (GB/s) of a
 * plain vectorised load kernel over `bytes`, averaged over `iters`. */
ssd_status ssd_bench_read_bw(ssd_engine* e, int64_t bytes, int32_t iters, double* gbs);

/* mt19937_64 parity: n outputs of Stream(seed).next_u64() computed on the GPU. */
ssd_status ssd_rng_u64(ssd_engine* e, uint64_t seed, int32_t n, uint64_t* out);

/* Weight-generator parity: bf16 bits of logical elements (kind 0..6 = q,k,v,
 * o,gate,up,down of `layer`; 100 = embedding; 101 = LM head). */
ssd_status ssd_weight_bits(ssd_engine* e, int32_t which, int32_t layer, int32_t kind,
                           const int64_t* rows, const int64_t* cols, int32_t n, uint16_t* out);

/* ------------------------------------------------ paged KV block manager
 * SURVEY §8f row 4, the paper's engine: pages of
 * page_tokens KV slots shared by the target and the draft cache; lookahead
 * reservation for the K+1 verify / draft steps, reconciliation after
 * verification (finalize full pages under a chained prefix hash, roll back
 * pages reserved beyond the accepted suffix), and a prefix cache that maps a
 * new prompt's cached full pages read-only (LRU eviction of unreferenced
 * cached pages). Host bookkeeping (csrc/paged.cpp); the engine consumes the
 * block tables (ssd_engine_set_block_table). Out of pages: SSD_TOO_LARGE
 * (the caller preempts a sequence and retries). */
typedef struct ssd_kv_pool ssd_kv_pool;
typedef struct ssd_kv_stats {
  int32_t n_pages, free_pages, used_pages, cached_pages, cached_evictable, sequences;
  int64_t allocated, evictions, finalized, prefix_hit_pages, prefix_miss_pages, reserved_pages, rolled_back_pages;
} ssd_kv_stats;
ssd_status ssd_kv_pool_create(int32_t n_pages, int32_t page_tokens, ssd_kv_pool** out);
void ssd_kv_pool_destroy(ssd_kv_pool* pool);
/* Admit a prompt: maps its cached full prefix pages (*cached_tokens tokens
 * whose KV need not be prefilled; never the page of the last token) and
 * allocates the rest. */
ssd_status ssd_kv_seq_admit(ssd_kv_pool* pool, int64_t seq, const int32_t* tokens, int32_t n, int32_t* cached_tokens);
/* Ensure pages for committed length + lookahead (K + 1 before a round). */
ssd_status ssd_kv_seq_reserve(ssd_kv_pool* pool, int64_t seq, int32_t lookahead);
/* After verification: append the accepted tokens (k + 1), finalize full
 * pages, release the reserved pages beyond them (*pages_released). */
ssd_status ssd_kv_seq_commit(ssd_kv_pool* pool, int64_t seq, const int32_t* accepted, int32_t n_accepted,
                             int32_t* pages_released);
ssd_status ssd_kv_seq_release(ssd_kv_pool* pool, int64_t seq);
ssd_status ssd_kv_seq_table(const ssd_kv_pool* pool, int64_t seq, int32_t* pages, int32_t cap, int32_t* n_pages,
                            int32_t* n_tokens);
ssd_status ssd_kv_pool_stats(const ssd_kv_pool* pool, ssd_kv_stats* out);
ssd_status ssd_kv_page_refs(const ssd_kv_pool* pool, int32_t* refs, int32_t cap);

/* The engine side of the paged KV cache: the main caches of both models as
 * pages of page_tokens slots (page p = page p % ppl of lane p / ppl's main
 * region, ppl = max_ctx / page_tokens; the same index in the target and the
 * draft arena: *n_pages = lanes * ppl, the pool size). A lane's block table
 * maps its logical pages to physical ones; its first cached_tokens prompt
 * tokens already have their KV there (ssd_kv_seq_admit's prefix hit) and are
 * not prefilled. page_tokens: a power of two dividing max_ctx. Branch slots
 * (pre-speculation) are never paged. */
ssd_status ssd_engine_kv_pages(ssd_engine* e, int32_t page_tokens, int32_t* n_pages);
ssd_status ssd_engine_set_block_table(ssd_engine* e, int32_t lane, const int32_t* pages, int32_t n_pages,
                                      int32_t page_tokens, int32_t cached_tokens);
ssd_status ssd_engine_clear_block_tables(ssd_engine* e);

/* B200 execution knob, no reference counterpart: the colocated SSD round
 * runs its verifier branch and its speculator branch on disjoint SM sets
 * (two CUDA green contexts). verifier_sms > 0 sets the verifier's share
 * (rounded by the driver to its partition granularity; the speculator gets
 * the rest), 0 shares all SMs between the two streams, < 0 leaves the
 * partition unchanged. *out_verifier / *out_speculator (nullable) receive
 * the SM counts in effect (0, 0 when shared). Colocated single-GPU engines
 * only (SSD_CONFIG otherwise); the default is 3/8 of the SMs. */
ssd_status ssd_engine_sm_partition(ssd_engine* e, int32_t verifier_sms, int32_t* out_verifier,
                                   int32_t* out_speculator);

#ifdef __cplusplus
}
#endif
#endif /* SSD_B200_H_ */
