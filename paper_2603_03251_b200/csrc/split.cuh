// Split verifier / speculator processes: the
// reference's two-process protocol (sim.cpp:258-601 — Channel, VerifierProcess,
// DraftProcess) across GPUs. Each process owns an Inbox in its own HBM,
// exported by CUDA IPC and mapped by its peers over NVLink / NVSwitch; a
// message is written straight into the receiver's inbox by the sender's
// kernel (payload stores, system-scope fence, release store of the sequence
// number) and picked up by the receiver's kernel with acquire loads. The
// whole round stays inside one CUDA graph per process: no host hop, no NCCL
// launch. Exactly one message pair per round, draft first (sim.cpp:524-577):
//   d2v seq base+r+1: speculation for round r (hit bit implied by
//                     origin/src, K tokens, draft rows [K][V] unless uniform)
//   v2d seq base+r+1: outcome of round r (k*, t*) + the verifier's history length
// Sequence numbers grow monotonically across runs (`seq_base`), so a stale
// message of an earlier run is never mistaken for a new one.
// With G > 1 speculators (branch sharding) the owner of the hit slot also
// broadcasts the next speculation's tokens to the other speculators
// (`peer` slot), since only it decoded that branch.
#pragma once

#include "kernels.cuh"

namespace ssd {

struct alignas(128) MsgV2D {
  int seq;
  int k, t, n;
};

struct alignas(128) MsgD2V {
  int seq;
  int origin, src, uniform;
  int tokens[kMaxK];
};

// Header of every process's inbox; the verifier's draft-row payload
// [2][K][V] fp32 (double-buffered by sequence parity: the ranks of a
// tensor-parallel verifier may still read round r's rows while round r + 1's
// arrive) follows at kInboxRows bytes.
// Speculator slots are double-buffered by sequence parity, with credit flow
// control: a speculator publishes `done` (the sequence number of its last
// finished round) and a sender overwrites a slot only once the message that
// last used it has been consumed. A speculator that neither sends nor is
// waited on may therefore trail by a round but never lose a message.
struct alignas(128) Credit {
  int done;
};
struct Inbox {
  MsgV2D v2d[2];   // speculator inbox: outcome from the verifier
  MsgD2V d2v;      // verifier inbox: next speculation
  MsgD2V peer[2];  // speculator inbox: tokens of a hit owned by another speculator
  Credit credit;   // speculator inbox: read remotely by the senders
};
constexpr size_t kInboxRows = 1024;
static_assert(sizeof(Inbox) <= kInboxRows, "inbox header");

constexpr unsigned long long kMailTimeoutNs = 60ull * 1000 * 1000 * 1000;  // 60 s: then SSD_PROTOCOL_VIOLATION

__device__ __forceinline__ int ld_acquire_sys(const int* p) {
  int v;
  asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(int* p, int v) {
  asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Spin (with back-off) until *seq >= want. A peer that never answers turns
// into SSD_PROTOCOL_VIOLATION (the reference's ProtocolViolationError for a
// missing message, sim.cpp:276-293, 579-581) instead of a hung GPU.
__device__ bool wait_seq(const int* seq, int want, LoopState* st) {
  const unsigned long long t0 = now_ns();
  unsigned ns = 32;
  while (ld_acquire_sys(seq) < want) {
    __nanosleep(ns);
    if (ns < 2048) ns <<= 1;
    if (now_ns() - t0 > kMailTimeoutNs) {
      st->error = 10;
      return false;
    }
  }
  return true;
}

// Verifier: wait for the speculation of round st->round and install it
// (the verifier-side half of Channel::send_speculations, sim.cpp:275-288).
__global__ void recv_spec_kernel(LoopState* st, const Inbox* in, const float* rows2, int V) {
  if (threadIdx.x != 0 || st->error) return;
  const int seq = st->seq_base + st->round + 1;
  if (!wait_seq(&in->d2v.seq, seq, st)) return;
  const int K = st->K;
  const float* rows = rows2 + size_t(seq & 1) * K * V;
  st->spec_origin = in->d2v.origin;
  st->spec_src = in->d2v.src;
  st->spec_uniform = in->d2v.uniform;
  for (int i = 0; i < K; ++i) {
    st->spec[i] = in->d2v.tokens[i];
    st->spec_rows[i] = in->d2v.uniform ? nullptr : rows + size_t(i) * V;
  }
}

// Verifier: send (k*, t*) of round st->round to every speculator
// (Channel::send_outcomes, sim.cpp:290-303); log it.
__global__ void send_outcome_kernel(LoopState* st, Inbox* const* peers, int G, int* log_outcomes) {
  if (threadIdx.x != 0 || st->error) return;
  const int r = st->round;
  const int seq = st->seq_base + r + 1;
  const int b = seq & 1;
  for (int g = 0; g < G; ++g) {
    // slot b last carried seq - 2: wait until speculator g finished that round
    if (!wait_seq(&peers[g]->credit.done, seq - 2, st)) return;
    MsgV2D& m = peers[g]->v2d[b];
    m.k = st->out_k;
    m.t = st->out_t;
    m.n = st->n;
  }
  __threadfence_system();
  for (int g = 0; g < G; ++g) st_release_sys(&peers[g]->v2d[b].seq, seq);
  if (log_outcomes) {
    log_outcomes[2 * r] = st->out_k;
    log_outcomes[2 * r + 1] = st->out_t;
  }
}

// Speculator: wait for the outcome of round st->round and rebuild the
// emitted tokens from its own speculation + (k*, t*) (DraftProcess::
// handle_outcomes, sim.cpp:435-440). Counts tokens / accepted like verify.
__global__ void recv_outcome_kernel(LoopState* st, const Inbox* in, int* hist) {
  if (threadIdx.x != 0 || st->error) return;
  const int want = st->seq_base + st->round + 1;
  const MsgV2D& m = in->v2d[want & 1];
  if (!wait_seq(&m.seq, want, st)) return;
  const int k = m.k, t = m.t, n = st->n;
  if (m.seq != want || m.n != n || k < 0 || k > st->K) {  // histories out of step
    st->error = 10;
    return;
  }
  for (int i = 0; i < k; ++i) hist[n + i] = st->spec[i];
  hist[n + k] = t;
  st->out_k = k;
  st->out_t = t;
  st->tokens += k + 1;
  st->accepted_sum += double(k);
}

// Speculator: send the speculation for round st->round (after lookup /
// backup) to the verifier. Sender: the owner of a hit, or speculator 0 for a
// backup (every speculator computes the identical backup) or the initial /
// JIT draft (force). Rows [K][V] are copied by all CTAs (with_rows = 1: the
// verification reads them in every mode); the last CTA to finish publishes
// the header (release) so the rows are visible first.
// peers[0..T) = verifier inboxes (the ranks of a tensor-parallel verifier
// all verify the same speculation), peers[T..T+G) = speculator inboxes.
__global__ void __launch_bounds__(256) send_spec_kernel(LoopState* st, Inbox* const* peers, int T, int G, int rank,
                                                        int V, int force, int* counter, int with_rows) {
  __shared__ int s_send, s_last;
  const int K = st->K;
  const int rslot = (st->seq_base + st->round + 1) & 1;  // rows slot of this message
  if (threadIdx.x == 0) {
    int send = 0;
    if (!st->error && st->round < st->rounds) {
      if (force) send = rank == 0;
      else if (st->hit) send = st->own;
      else send = rank == 0 && st->backup_kind == 1;
    }
    s_send = send;
  }
  __syncthreads();
  if (!s_send) return;
  if (!st->spec_uniform && with_rows) {
    const size_t n4 = size_t(V) / 4;  // V % 4 == 0 (checked on the host)
    for (int i = 0; i < K; ++i) {
      const float4* src = reinterpret_cast<const float4*>(st->spec_rows[i]);
      for (size_t j = blockIdx.x * size_t(blockDim.x) + threadIdx.x; j < n4; j += size_t(gridDim.x) * blockDim.x) {
        const float4 v = src[j];
        for (int vr = 0; vr < T; ++vr)
          reinterpret_cast<float4*>(reinterpret_cast<char*>(peers[vr]) + kInboxRows)[(size_t(rslot) * K + i) * (V / 4) + j] = v;
      }
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(counter, 1) == int(gridDim.x) - 1;
  __syncthreads();
  if (!s_last || threadIdx.x != 0) return;
  *counter = 0;
  __threadfence_system();
  const int seq = st->seq_base + st->round + 1;
  MsgD2V m;
  m.origin = st->spec_origin;
  m.src = st->spec_src;
  m.uniform = st->spec_uniform;
  for (int i = 0; i < K; ++i) m.tokens[i] = st->spec[i];
  for (int vr = 0; vr < T; ++vr) {
    Inbox* vin = peers[vr];
    vin->d2v.origin = m.origin;
    vin->d2v.src = m.src;
    vin->d2v.uniform = m.uniform;
    for (int i = 0; i < K; ++i) vin->d2v.tokens[i] = m.tokens[i];
  }
  const bool bcast = !force && st->hit;  // others lack this branch's tokens
  if (bcast)
    for (int g = 0; g < G; ++g) {
      if (g == rank) continue;
      // slot seq & 1 last carried seq - 2, read in speculator g's round done = seq - 3
      if (!wait_seq(&peers[T + g]->credit.done, seq - 3, st)) return;
      MsgD2V& p = peers[T + g]->peer[seq & 1];
      p.origin = m.origin;
      p.src = m.src;
      p.uniform = m.uniform;
      for (int i = 0; i < K; ++i) p.tokens[i] = m.tokens[i];
    }
  __threadfence_system();
  for (int vr = 0; vr < T; ++vr) st_release_sys(&peers[vr]->d2v.seq, seq);
  if (bcast)
    for (int g = 0; g < G; ++g)
      if (g != rank) st_release_sys(&peers[T + g]->peer[seq & 1].seq, seq);
}

// Speculator that does not own the hit slot: take the next speculation's
// tokens from the owner's broadcast.
// Ends every speculator round: publishes the round's credit.
__global__ void recv_peer_spec_kernel(LoopState* st, Inbox* in) {
  if (threadIdx.x != 0 || st->error) return;
  if (st->round < st->rounds && st->hit && !st->own) {
    const int want = st->seq_base + st->round + 1;
    const MsgD2V& m = in->peer[want & 1];
    if (!wait_seq(&m.seq, want, st)) return;
    if (m.seq != want) {
      st->error = 10;
      return;
    }
    for (int i = 0; i < st->K; ++i) {
      st->spec[i] = m.tokens[i];
      st->spec_rows[i] = nullptr;
    }
  }
  // round st->round - 1 (0-based) consumed v2d seq base + round and peer seq base + round + 1
  __threadfence_system();
  st_release_sys(&in->credit.done, st->seq_base + st->round);
}

}  // namespace ssd
