// Paged KV block manager with lookahead reservation, post-verification
// reconciliation / rollback and a prefix-cache hash (the
// paper's engine: "the scheduler ensures the target has
// sufficient pages for K+1 multi-query decoding steps ... After verification,
// both page tables are reconciled: completed pages are finalized (hashed for
// prefix caching), and any pages allocated beyond the accepted suffix are
// deallocated").
//
// Host-side bookkeeping, one pool per engine: pages of `page_tokens` KV
// slots, shared by the target and the draft model (a page index names the
// same token range in both models' caches). The device side consumes the
// per-sequence block tables (ssd_engine_set_block_table): the attention
// kernels translate main-cache slots through them.
//
// Prefix cache: a full page is finalized with the chained hash
// h_i = mix(h_{i-1}, tokens of page i) and registered under it, together
// with its tokens (lookups compare them: no false sharing on a 64-bit hash
// collision). A later sequence whose prompt starts with the same full pages
// maps them read-only (refcount) and skips their prefill. Pages whose
// refcount drops to zero stay cached and are evicted least-recently-used
// when the free list runs dry. Writes never touch a shared page: only full
// pages are shared, and the page holding the last prompt token is always
// private (its logits must be recomputed).
#include <algorithm>
#include <cstdint>
#include <list>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/ssd_b200.h"

namespace ssd {
extern thread_local std::string g_last_error;
}

struct ssd_kv_pool {
  int n_pages = 0, page_tokens = 0;
  std::vector<int> ref;                      // per page
  std::vector<uint64_t> hash;                // finalized prefix hash (valid when cached[p])
  std::vector<char> cached;                  // registered in the prefix cache
  std::vector<std::vector<int32_t>> toks;    // tokens of a cached page (collision check)
  std::vector<int> free_list;                // ref 0, not cached (LIFO)
  std::list<int> lru;                        // ref 0, cached: evictable, least recent first
  std::vector<std::list<int>::iterator> lru_at;
  std::vector<char> in_lru;
  std::unordered_multimap<uint64_t, int> index;  // hash -> cached page
  struct Seq {
    std::vector<int> pages;      // block table
    std::vector<int32_t> tokens; // committed tokens (KV written and accepted)
    int finalized = 0;           // leading pages finalized (hashed)
    uint64_t chain = 0;          // hash of the last finalized page
  };
  std::unordered_map<int64_t, Seq> seqs;
  ssd_kv_stats st{};
};

namespace {

struct KvError {
  ssd_status code;
  std::string msg;
};

constexpr uint64_t kHashSeed = 0x9E3779B97F4A7C15ULL;

uint64_t mix64(uint64_t x) {  // splitmix64 finaliser
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

uint64_t page_hash(uint64_t parent, const int32_t* t, int n) {
  uint64_t h = mix64(parent ^ kHashSeed);
  for (int i = 0; i < n; ++i) h = mix64(h ^ uint64_t(uint32_t(t[i])));
  return h == 0 ? 1 : h;  // 0 is "no parent"
}

void lru_remove(ssd_kv_pool& P, int p) {
  if (!P.in_lru[size_t(p)]) return;
  P.lru.erase(P.lru_at[size_t(p)]);
  P.in_lru[size_t(p)] = 0;
}

void uncache(ssd_kv_pool& P, int p) {
  auto r = P.index.equal_range(P.hash[size_t(p)]);
  for (auto it = r.first; it != r.second; ++it)
    if (it->second == p) { P.index.erase(it); break; }
  P.cached[size_t(p)] = 0;
  P.toks[size_t(p)].clear();
}

// a page with ref 0: cached ones become evictable, the rest free
void park(ssd_kv_pool& P, int p) {
  if (P.cached[size_t(p)]) {
    P.lru.push_back(p);
    P.lru_at[size_t(p)] = std::prev(P.lru.end());
    P.in_lru[size_t(p)] = 1;
  } else {
    P.free_list.push_back(p);
  }
}

int alloc_page(ssd_kv_pool& P) {
  int p;
  if (!P.free_list.empty()) {
    p = P.free_list.back();
    P.free_list.pop_back();
  } else if (!P.lru.empty()) {  // evict the least recently used cached page
    p = P.lru.front();
    lru_remove(P, p);
    uncache(P, p);
    ++P.st.evictions;
  } else {
    throw KvError{SSD_TOO_LARGE, "kv pool: out of pages (reserve failed: preempt a sequence)"};
  }
  P.ref[size_t(p)] = 1;
  ++P.st.allocated;
  return p;
}

void release_page(ssd_kv_pool& P, int p) {
  if (--P.ref[size_t(p)] == 0) park(P, p);
}

int cached_lookup(const ssd_kv_pool& P, uint64_t h, const int32_t* t) {
  auto r = P.index.equal_range(h);
  for (auto it = r.first; it != r.second; ++it) {
    const std::vector<int32_t>& pt = P.toks[size_t(it->second)];
    if (std::equal(pt.begin(), pt.end(), t)) return it->second;
  }
  return -1;
}

// Finalize the full pages of s beyond s.finalized: chained hash, register
// (unless an identical page is cached already: then ours stays private).
void finalize(ssd_kv_pool& P, ssd_kv_pool::Seq& s) {
  const int ps = P.page_tokens;
  const int full = int(s.tokens.size()) / ps;
  for (int i = s.finalized; i < full && i < int(s.pages.size()); ++i) {
    const int32_t* t = s.tokens.data() + size_t(i) * ps;
    const uint64_t h = page_hash(s.chain, t, ps);
    s.chain = h;
    const int p = s.pages[size_t(i)];
    if (!P.cached[size_t(p)] && cached_lookup(P, h, t) < 0) {
      P.cached[size_t(p)] = 1;
      P.hash[size_t(p)] = h;
      P.toks[size_t(p)].assign(t, t + ps);
      P.index.emplace(h, p);
      ++P.st.finalized;
    }
    s.finalized = i + 1;
  }
}

ssd_kv_pool::Seq& seq_of(ssd_kv_pool& P, int64_t id) {
  auto it = P.seqs.find(id);
  if (it == P.seqs.end()) throw KvError{SSD_CONFIG, "kv pool: unknown sequence " + std::to_string(id)};
  return it->second;
}

template <class F>
ssd_status guard(F&& f) {
  try {
    f();
    return SSD_OK;
  } catch (const KvError& e) {
    ssd::g_last_error = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    ssd::g_last_error = e.what();
    return SSD_ERROR;
  }
}

}  // namespace

extern "C" {

ssd_status ssd_kv_pool_create(int32_t n_pages, int32_t page_tokens, ssd_kv_pool** out) {
  return guard([&] {
    if (!out || n_pages < 1 || page_tokens < 1) throw KvError{SSD_CONFIG, "kv pool: n_pages and page_tokens >= 1"};
    auto* P = new ssd_kv_pool;
    P->n_pages = n_pages;
    P->page_tokens = page_tokens;
    P->ref.assign(size_t(n_pages), 0);
    P->hash.assign(size_t(n_pages), 0);
    P->cached.assign(size_t(n_pages), 0);
    P->toks.resize(size_t(n_pages));
    P->lru_at.resize(size_t(n_pages));
    P->in_lru.assign(size_t(n_pages), 0);
    for (int p = n_pages - 1; p >= 0; --p) P->free_list.push_back(p);  // page 0 first
    *out = P;
  });
}

void ssd_kv_pool_destroy(ssd_kv_pool* P) { delete P; }

ssd_status ssd_kv_seq_admit(ssd_kv_pool* P, int64_t id, const int32_t* tokens, int32_t n, int32_t* cached_tokens) {
  return guard([&] {
    if (!P || (!tokens && n > 0) || n < 1) throw KvError{SSD_CONFIG, "kv admit: empty prompt"};
    if (P->seqs.count(id)) throw KvError{SSD_CONFIG, "kv admit: sequence already admitted"};
    const int ps = P->page_tokens;
    ssd_kv_pool::Seq s;
    // prefix-cache hits: full pages strictly before the last prompt token's page
    const int shareable = (n - 1) / ps;
    std::vector<int> hits;
    uint64_t chain = 0;
    for (int i = 0; i < shareable; ++i) {
      const uint64_t h = page_hash(chain, tokens + size_t(i) * ps, ps);
      const int p = cached_lookup(*P, h, tokens + size_t(i) * ps);
      if (p < 0) break;
      hits.push_back(p);
      chain = h;
    }
    const int need = (n + ps - 1) / ps - int(hits.size());
    // capacity check before any state change: free pages + evictable (not among the hits)
    int evictable = int(P->lru.size());
    for (int p : hits)
      if (P->in_lru[size_t(p)]) --evictable;
    if (need > int(P->free_list.size()) + evictable)
      throw KvError{SSD_TOO_LARGE, "kv admit: out of pages for the prompt"};
    for (int p : hits) {
      lru_remove(*P, p);
      ++P->ref[size_t(p)];
      s.pages.push_back(p);
    }
    for (int i = 0; i < need; ++i) s.pages.push_back(alloc_page(*P));
    s.tokens.assign(tokens, tokens + n);
    s.finalized = int(hits.size());
    s.chain = chain;
    // the prompt's own full pages are registered now: the caller prefills
    // them before any later forward (stream order), so a sequence admitted
    // after this one reads written KV
    finalize(*P, s);
    P->st.prefix_hit_pages += int64_t(hits.size());
    P->st.prefix_miss_pages += int64_t(shareable - int(hits.size()));
    if (cached_tokens) *cached_tokens = int32_t(hits.size()) * ps;
    P->seqs.emplace(id, std::move(s));
  });
}

ssd_status ssd_kv_seq_reserve(ssd_kv_pool* P, int64_t id, int32_t lookahead) {
  return guard([&] {
    if (!P || lookahead < 0) throw KvError{SSD_CONFIG, "kv reserve: bad arguments"};
    ssd_kv_pool::Seq& s = seq_of(*P, id);
    const int ps = P->page_tokens;
    const int want = (int(s.tokens.size()) + lookahead + ps - 1) / ps;
    const int need = want - int(s.pages.size());
    if (need > int(P->free_list.size()) + int(P->lru.size()))
      throw KvError{SSD_TOO_LARGE, "kv reserve: out of pages for the lookahead (preempt a sequence)"};
    for (int i = 0; i < need; ++i) s.pages.push_back(alloc_page(*P));
    P->st.reserved_pages += need > 0 ? need : 0;
  });
}

ssd_status ssd_kv_seq_commit(ssd_kv_pool* P, int64_t id, const int32_t* accepted, int32_t n_accepted,
                             int32_t* pages_released) {
  return guard([&] {
    if (!P || n_accepted < 0 || (!accepted && n_accepted > 0)) throw KvError{SSD_CONFIG, "kv commit: bad arguments"};
    ssd_kv_pool::Seq& s = seq_of(*P, id);
    const int ps = P->page_tokens;
    const int len = int(s.tokens.size()) + n_accepted;
    if ((len + ps - 1) / ps > int(s.pages.size()))
      throw KvError{SSD_PROTOCOL_VIOLATION, "kv commit: accepted tokens beyond the reserved pages"};
    s.tokens.insert(s.tokens.end(), accepted, accepted + n_accepted);
    finalize(*P, s);
    // rollback: pages reserved beyond the accepted suffix
    const int keep = (len + ps - 1) / ps;
    int released = 0;
    while (int(s.pages.size()) > keep) {
      release_page(*P, s.pages.back());
      s.pages.pop_back();
      ++released;
    }
    P->st.rolled_back_pages += released;
    if (pages_released) *pages_released = released;
  });
}

ssd_status ssd_kv_seq_release(ssd_kv_pool* P, int64_t id) {
  return guard([&] {
    if (!P) throw KvError{SSD_CONFIG, "kv release: null pool"};
    ssd_kv_pool::Seq& s = seq_of(*P, id);
    for (auto it = s.pages.rbegin(); it != s.pages.rend(); ++it) release_page(*P, *it);
    P->seqs.erase(id);
  });
}

ssd_status ssd_kv_seq_table(const ssd_kv_pool* P, int64_t id, int32_t* pages, int32_t cap, int32_t* n_pages,
                            int32_t* n_tokens) {
  return guard([&] {
    if (!P) throw KvError{SSD_CONFIG, "kv table: null pool"};
    auto it = P->seqs.find(id);
    if (it == P->seqs.end()) throw KvError{SSD_CONFIG, "kv table: unknown sequence " + std::to_string(id)};
    const auto& s = it->second;
    if (n_pages) *n_pages = int32_t(s.pages.size());
    if (n_tokens) *n_tokens = int32_t(s.tokens.size());
    if (pages) {
      if (cap < int(s.pages.size())) throw KvError{SSD_TOO_LARGE, "kv table: buffer too small"};
      for (size_t i = 0; i < s.pages.size(); ++i) pages[i] = s.pages[i];
    }
  });
}

ssd_status ssd_kv_pool_stats(const ssd_kv_pool* P, ssd_kv_stats* out) {
  return guard([&] {
    if (!P || !out) throw KvError{SSD_CONFIG, "kv stats: null argument"};
    *out = P->st;
    out->n_pages = P->n_pages;
    out->free_pages = int32_t(P->free_list.size());
    out->cached_evictable = int32_t(P->lru.size());
    out->cached_pages = int32_t(P->index.size());
    int used = 0;
    for (int r : P->ref) used += r > 0;
    out->used_pages = used;
    out->sequences = int32_t(P->seqs.size());
  });
}

ssd_status ssd_kv_page_refs(const ssd_kv_pool* P, int32_t* refs, int32_t cap) {
  return guard([&] {
    if (!P || !refs || cap < P->n_pages) throw KvError{SSD_CONFIG, "kv refs: buffer too small"};
    for (int p = 0; p < P->n_pages; ++p) refs[p] = P->ref[size_t(p)];
  });
}

}  // extern "C"
