"""Pure-Python model of the paged KV block manager (TEST INFRASTRUCTURE): the
semantics csrc/paged.cpp implements,
restated independently for a differential test."""
from __future__ import annotations

M64 = (1 << 64) - 1


def mix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def page_hash(parent: int, toks) -> int:
    h = mix64(parent ^ 0x9E3779B97F4A7C15)
    for t in toks:
        h = mix64(h ^ (t & 0xFFFFFFFF))
    return h or 1


class OutOfPages(Exception):
    pass


class KvModel:
    def __init__(self, n_pages: int, ps: int):
        self.n, self.ps = n_pages, ps
        self.ref = [0] * n_pages
        self.cached = {}          # page -> (hash, tokens)
        self.index = {}           # hash -> [pages]
        self.free = list(range(n_pages - 1, -1, -1))
        self.lru = []             # evictable cached pages, least recent first
        self.seqs = {}            # id -> dict(pages, tokens, finalized, chain)
        self.evictions = 0

    def _lookup(self, h, toks):
        for p in self.index.get(h, []):
            if self.cached[p][1] == list(toks):
                return p
        return -1

    def _alloc(self):
        if self.free:
            p = self.free.pop()
        elif self.lru:
            p = self.lru.pop(0)
            h, _ = self.cached.pop(p)
            self.index[h].remove(p)
            self.evictions += 1
        else:
            raise OutOfPages
        self.ref[p] = 1
        return p

    def _release(self, p):
        self.ref[p] -= 1
        if self.ref[p] == 0:
            (self.lru if p in self.cached else self.free).append(p)

    def _finalize(self, s):
        full = len(s["tokens"]) // self.ps
        i = s["finalized"]
        while i < full and i < len(s["pages"]):
            t = s["tokens"][i * self.ps:(i + 1) * self.ps]
            h = page_hash(s["chain"], t)
            s["chain"] = h
            p = s["pages"][i]
            if p not in self.cached and self._lookup(h, t) < 0:
                self.cached[p] = (h, list(t))
                self.index.setdefault(h, []).append(p)
            i += 1
            s["finalized"] = i

    def admit(self, sid, toks):
        ps = self.ps
        hits, chain = [], 0
        for i in range((len(toks) - 1) // ps):
            t = toks[i * ps:(i + 1) * ps]
            h = page_hash(chain, t)
            p = self._lookup(h, t)
            if p < 0:
                break
            hits.append(p)
            chain = h
        need = -(-len(toks) // ps) - len(hits)
        if need > len(self.free) + len([p for p in self.lru if p not in hits]):
            raise OutOfPages
        pages = []
        for p in hits:
            if p in self.lru:
                self.lru.remove(p)
            self.ref[p] += 1
            pages.append(p)
        pages += [self._alloc() for _ in range(need)]
        s = {"pages": pages, "tokens": list(toks), "finalized": len(hits), "chain": chain}
        self._finalize(s)
        self.seqs[sid] = s
        return len(hits) * ps

    def reserve(self, sid, k):
        s = self.seqs[sid]
        need = -(-(len(s["tokens"]) + k) // self.ps) - len(s["pages"])
        if need > len(self.free) + len(self.lru):
            raise OutOfPages
        for _ in range(max(need, 0)):
            s["pages"].append(self._alloc())

    def commit(self, sid, acc):
        s = self.seqs[sid]
        s["tokens"] += list(acc)
        self._finalize(s)
        keep = -(-len(s["tokens"]) // self.ps)
        rel = 0
        while len(s["pages"]) > keep:
            self._release(s["pages"].pop())
            rel += 1
        return rel

    def release(self, sid):
        for p in reversed(self.seqs.pop(sid)["pages"]):
            self._release(p)
