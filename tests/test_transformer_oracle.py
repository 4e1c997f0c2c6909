"""Pins the CPU transformer oracle (oracle/transformer_lm.cpp), which has no
counterpart in the reference: an independent torch-fp32 restatement of the
same synthetic weights (regenerated here in numpy) and the same
decode math must give the same logits."""
import numpy as np
import pytest
import torch

MASK = np.uint64(0xFFFFFFFFFFFFFFFF)
GOLD = np.uint64(0x9E3779B97F4A7C15)


def splitmix(x):
    with np.errstate(over="ignore"):
        x = (x + GOLD) & MASK
        x = ((x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & MASK
        x = ((x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & MASK
        return x ^ (x >> np.uint64(31))


def derive(root, idx):
    with np.errstate(over="ignore"):
        return splitmix((np.uint64(root) + (np.asarray(idx, dtype=np.uint64) + np.uint64(1)) * GOLD) & MASK)


def unit(key, idx):
    h = derive(key, idx)
    top = (h >> np.uint64(32)).astype(np.uint32).view(np.int32)
    return (top >> 8).astype(np.float32) * np.float32(2.0 ** -23)


def bf16(x):
    return torch.from_numpy(np.asarray(x, dtype=np.float32)).to(torch.bfloat16).to(torch.float32)


def tensor_key(seed, tid):
    return int(derive(seed, np.uint64(tid)))


def layer_w(self, dr, p, role, l, kind):
    """oracle layer_elem for a whole logical tensor."""
    d, H, KVH, hd, F = self["d"], self["heads"], self["kv_heads"], self["head_dim"], self["ffn"]
    rows = {0: H * hd, 1: KVH * hd, 2: KVH * hd, 3: d, 4: F, 5: F, 6: d}[kind]
    ind = {3: H * hd, 6: F}.get(kind, d)
    scale = np.float32(1.0) / np.sqrt(np.float32(ind))
    if kind == 3:
        scale = np.float32(p["block_out_scale"]) * scale
    if kind == 6:
        scale = np.float32(p["shared_mlp_scale"] if (role == 1 and l == 0) else p["block_out_scale"]) * scale
    key = tensor_key(p["seed"], (role << 24) | (l << 8) | kind)
    r = np.arange(rows, dtype=np.uint64)[:, None]
    c = np.arange(ind, dtype=np.uint64)[None, :]
    w = bf16(unit(key, r * np.uint64(ind) + c) * scale)
    if role == 0 and l == 0 and kind in (4, 5, 6):
        sub = layer_w(dr, dr, p, 1, 0, kind)
        w[: sub.shape[0], : sub.shape[1]] = sub
    return w


def sign(key, i):
    return np.where(unit(key, np.arange(i, dtype=np.uint64)) < 0, np.float32(-1), np.float32(1))


def build(self, dr, p, role):
    V, d, ds = self["vocab"], self["d"], dr["d"]
    v = np.arange(V, dtype=np.uint64)[:, None]
    S = unit(tensor_key(p["seed"], 0xE0000001), v * np.uint64(ds) + np.arange(ds, dtype=np.uint64)[None, :])
    emb = np.empty((V, d), np.float32)
    head = np.empty((V, d), np.float32)
    emb[:, :ds] = S * np.float32(p["embed_scale"])
    head[:, :ds] = emb[:, :ds]
    if d > ds:
        j = v * np.uint64(d - ds) + np.arange(d - ds, dtype=np.uint64)[None, :]
        emb[:, ds:] = unit(tensor_key(p["seed"], 0xE0000002), j) * np.float32(p["target_private_embed"])
        head[:, ds:] = unit(tensor_key(p["seed"], 0xE0000003), j) * np.float32(p["target_private_head"])
    gs = sign(tensor_key(p["seed"], 0xE0000004), ds)
    g0 = np.ones(d, np.float32)
    if role == 1:
        gn = sign(tensor_key(p["seed"], 0xE0000005), ds)
        fg = np.float32(p["logit_scale"]) * ((np.float32(1) - np.float32(p["draft_gain_mix"])) * gs +
                                              np.float32(p["draft_gain_mix"]) * gn)
    else:
        fg = np.float32(p["logit_scale"]) * np.concatenate([gs, sign(tensor_key(p["seed"], 0xE0000006), d - ds)])
        g0[:ds] = np.sqrt(np.float32(ds) / np.float32(d))
    layers = [[layer_w(self, dr, p, role, l, k) for k in range(7)] for l in range(self["layers"])]
    return bf16(emb), bf16(head), torch.from_numpy(fg.astype(np.float32)), torch.from_numpy(g0), layers


def forward(self, m, ctx):
    emb, head, fg, g0, layers = m
    d, H, KVH, hd = self["d"], self["heads"], self["kv_heads"], self["head_dim"]
    n, half = len(ctx), hd // 2
    inv = torch.tensor([500000.0 ** (-2.0 * i / hd) for i in range(half)], dtype=torch.float64)
    ang = torch.arange(n, dtype=torch.float64)[:, None] * inv[None, :]
    cs, sn = ang.cos().float(), ang.sin().float()

    def norm(x, g=None):
        r = 1.0 / torch.sqrt((x * x).mean(-1, keepdim=True) + 1e-5)
        y = x * r
        return (y * g if g is not None else y).to(torch.bfloat16).float()

    def rope(t):  # [n, heads, hd]
        a, b = t[..., :half], t[..., half:]
        return torch.cat([a * cs[:, None] - b * sn[:, None], b * cs[:, None] + a * sn[:, None]], -1)

    x = emb[torch.tensor(ctx)]
    for li, (wq, wk, wv, wo, wg, wu, wd) in enumerate(layers):
        h = norm(x)
        q = rope((h @ wq.T).view(n, H, hd))
        k = rope((h @ wk.T).view(n, KVH, hd)).to(torch.bfloat16).float()
        v = (h @ wv.T).view(n, KVH, hd).to(torch.bfloat16).float()
        k = k.repeat_interleave(H // KVH, 1)
        v = v.repeat_interleave(H // KVH, 1)
        s = torch.einsum("qhd,khd->hqk", q, k) / np.sqrt(hd)
        s = s + torch.triu(torch.full((n, n), -np.inf), 1)
        o = torch.einsum("hqk,khd->qhd", torch.softmax(s, -1), v).reshape(n, H * hd).to(torch.bfloat16).float()
        x = x + o @ wo.T
        h2 = norm(x, g0 if li == 0 else None)
        g, u = h2 @ wg.T, h2 @ wu.T
        act = (g / (1 + torch.exp(-g)) * u).to(torch.bfloat16).float()
        x = x + act @ wd.T
    return norm(x[-1:], fg) @ head.T


SMALL_T = {"vocab": 512, "d": 128, "layers": 2, "heads": 4, "kv_heads": 2, "head_dim": 32, "ffn": 256, "tied": False}
SMALL_D = {"vocab": 512, "d": 64, "layers": 1, "heads": 2, "kv_heads": 1, "head_dim": 32, "ffn": 128, "tied": True}
PAIR = {"seed": 99, "embed_scale": 1.0, "shared_mlp_scale": 8.0, "block_out_scale": 0.1, "target_private_embed": 0.1,
        "target_private_head": 0.25, "draft_gain_mix": 0.2, "logit_scale": 0.25}


@pytest.fixture(scope="module")
def pair(oracle_lib):
    p = oracle_lib.TfPair(SMALL_T, SMALL_D, PAIR, threads=2)
    yield p
    p.close()


@pytest.mark.parametrize("which", [0, 1])
def test_oracle_logits_match_independent_torch(pair, which):
    torch.set_num_threads(4)
    self = SMALL_T if which == 0 else SMALL_D
    m = build(self, SMALL_D, PAIR, which)
    rng = np.random.default_rng(which)
    for n in (1, 5, 23):
        ctx = rng.integers(0, 512, n).tolist()
        ref = forward(self, m, ctx)[0].numpy()
        got = pair.logits(which, ctx)
        assert np.max(np.abs(ref - got)) < 2e-3, (n, np.max(np.abs(ref - got)))


def test_oracle_weights_match_numpy_generator(pair):
    m = build(SMALL_T, SMALL_D, PAIR, 0)
    rng = np.random.default_rng(5)
    for kind in range(7):
        w = m[4][1][kind].numpy()
        r = rng.integers(0, w.shape[0], 50)
        c = rng.integers(0, w.shape[1], 50)
        bits = pair.weight_bits(0, 1, kind, r.tolist(), c.tolist())
        got = (bits.astype(np.uint32) << 16).view(np.float32)
        assert np.array_equal(got, w[r, c])
    # layer 0 of the target embeds the draft's layer-0 MLP
    md = build(SMALL_D, SMALL_D, PAIR, 1)
    assert torch.equal(m[4][0][4][:128, :64], md[4][0][4])


def test_kv_cache_reuse_is_exact(pair):
    """Longest-common-prefix reuse must not change logits (oracle bookkeeping)."""
    a = pair.logits(0, [1, 2, 3, 4, 5])
    pair.logits(0, [1, 2, 9, 9])
    b = pair.logits(0, [1, 2, 3, 4, 5])
    assert np.array_equal(a, b)
