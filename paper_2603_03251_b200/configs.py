"""Model shapes of BASELINE.json's configs (public Llama model-card shapes;
SURVEY.md Appendix A). Random-init weights, synthetic prompts."""
from __future__ import annotations

from .api import model_shape

V_LLAMA3 = 128256

# configs[0]: the tiny pair (8-layer d=512 target, 2-layer d=256 draft)
TINY_TARGET = dict(vocab=32000, d_model=512, n_layers=8, n_heads=8, n_kv_heads=8, head_dim=64, ffn=1536)
TINY_DRAFT = dict(vocab=32000, d_model=256, n_layers=2, n_heads=4, n_kv_heads=4, head_dim=64, ffn=768, tied=True)

# configs[1..2]: Llama-3.1-8B target + Llama-3.2-1B draft
LLAMA_8B = dict(vocab=V_LLAMA3, d_model=4096, n_layers=32, n_heads=32, n_kv_heads=8, head_dim=128, ffn=14336)
LLAMA_1B = dict(vocab=V_LLAMA3, d_model=2048, n_layers=16, n_heads=32, n_kv_heads=8, head_dim=64, ffn=8192, tied=True)

# configs[3]: Llama-3.1-70B target (tensor-parallel over 4 GPUs in the split
# run: bench.py --config llama70b_1b --gpus 8 --tp 4) + Llama-3.2-1B draft.
# 141 GB of bf16 weights: a TP4 shard is 35 GB per GPU.
LLAMA_70B = dict(vocab=V_LLAMA3, d_model=8192, n_layers=80, n_heads=64, n_kv_heads=8, head_dim=128, ffn=28672)

CONFIGS = {
    "tiny": (TINY_TARGET, TINY_DRAFT),
    "llama8b_1b": (LLAMA_8B, LLAMA_1B),
    "llama70b_1b": (LLAMA_70B, LLAMA_1B),
}


def shapes(name: str, max_ctx: int = 4096, target_layers: int = 0, draft_layers: int = 0):
    """target_layers / draft_layers > 0: the same per-layer shapes at reduced
    depth (parity tests on the exact kernel instantiations)."""
    t, d = dict(CONFIGS[name][0]), dict(CONFIGS[name][1])
    if target_layers:
        t["n_layers"] = target_layers
    if draft_layers:
        d["n_layers"] = draft_layers
    return model_shape(**t, max_ctx=max_ctx), model_shape(**d, max_ctx=max_ctx)
