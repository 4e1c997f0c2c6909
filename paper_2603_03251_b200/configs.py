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

# configs[3]: Llama-3.1-70B (TP4 target) — shape only; not runnable on one GPU
LLAMA_70B = dict(vocab=V_LLAMA3, d_model=8192, n_layers=80, n_heads=64, n_kv_heads=8, head_dim=128, ffn=28672)

CONFIGS = {
    "tiny": (TINY_TARGET, TINY_DRAFT),
    "llama8b_1b": (LLAMA_8B, LLAMA_1B),
}


def shapes(name: str, max_ctx: int = 4096):
    t, d = CONFIGS[name]
    return model_shape(**t, max_ctx=max_ctx), model_shape(**d, max_ctx=max_ctx)
