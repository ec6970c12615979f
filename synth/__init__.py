"""Seeded synthetic inputs for the HATA decode hot path.

Shared by the CUDA path's tests/bench and by the oracle's tests.  This module
holds NO arithmetic of the method (no hashing, scoring, selection or
attention): only shapes, random draws and structure, so that neither side can
inherit a bug from the other through it.

Recipe:
  * K, V ~ N(0, 1), stored bf16 (fp32 for CFG-1).
  * W[g] ~ N(0, 1) per KV head (reading R4), same dtype as K.
  * Queries: per (b, KV head) a base u ~ N(0, 1)^d; q_h = u + 0.5 N(0, 1) for the
    G query heads of the group (correlated GQA heads).
  * Planted relevance (sink / recent / needle structure of real attention):
    rows {0..3} U {N-64..N-1} U ceil(k/8) random rows of every (b, g) get
    K <- 0.5 K + u.
  * Tie-stress variants: "equal" (every key row equal), "pool8" (key rows
    drawn from 8 distinct rows), "dup" (a few rows duplicated across chunk
    boundaries of 1024 tokens).
All draws come from a torch.Generator seeded with ``seed`` on ``device``.
"""
from __future__ import annotations

import dataclasses
import math

import torch


@dataclasses.dataclass(frozen=True)
class Shape:
    name: str
    B: int
    Hq: int
    Hkv: int
    d: int
    rbits: int
    N: int          # context length after the decode step's append
    k: int          # token budget per (b, KV head)
    dtype: str      # "bf16" | "f32"
    note: str = ""

    @property
    def G(self) -> int:
        return self.Hq // self.Hkv


# BASELINE.json configs (shapes only).  CFG-5 is per layer (32 layers per step).
CONFIGS = {
    "cfg1": Shape("cfg1", 1, 1, 1, 128, 128, 1024, 64, "f32", "single KV head, fp32"),
    "cfg2": Shape("cfg2", 1, 32, 8, 128, 128, 32768, 1024, "bf16", "Llama-3.1-8B layer, 32K"),
    "cfg3": Shape("cfg3", 16, 32, 8, 128, 128, 32768, 1024, "bf16", "Llama-3.1-8B, 32K, batch 16"),
    "cfg4": Shape("cfg4", 1, 32, 8, 128, 128, 131072, 2048, "bf16", "Llama-3.1-8B, 128K"),
    "cfg5": Shape("cfg5", 8, 40, 8, 128, 256, 65536, 1024, "bf16", "Qwen2.5-14B layer, 64K, batch 8"),
}


def torch_dtype(name: str) -> torch.dtype:
    return {"bf16": torch.bfloat16, "f32": torch.float32}[name]


def make_case(shape: Shape, seed: int, device="cpu", variant: str = "planted",
              cap: int | None = None):
    """Inputs of one decode step.

    Returns a dict of torch tensors on ``device``:
      q [B, Hq, d], K, V [B, Hkv, cap, d] (rows >= N-1 are zero: the step
      appends row N-1), W [Hkv, d, rbits], k_new, v_new [B, Hkv, d],
      n_before [B] int64 (= N-1), plus the shape.
    variant: "planted" | "plain" | "equal" | "pool8" | "dup".
    """
    B, Hq, Hkv, d, N = shape.B, shape.Hq, shape.Hkv, shape.d, shape.N
    cap = N if cap is None else cap
    dt = torch_dtype(shape.dtype)
    g = torch.Generator(device=device)
    g.manual_seed(seed)

    def randn(*sz):
        return torch.randn(*sz, generator=g, device=device, dtype=torch.float32)

    K = randn(B, Hkv, cap, d)
    V = randn(B, Hkv, cap, d)
    W = randn(Hkv, d, shape.rbits)
    u = randn(B, Hkv, d)
    q = u.repeat_interleave(shape.G, dim=1) + 0.5 * randn(B, Hq, d)

    if variant == "planted":
        n_rand = math.ceil(shape.k / 8)
        for b in range(B):
            for h in range(Hkv):
                rows = torch.randint(4, max(5, N - 64), (n_rand,), generator=g, device=device)
                sel = torch.cat([torch.arange(0, min(4, N), device=device),
                                 torch.arange(max(0, N - 64), N, device=device), rows])
                K[b, h, sel] = 0.5 * K[b, h, sel] + u[b, h]
    elif variant == "equal":
        K[:] = K[:, :, :1, :]
    elif variant == "pool8":
        pick = torch.randint(0, 8, (B, Hkv, cap), generator=g, device=device)
        pool = K[:, :, :8, :].clone()
        K = torch.gather(pool, 2, pick[..., None].expand(B, Hkv, cap, d))
    elif variant == "dup":
        # duplicate a row across every 1024-token chunk boundary
        for b in range(B):
            for h in range(Hkv):
                for s in range(1024, N, 1024):
                    K[b, h, s - 1] = K[b, h, 0]
                    K[b, h, s] = K[b, h, 0]
    elif variant != "plain":
        raise ValueError(variant)

    n_before = torch.full((B,), N - 1, dtype=torch.int64, device=device)
    k_new = K[:, :, N - 1, :].clone()
    v_new = V[:, :, N - 1, :].clone()
    K[:, :, N - 1:, :] = 0
    V[:, :, N - 1:, :] = 0
    return dict(q=q.to(dt), K=K.to(dt), V=V.to(dt), W=W.to(dt), k_new=k_new.to(dt),
                v_new=v_new.to(dt), n_before=n_before, shape=shape)


def random_codes(n_rows: int, rbits: int, seed: int, pool: int | None = None):
    """Random packed codes [n_rows, rbits/32] as int64 tensor holding uint32
    values (torch has no uint32 arithmetic on CPU); ``pool`` draws rows from
    that many distinct rows (massive ties)."""
    g = torch.Generator().manual_seed(seed)
    W = rbits // 32
    if pool is None:
        return torch.randint(0, 2**32, (n_rows, W), generator=g, dtype=torch.int64)
    base = torch.randint(0, 2**32, (pool, W), generator=g, dtype=torch.int64)
    pick = torch.randint(0, pool, (n_rows,), generator=g)
    return base[pick]


def make_training_sequence(n: int, d: int, G: int, seed: int, device="cpu", topics: int = 16,
                           offset: float = 3.0):
    """Synthetic prefill activations of one KV head for hash training (NEXT-3):
    anisotropic keys and queries with a large shared offset (a common key bias
    direction, as in LLM keys) and topic structure (position t belongs to topic
    c(t); its key and its G queries share the topic direction), so exact
    top-k attention is structured and sign(x W) with random W wastes bits on
    the shared offset.  Returns Q [n, G, d], K [n, d] (fp32).  No method
    arithmetic: draws only."""
    g = torch.Generator(device=device)
    g.manual_seed(seed)

    def randn(*sz):
        return torch.randn(*sz, generator=g, device=device, dtype=torch.float32)
    scale = 0.2 + 2.0 * torch.exp(-torch.arange(d, device=device, dtype=torch.float32) / (d / 4))
    mu_k = offset * randn(d)
    mu_q = offset * randn(d)
    topic = 2.0 * randn(topics, d)
    c = torch.randint(0, topics, (n,), generator=g, device=device)
    K = mu_k + scale * (randn(n, d) + topic[c])
    Q = mu_q + scale * (randn(n, G, d) + topic[c][:, None, :])
    return Q, K
