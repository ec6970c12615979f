"""Batch/head-sharded HATA decode across P ranks.

Rank r owns the KV heads [r*H_kv/P, (r+1)*H_kv/P) of every sequence, with the
G query heads that read them (query head h reads KV head h // G, reading R5),
the hash weights W of those heads (one W_H per KV head, R4) and their K, V and
code caches.  A (b, KV head) unit's decode step (Alg. 3) touches
only that unit's data, so the ranks run the single-GPU fused step
(hata_decode_step) on their own heads with NO collective in the data path:
step time = max over ranks.  The attention output stays sharded by head,
which is the layout a tensor-parallel output projection consumes.

``HeadShardModel`` strings L layers together (CFG-5: the 32 attention layers
of one decode step) with the layer policy of the paper's setup, "vanilla
attention for the first two layers": a dense layer runs the same
kernel with k = its whole context, so the selection degenerates to every
token (k = N is dense attention, the O7 check) and the layer still hashes and
appends its new key.

``ops`` defaults to the CUDA library; it exists so that the orchestration
(head ranges, slicing, layer policy) can be exercised by world-size-2
``gloo`` tests on CPU with an oracle stand-in.
"""
from __future__ import annotations

import torch


def head_range(H_kv: int, world: int, rank: int):
    """KV heads [lo, hi) owned by ``rank`` (contiguous, ascending in rank).
    Every rank gets the same count; H_kv must be a multiple of the world size."""
    if H_kv % world:
        raise ValueError(f"H_kv={H_kv} is not a multiple of the world size {world}")
    per = H_kv // world
    return rank * per, (rank + 1) * per


class HeadShardDecode:
    """One attention layer's state on one rank: its KV-head slice.

    K, V: [B, H_kv/P, cap, d] (any strides with d contiguous; K and V share
    them); codes [B, H_kv/P, cap, rbits/32]; W [H_kv/P, d, rbits].  ``G`` is
    the query heads per KV head of the whole model.  ``dense``: attend to every
    token (the paper's dense first layers).
    """

    def __init__(self, K, V, codes, W, G: int, k: int, rank: int, world: int, H_kv_total: int,
                 dense: bool = False, ops=None, out_dtype=torch.float32):
        if ops is None:
            import paper_2506_02572_b200 as ops
        self.ops = ops
        self.K, self.V, self.codes, self.W = K, V, codes, W
        self.B, self.Hkv, self.cap, self.d = K.shape
        self.G, self.rank, self.world = G, rank, world
        self.lo, self.hi = head_range(H_kv_total, world, rank)
        assert self.hi - self.lo == self.Hkv, "local slice does not match the owned head range"
        self.Hq = G * self.Hkv
        self.rbits = W.shape[2]
        self.dense = dense
        self.k = self.cap if dense else k
        dev = K.device
        self.out = torch.empty(self.B, self.Hq, self.d, dtype=out_dtype, device=dev)
        self.workspace = None
        if hasattr(ops, "decode_workspace_size") and K.is_cuda:
            ws = ops.decode_workspace_size(self.B, self.Hq, self.Hkv, self.d, self.rbits, self.cap, self.k, K.dtype)
            self.workspace = torch.zeros(max(ws, 1), dtype=torch.uint8, device=dev)

    # slices of the replicated per-step inputs that belong to this rank
    def q_slice(self, q_full):
        """[B, H_q, d] -> the G*(hi-lo) query heads of this rank's KV heads."""
        return q_full[:, self.lo * self.G:self.hi * self.G]

    def kv_slice(self, x_full):
        """[B, H_kv, d] (k_new / v_new) -> this rank's KV heads."""
        return x_full[:, self.lo:self.hi]

    def step(self, q_local, k_new_local, v_new_local, n, n_max: int, out_idx=None, out_score=None):
        """Alg. 3 lines 2-17 on the owned heads, one fused launch.  ``n``:
        tokens per sequence including the new one (device int64 [B]).
        Returns out [B, G*(hi-lo), d]."""
        k = n_max if self.dense else self.k
        self.ops.decode_step(q_local, k_new_local, v_new_local, self.K, self.V, self.codes, self.W, n, k,
                             n_max=n_max, out=self.out, out_idx=out_idx, out_score=out_score,
                             workspace=self.workspace)
        return self.out


class HeadShardModel:
    """L attention layers of one decode step on one rank (CFG-5: 32 layers).

    layers: list of HeadShardDecode (one per layer, each with its own caches,
    W and workspace).  ``step`` runs them in order -- in a model the q, k_new
    and v_new of layer l come from layer l-1's output through the projections
    (not part of this path), so they are inputs here.
    """

    def __init__(self, layers):
        self.layers = list(layers)

    @staticmethod
    def dense_policy(L: int, n_dense: int = 2):
        """Layer l is dense iff l < n_dense ("vanilla attention for the first
        two layers")."""
        return [l < n_dense for l in range(L)]

    def step(self, qs, kns, vns, n, n_max: int):
        """qs/kns/vns: per-layer LOCAL inputs.  Returns the per-layer outputs."""
        return [lay.step(q, kn, vn, n, n_max) for lay, q, kn, vn in zip(self.layers, qs, kns, vns)]
