"""Sequence-sharded HATA decode across P ranks.

Rank r owns the contiguous global token range [r*C, (r+1)*C) of every
(b, KV head), C = ceil(cap_total / P), for the K, V and code caches; q and W
are replicated.  One decode step (Alg. 3, split over token ranges):

  0. append   the rank holding row n[b]-1 writes k_new/v_new and its key code
              (Alg. 3 lines 2-9) -- hata_append, rows of other ranks skipped;
  1. local    q-hash + Hamming score + local top-k' candidates (D, global idx)
              (Alg. 3 lines 6, 10-13 on the slice) -- hata_shard_candidates,
              written into ONE packed [2, B, H_kv, k] int32 buffer (D | idx);
  C1          one all-gather of the packed candidates (NCCL; 8 B x k per (b, g)
              per rank);
  2. select   global k' smallest (D, idx) -- identical on every rank, and equal
              to the unsharded selection: any global top-k' token is in its
              shard's local top-k', and because ranges ascend with the rank,
              "lowest index wins" (R8) is "lower rank first, then local order"
              -- hata_shard_select;
  3. partial  attention over the own selected rows, split over S CTAs per
              (b, g) on the tensor cores -> S x (m, l, acc) -- hata_shard_partial_attn;
  C2          all-gather of the partials (fp32, S x (d+2) x H_q per b per rank);
  4. combine  rank- then split-ordered flash-decoding merge -- hata_shard_combine.

Every step is stream-ordered with no host synchronisation, so a whole step
(kernels and NCCL collectives) can be captured in one CUDA graph.

The collectives are the only host-visible exchange; every arithmetic step is
one of libhata's kernels.  ``ops`` defaults to the CUDA library; it exists so
that the orchestration (ranges, ownership of the append slot, exchange order)
can be exercised by world-size-2 ``gloo`` tests on CPU with a stand-in.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(cap_total: int, world: int, rank: int):
    """Global token range [lo, hi) owned by ``rank`` (contiguous, ascending in rank)."""
    C = (cap_total + world - 1) // world
    lo = min(rank * C, cap_total)
    return lo, min(lo + C, cap_total)


def _all_gather(t: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """Rank-major stack [P, ...] of ``t`` from every rank (NCCL: one
    all_gather_into_tensor, also at world size 1 when a process group exists)."""
    if not dist.is_initialized():
        assert world == 1
        return t.unsqueeze(0)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        dist.all_gather_into_tensor(out, t.contiguous(), group=group)
        return out
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t.contiguous(), group=group)
    return torch.stack(parts)


class SeqShardDecode:
    """Per-rank state of the sequence-sharded decode step (buffers preallocated).

    K, V: this rank's [B, H_kv, C, d] slices; codes: [B, H_kv, C, rbits//32];
    W: [H_kv, d, rbits] (replicated).  ``cap_total`` is the global row capacity.
    """

    def __init__(self, K, V, codes, W, Hq: int, k: int, cap_total: int, rank: int, world: int, group=None,
                 ops=None, out_dtype=torch.float32, splits: int | None = None):
        if ops is None:
            import paper_2506_02572_b200 as ops
        self.ops = ops
        self.K, self.V, self.codes, self.W = K, V, codes, W
        self.B, self.Hkv, self.C, self.d = K.shape
        self.Hq, self.k = Hq, k
        self.G = Hq // self.Hkv
        self.rbits = W.shape[2]
        self.rank, self.world, self.group = rank, world, group
        self.lo, self.hi = shard_range(cap_total, world, rank)
        assert self.hi - self.lo <= self.C, "local slice smaller than the owned range"
        dev = K.device
        B, Hkv = self.B, self.Hkv
        self.cand = torch.empty(2, B, Hkv, k, dtype=torch.int32, device=dev)   # packed (D | idx): one collective
        self.cand_D, self.cand_idx = self.cand[0], self.cand[1]
        self.own_idx = torch.empty(B, Hkv, k, dtype=torch.int32, device=dev)
        self.own_cnt = torch.empty(B, Hkv, dtype=torch.int32, device=dev)
        self.sel_idx = torch.empty(B, Hkv, k, dtype=torch.int32, device=dev)
        self.sel_score = torch.empty(B, Hkv, k, dtype=torch.int32, device=dev)
        if splits is None:   # CTAs per (b, KV head) for the partial attention: fill the SMs once
            sms = torch.cuda.get_device_properties(dev).multi_processor_count if K.is_cuda else 1
            splits = max(1, min(16, sms // max(1, B * Hkv)))
        self.splits = splits
        self.partial = torch.empty(splits, B, Hq, self.d + 2, dtype=torch.float32, device=dev)
        self.out = torch.empty(B, Hq, self.d, dtype=out_dtype, device=dev)
        self.workspace = None
        if hasattr(ops, "decode_workspace_size") and K.is_cuda:
            ws = ops.decode_workspace_size(B, Hq, Hkv, self.d, self.rbits, max(self.hi - self.lo, 1), k, K.dtype)
            self.workspace = torch.zeros(max(ws, 1), dtype=torch.uint8, device=dev)

    def local_sizes(self, n: torch.Tensor):
        """n: global tokens per sequence (device int64 [B]) -> (n_local, pos_local of row n-1)."""
        n_local = (n - self.lo).clamp(0, self.hi - self.lo)
        pos_local = n - 1 - self.lo            # outside [0, C) -> the append kernel skips the row
        return n_local, pos_local

    # the three local phases between the two exchanges (also driven directly by
    # the single-GPU loopback test, which stacks the ranks' tensors itself)
    def phase_local(self, q, n, n_max: int, k_new=None, v_new=None):
        """Steps 0-1: append (owner rank only) + local candidates -> (cand_D, cand_idx)."""
        ops = self.ops
        n_local, pos_local = self.local_sizes(n)
        if k_new is not None:
            ops.append(k_new, v_new, self.W, self.K, self.V, self.codes, pos_local)
        nl_max = max(0, min(n_max, self.hi) - self.lo)
        if nl_max > 0:
            ops.shard_candidates(q, self.codes, self.W, n_local, nl_max, self.lo, self.k, self.cand_D,
                                 self.cand_idx, workspace=self.workspace)
        else:
            self.cand_D.fill_(0x7FFFFFFF)
            self.cand_idx.fill_(-1)
        return self.cand_D, self.cand_idx

    def phase_select_attend(self, q, n, all_D, all_idx, scale: float = 0.0):
        """Steps 2-3: global selection from the gathered candidates + own partial."""
        ops = self.ops
        ops.shard_select(all_D, all_idx, n, self.lo, self.hi, self.G, self.rbits, self.own_idx, self.own_cnt,
                         self.sel_idx, self.sel_score)
        ops.shard_partial_attn(q, self.K, self.V, self.own_idx, self.own_cnt, self.k, self.partial, scale=scale)
        return self.partial

    def phase_combine(self, parts):
        """Step 4: rank-ordered (then split-ordered) combine of the gathered
        partials [P, S, B, H_q, d+2]."""
        self.ops.shard_combine(parts.reshape(-1, *parts.shape[-3:]), self.out)
        return self.out

    def step(self, q, n, n_max: int, k_new=None, v_new=None, scale: float = 0.0):
        """One decode step; returns out [B, H_q, d] (identical on every rank)."""
        self.phase_local(q, n, n_max, k_new, v_new)
        allc = _all_gather(self.cand, self.world, self.group)          # [P, 2, B, H_kv, k]
        part = self.phase_select_attend(q, n, allc[:, 0], allc[:, 1], scale)
        return self.phase_combine(_all_gather(part, self.world, self.group))
