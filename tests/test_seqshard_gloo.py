"""World-size-2 (and 3) CPU test of the sequence-sharded orchestration
(paper_2506_02572_b200.seqshard) over torch.distributed ``gloo``.

The CUDA phases are replaced by a CPU stand-in built from the oracle (test
code only), so this checks what the host side owns: the token ranges, which
rank writes the appended row, the rank-major exchange order of candidates and
partials, the ragged / empty-slice cases -- and that the sharded step equals
the UNSHARDED oracle decode (indices exactly; outputs to the fp32 rounding of
the ABI's (m, l, acc) partial buffers).
"""
import dataclasses
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle.hata_oracle as O
import synth
from paper_2506_02572_b200.seqshard import SeqShardDecode, shard_range


class CpuOps:
    """Oracle-based stand-in for the four shard phases + append (same signatures)."""

    @staticmethod
    def append(k_new, v_new, W, K, V, codes, pos):
        Wn = W.double().numpy()
        for b in range(K.shape[0]):
            p = int(pos[b])
            if 0 <= p < K.shape[2]:
                for g in range(K.shape[1]):
                    K[b, g, p] = k_new[b, g]
                    V[b, g, p] = v_new[b, g]
                    c, _ = O.hash_encode(k_new[b, g].double().numpy()[None], Wn[g])
                    codes[b, g, p] = torch.from_numpy(c[0].view(np.int32))

    @staticmethod
    def shard_candidates(q, codes, W, n_local, n_local_max, token_offset, k, cand_D, cand_idx, workspace=None):
        G = q.shape[1] // codes.shape[1]
        qc, _ = O.query_codes(q.double().numpy(), W.double().numpy())
        D = O.score(qc, codes.numpy().view(np.uint32), n_local.numpy(), G)
        cand_D.fill_(0x7FFFFFFF)
        cand_idx.fill_(-1)
        for b in range(codes.shape[0]):
            for g in range(codes.shape[1]):
                if int(n_local[b]) == 0:
                    continue
                idx = O.topk(D[b][g], k)
                cand_D[b, g, :len(idx)] = torch.from_numpy(D[b][g][idx].astype(np.int32))
                cand_idx[b, g, :len(idx)] = torch.from_numpy((idx + token_offset).astype(np.int32))

    @staticmethod
    def shard_select(all_D, all_idx, n_total, lo, hi, G, rbits, own_idx, own_cnt, sel_idx=None, sel_score=None):
        P, B, Hkv, k = all_D.shape
        own_idx.fill_(-1)
        for b in range(B):
            kp = min(k, int(n_total[b]))
            for g in range(Hkv):
                Dv = all_D[:, b, g].reshape(-1).numpy().astype(np.int64)
                iv = all_idx[:, b, g].reshape(-1).numpy().astype(np.int64)
                keep = iv >= 0
                Dv, iv = Dv[keep], iv[keep]
                order = np.lexsort((iv, Dv))[:kp]
                sel = np.sort(iv[order])
                Ds = Dv[order][np.argsort(iv[order])]
                if sel_idx is not None:
                    sel_idx[b, g].fill_(-1)
                    sel_idx[b, g, :kp] = torch.from_numpy(sel.astype(np.int32))
                if sel_score is not None:
                    sel_score[b, g].fill_(0)
                    sel_score[b, g, :kp] = torch.from_numpy(O.similarity(Ds, G, rbits).astype(np.int32))
                mine = sel[(sel >= lo) & (sel < hi)] - lo
                own_cnt[b, g] = len(mine)
                own_idx[b, g, :len(mine)] = torch.from_numpy(mine.astype(np.int32))

    @staticmethod
    def shard_partial_attn(q, K, V, own_idx, own_cnt, k, partial, scale=0.0):
        # partial [S, B, H_q, d+2]: split s takes rows [s*cnt/S, (s+1)*cnt/S) (as the kernel does)
        S = partial.shape[0]
        B, Hq, d = q.shape
        G = Hq // K.shape[1]
        sc = scale or 1.0 / np.sqrt(d)
        for s in range(S):
            for b in range(B):
                for h in range(Hq):
                    g = h // G
                    cnt = int(own_cnt[b, g])
                    rows = own_idx[b, g, cnt * s // S:cnt * (s + 1) // S].long()
                    if len(rows) == 0:
                        partial[s, b, h, 0] = -float("inf")
                        partial[s, b, h, 1:] = 0
                        continue
                    z = (K[b, g, rows].double() @ q[b, h].double()) * sc
                    m = z.max()
                    e = torch.exp(z - m)
                    partial[s, b, h, 0] = m
                    partial[s, b, h, 1] = e.sum()
                    partial[s, b, h, 2:] = e @ V[b, g, rows].double()

    @staticmethod
    def shard_combine(parts, out):
        M = parts[:, :, :, 0].max(dim=0).values
        w = torch.where(parts[:, :, :, 0] == -float("inf"), torch.zeros(()), torch.exp(parts[:, :, :, 0] - M))
        L = (parts[:, :, :, 1] * w).sum(0)
        A = (parts[:, :, :, 2:] * w[..., None]).sum(0)
        out.copy_(A / L[..., None])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case(shape_kw, seed, nb):
    shape = dataclasses.replace(synth.CONFIGS["cfg1"], **shape_kw)
    case = synth.make_case(shape, seed, variant="planted", cap=shape.N)
    case["n_before"] = torch.tensor(nb, dtype=torch.int64)
    return shape, case


def _worker(rank, world, port, shape_kw, seed, nb, resq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shape, case = _case(shape_kw, seed, nb)
        K, V, W = case["K"].double(), case["V"].double(), case["W"].double()
        cap = K.shape[2]
        codes_full, _ = O.hash_keys(K.numpy(), W.numpy())
        codes_full = torch.from_numpy(codes_full.view(np.int32))
        lo, hi = shard_range(cap, world, rank)
        C = (cap + world - 1) // world
        def sl(t):
            s = torch.zeros(t.shape[0], t.shape[1], C, t.shape[3], dtype=t.dtype)
            s[:, :, :hi - lo] = t[:, :, lo:hi]
            return s
        # rows >= n_before are not yet in the cache
        for b in range(shape.B):
            codes_full[b, :, int(nb[b]):] = 0
        rk = SeqShardDecode(sl(K), sl(V), sl(codes_full), W, shape.Hq, shape.k, cap, rank, world, ops=CpuOps,
                            out_dtype=torch.float64, splits=2)
        n = case["n_before"] + 1
        out = rk.step(case["q"].double(), n, int(n.max()), case["k_new"].double(), case["v_new"].double())
        resq.put((rank, out.numpy().copy(), rk.sel_idx.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape_kw,nb", [
    (2, dict(B=2, Hq=4, Hkv=2, N=900, k=64), [899, 450]),
    (2, dict(B=1, Hq=2, Hkv=1, N=300, k=400), [299]),           # k > n: every token selected
    (3, dict(B=3, Hq=4, Hkv=2, N=600, k=50), [599, 150, 3]),     # ragged: ranks with empty slices
])
def test_seqshard_gloo(world, shape_kw, nb):
    seed = 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape_kw, seed, nb, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda x: x[0])
    # the unsharded oracle step on the same inputs
    shape, case = _case(shape_kw, seed, nb)
    K, V, W = (case[x].double().numpy() for x in ("K", "V", "W"))
    codes, _ = O.hash_keys(K, W)
    ref = O.decode_step(case["q"].double().numpy(), case["k_new"].double().numpy(), case["v_new"].double().numpy(),
                        K, V, codes, W, np.array(nb), shape.k)
    for r, out, sel in res:
        assert np.allclose(out, ref["out"], rtol=0, atol=1e-6), f"rank {r} output differs"
        for b in range(shape.B):
            kp = min(shape.k, nb[b] + 1)
            for g in range(shape.Hkv):
                assert np.array_equal(sel[b, g, :kp], ref["idx"][b][g]), f"rank {r} selection differs b={b} g={g}"
