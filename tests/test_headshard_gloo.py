"""World-size-2 (and 4) CPU test of the batch/head-sharded orchestration
(paper_2506_02572_b200.headshard) over torch.distributed ``gloo``.

The fused decode step is replaced by a CPU stand-in built from the oracle
(test code only), so this checks what the host side owns: which KV heads,
query heads, W slices and cache slices each rank takes, that the per-rank steps
need no exchange, and the layer policy (dense first layers) of a
multi-layer step.  The head-sharded step must equal the UNSHARDED oracle
decode of every layer (outputs gathered by head; selections exactly).
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
from paper_2506_02572_b200.headshard import HeadShardDecode, HeadShardModel, head_range


class CpuOps:
    """Oracle stand-in for hata_decode_step (same signature as the binding)."""

    @staticmethod
    def decode_step(q, k_new, v_new, K, V, codes, W, n, k, n_max=None, out=None, out_idx=None, out_score=None,
                    workspace=None):
        nb = (n - 1).numpy()
        res = O.decode_step(q.double().numpy(), k_new.double().numpy(), v_new.double().numpy(), K.double().numpy(),
                            V.double().numpy(), codes.numpy().view(np.uint32), W.double().numpy(), nb, k)
        K.copy_(torch.from_numpy(res["K"])); V.copy_(torch.from_numpy(res["V"]))
        codes.copy_(torch.from_numpy(res["codes"].view(np.int32)))
        out.copy_(torch.from_numpy(res["out"]))
        if out_idx is not None:
            out_idx.fill_(-1)
            for b in range(K.shape[0]):
                for g in range(K.shape[1]):
                    sel = res["idx"][b][g]
                    out_idx[b, g, :len(sel)] = torch.from_numpy(sel.astype(np.int32))
        return out


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _layers(shape_kw, L, nb):
    """Per-layer inputs of an L-layer step (layer l: seed 100 + l)."""
    shape = dataclasses.replace(synth.CONFIGS["cfg1"], **shape_kw)
    out = []
    for l in range(L):
        case = synth.make_case(shape, 100 + l, variant="planted", cap=shape.N)
        K, V, W = case["K"].double(), case["V"].double(), case["W"].double()
        codes, _ = O.hash_keys(K.numpy(), W.numpy())
        codes = torch.from_numpy(codes.view(np.int32))
        for b in range(shape.B):
            codes[b, :, int(nb[b]):] = 0        # rows >= n_before are not in the cache yet
        out.append(dict(case=case, K=K, V=V, W=W, codes=codes))
    return shape, out


def _worker(rank, world, port, shape_kw, L, n_dense, nb, resq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shape, lays = _layers(shape_kw, L, nb)
        lo, hi = head_range(shape.Hkv, world, rank)
        policy = HeadShardModel.dense_policy(L, n_dense)
        model = HeadShardModel([
            HeadShardDecode(x["K"][:, lo:hi].clone(), x["V"][:, lo:hi].clone(), x["codes"][:, lo:hi].clone(),
                            x["W"][lo:hi].clone(), shape.G, shape.k, rank, world, shape.Hkv, dense=policy[l],
                            ops=CpuOps, out_dtype=torch.float64)
            for l, x in enumerate(lays)])
        n = torch.tensor(nb, dtype=torch.int64) + 1
        qs = [model.layers[l].q_slice(x["case"]["q"].double()) for l, x in enumerate(lays)]
        kns = [model.layers[l].kv_slice(x["case"]["k_new"].double()) for l, x in enumerate(lays)]
        vns = [model.layers[l].kv_slice(x["case"]["v_new"].double()) for l, x in enumerate(lays)]
        outs = model.step(qs, kns, vns, n, int(n.max()))
        # verification only (not part of the step): gather every rank's heads
        full = []
        for o in outs:
            parts = [torch.empty_like(o) for _ in range(world)]
            dist.all_gather(parts, o.contiguous())
            full.append(torch.cat(parts, dim=1).numpy().copy())
        resq.put((rank, full))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape_kw,L,n_dense,nb", [
    (2, dict(B=2, Hq=8, Hkv=4, N=300, k=32), 3, 2, [299, 120]),
    (4, dict(B=1, Hq=4, Hkv=4, N=200, k=16), 2, 0, [199]),          # one KV head per rank, G = 1
    (2, dict(B=2, Hq=10, Hkv=2, N=150, k=200), 2, 1, [149, 60]),    # G = 5 (Qwen shape), k > n
])
def test_headshard_gloo(world, shape_kw, L, n_dense, nb):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape_kw, L, n_dense, nb, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    shape, lays = _layers(shape_kw, L, nb)
    policy = HeadShardModel.dense_policy(L, n_dense)
    for l, x in enumerate(lays):
        c = x["case"]
        K, V, W = x["K"].numpy(), x["V"].numpy(), x["W"].numpy()
        codes, _ = O.hash_keys(K, W)
        k = shape.N if policy[l] else shape.k
        ref = O.decode_step(c["q"].double().numpy(), c["k_new"].double().numpy(), c["v_new"].double().numpy(),
                            K, V, codes, W, np.array(nb), k)
        if policy[l]:   # dense layer == dense attention over the whole context (O7)
            for b in range(shape.B):
                for h in range(shape.Hq):
                    g = h // shape.G
                    dense = O.dense_attention(c["q"][b, h].double().numpy(), ref["K"][b, g, :nb[b] + 1],
                                              ref["V"][b, g, :nb[b] + 1])
                    assert np.allclose(ref["out"][b, h], dense, atol=1e-12)
        for r, full in res:
            assert np.allclose(full[l], ref["out"], rtol=0, atol=1e-12), f"rank {r} layer {l} differs"


def test_head_range_partition():
    for H_kv, P in [(8, 1), (8, 2), (8, 4), (8, 8), (40, 8)]:
        got = [head_range(H_kv, P, r) for r in range(P)]
        assert got[0][0] == 0 and got[-1][1] == H_kv
        assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
        assert len({hi - lo for lo, hi in got}) == 1
    with pytest.raises(ValueError):
        head_range(8, 3, 0)
