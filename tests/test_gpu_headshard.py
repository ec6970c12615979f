"""GPU parity of the batch/head-sharded decode:
P ranks are simulated on one GPU, each holding only its KV heads (with their
query heads, W slices and caches) and running the fused single-GPU step on
them -- no exchange.  The sharded step must select exactly what the unsharded
step selects (index sets and scores bit-exact) and, unit by unit, pass the
oracle parity protocol; a multi-layer step with the paper's dense first
layers must give dense attention on those layers."""
import dataclasses

import numpy as np
import pytest
import torch

import oracle.hata_oracle as O
import paper_2506_02572_b200 as H
import synth
from paper_2506_02572_b200.headshard import HeadShardDecode, HeadShardModel, head_range
from tests.hata_testutil import check_units, new_outputs, resident_setup, to_np64

pytestmark = pytest.mark.gpu


def _shape(name, **kw):
    return dataclasses.replace(synth.CONFIGS[name], **kw)


def _ranks(st, sh, P, dense=False):
    out = []
    for r in range(P):
        lo, hi = head_range(sh.Hkv, P, r)
        out.append(HeadShardDecode(st["K"][:, lo:hi], st["V"][:, lo:hi], st["codes"][:, lo:hi], st["W"][lo:hi],
                                   sh.G, sh.k, r, P, sh.Hkv, dense=dense))
    return out


@pytest.mark.parametrize("name,shape", [
    ("cfg3_8k", _shape("cfg3", N=8192, k=512)),
    ("cfg5_16k", _shape("cfg5", N=16384, k=512)),
], ids=["cfg3_8k", "cfg5_16k"])
@pytest.mark.parametrize("P", [2, 4, 8])
def test_headshard_equals_unsharded(name, shape, P):
    sh = shape
    case = synth.make_case(sh, seed=41, device="cuda")
    # unsharded reference run on its own caches
    ref_st = resident_setup(case, case["n_before"], kv_pair=True)
    ref_o = new_outputs(sh, sh.k)
    n = ref_st["nb"] + 1
    H.decode_step(case["q"], case["k_new"], case["v_new"], ref_st["K"], ref_st["V"], ref_st["codes"], ref_st["W"], n,
                  sh.k, n_max=sh.N, out=ref_o["out"], out_idx=ref_o["idx"], out_score=ref_o["score"],
                  out_qcodes=ref_o["qc"])
    # P ranks, each on its own head slice of a second copy of the caches
    st = resident_setup(case, case["n_before"], kv_pair=True)
    ranks = _ranks(st, sh, P)
    outs, idxs, scores = [], [], []
    for rk in ranks:
        ix = torch.full((sh.B, rk.Hkv, sh.k), -7, dtype=torch.int32, device="cuda")
        sc = torch.zeros_like(ix)
        o = rk.step(rk.q_slice(case["q"]), rk.kv_slice(case["k_new"]), rk.kv_slice(case["v_new"]), n, sh.N,
                    out_idx=ix, out_score=sc)
        outs.append(o.clone()); idxs.append(ix); scores.append(sc)
    torch.cuda.synchronize()
    idx, score = torch.cat(idxs, dim=1), torch.cat(scores, dim=1)
    assert torch.equal(idx, ref_o["idx"]), "head-sharded selection differs from the unsharded one"
    assert torch.equal(score, ref_o["score"])
    out = torch.cat(outs, dim=1)
    res = dict(K=st["K"], V=st["V"], codes=st["codes"], out=out, idx=idx, score=score, qc=ref_o["qc"], n=n)
    units = [(0, 0), (sh.B - 1, sh.Hkv - 1), (sh.B // 2, sh.Hkv // 2)]
    print(name, P, check_units(case, res, sh.k, units))


def test_headshard_model_dense_first_layers():
    """Three layers, P = 2, the first two dense: dense layers equal
    dense attention over the whole context (oracle O7), the HATA layer passes
    the parity protocol; every layer appends its new key (codes included)."""
    sh = _shape("cfg5", B=2, N=3000, k=128)
    P, L = 2, 3
    cases = [synth.make_case(sh, seed=50 + l, device="cuda") for l in range(L)]
    sts = [resident_setup(c, c["n_before"], kv_pair=True) for c in cases]
    policy = HeadShardModel.dense_policy(L, 2)
    models = []
    for r in range(P):
        lo, hi = head_range(sh.Hkv, P, r)
        models.append(HeadShardModel([
            HeadShardDecode(s["K"][:, lo:hi], s["V"][:, lo:hi], s["codes"][:, lo:hi], s["W"][lo:hi], sh.G, sh.k, r, P,
                            sh.Hkv, dense=policy[l]) for l, s in enumerate(sts)]))
    n = sts[0]["nb"] + 1
    outs = []
    for m in models:
        lay = m.layers
        o = m.step([lay[l].q_slice(c["q"]) for l, c in enumerate(cases)],
                   [lay[l].kv_slice(c["k_new"]) for l, c in enumerate(cases)],
                   [lay[l].kv_slice(c["v_new"]) for l, c in enumerate(cases)], n, sh.N)
        outs.append([x.clone() for x in o])
    torch.cuda.synchronize()
    for l, c in enumerate(cases):
        out = torch.cat([outs[r][l] for r in range(P)], dim=1).double().cpu().numpy()
        K64 = to_np64(sts[l]["K"]); V64 = to_np64(sts[l]["V"])
        W64 = to_np64(c["W"])
        for b in range(sh.B):
            nb = int(n[b])
            for g in (0, sh.Hkv - 1):
                code = sts[l]["codes"][b, g, nb - 1].cpu().numpy().view(np.uint32)
                ref_code, nz = O.hash_encode(to_np64(c["k_new"][b, g])[None], W64[g])
                diff = O.bit_unpack(code[None], sh.rbits) != O.bit_unpack(ref_code, sh.rbits)
                assert not np.any(diff & ~nz), f"layer {l}: appended key code wrong"
                if policy[l]:
                    for h in range(g * sh.G, (g + 1) * sh.G):
                        ref = O.dense_attention(to_np64(c["q"][b, h]), K64[b, g, :nb], V64[b, g, :nb])
                        err = float(np.max(np.abs(out[b, h] - ref)))
                        assert err <= 2e-3, f"dense layer {l} err {err}"
        if not policy[l]:
            o = new_outputs(sh, sh.k)
            # the HATA layer's selection, recomputed unsharded on a fresh copy, must give the same output
            st2 = resident_setup(c, c["n_before"], kv_pair=True)
            H.decode_step(c["q"], c["k_new"], c["v_new"], st2["K"], st2["V"], st2["codes"], st2["W"], n, sh.k,
                          n_max=sh.N, out=o["out"], out_idx=o["idx"], out_score=o["score"], out_qcodes=o["qc"])
            torch.cuda.synchronize()
            res = dict(K=st2["K"], V=st2["V"], codes=st2["codes"], out=o["out"], idx=o["idx"], score=o["score"],
                       qc=o["qc"], n=n)
            check_units(c, res, sh.k, [(0, 0), (1, 7)])
            assert np.max(np.abs(out - o["out"].double().cpu().numpy())) <= 2e-3
