"""Paged KV caches ("pluggable into FlashInfer /
vLLM"): K/V and code caches in physical page pools addressed through a block
table, pages scattered in random order.  The fused step must give exactly the
contiguous step's selection and pass the oracle parity protocol on the logical
caches (reassembled from the pools after the step's append)."""
import dataclasses

import pytest
import torch

import paper_2506_02572_b200 as H
import synth
from tests.hata_testutil import check_units, new_outputs, resident_setup

pytestmark = pytest.mark.gpu


def _shape(name, **kw):
    return dataclasses.replace(synth.CONFIGS[name], **kw)


def _paged(case, ps, kv_pair, seed):
    sh = case["shape"]
    B, Hkv, cap, d = case["K"].shape
    maxp = -(-cap // ps)
    npages = B * maxp + 3                                            # a few pages never referenced
    g = torch.Generator().manual_seed(seed)
    perm = torch.randperm(npages, generator=g)[:B * maxp].view(B, maxp).to(torch.int32)
    dt = case["K"].dtype
    if kv_pair:
        kv = torch.zeros(npages, Hkv, ps, 2, d, dtype=dt, device="cuda")
        Kp, Vp = kv[:, :, :, 0], kv[:, :, :, 1]
    else:
        Kp = torch.zeros(npages, Hkv, ps, d, dtype=dt, device="cuda")
        Vp = torch.zeros_like(Kp)
    for b in range(B):
        for lp in range(maxp):
            a, z = lp * ps, min(cap, (lp + 1) * ps)
            pp = int(perm[b, lp])
            Kp[pp, :, :z - a] = case["K"][b, :, a:z]
            Vp[pp, :, :z - a] = case["V"][b, :, a:z]
    codes = torch.zeros(npages, Hkv, ps, sh.rbits // 32, dtype=torch.int32, device="cuda")
    H.hash_keys(Kp, case["W"].contiguous(), codes)                  # the pool viewed as [pages, H_kv, ps, d]
    return Kp, Vp, codes, perm.cuda()


def _logical(pool, pt, cap):
    B, maxp = pt.shape
    ps = pool.shape[2]
    rows = [torch.cat([pool[int(pt[b, lp])] for lp in range(maxp)], dim=1)[:, :cap] for b in range(B)]
    return torch.stack(rows)


CASES = [
    ("g4_9k_ps64_pair", _shape("cfg2", B=2, N=9000, k=300), 64, True),
    ("g4_9k_ps16_split", _shape("cfg2", B=2, N=9000, k=300), 16, False),
    ("g5_r256_ps32", _shape("cfg5", B=2, N=6000, k=200), 32, True),
    ("m1_recycle_ps128", _shape("cfg3", N=20000, k=500), 128, True),     # one rank per unit, ring recycled
    ("cfg4_ps64", synth.CONFIGS["cfg4"], 64, True),
]


@pytest.mark.parametrize("name,shape,ps,kv_pair", CASES, ids=[c[0] for c in CASES])
def test_paged_decode_parity(name, shape, ps, kv_pair):
    sh = shape
    case = synth.make_case(sh, seed=71, device="cuda")
    Kp, Vp, codes, pt = _paged(case, ps, kv_pair, seed=72)
    n = case["n_before"].cuda() + 1
    o = new_outputs(sh, sh.k)
    B, Hkv, cap, d = case["K"].shape
    ws = torch.zeros(max(H.decode_workspace_size(B, sh.Hq, Hkv, d, sh.rbits, sh.N, sh.k), 1), dtype=torch.uint8,
                     device="cuda")
    # the contiguous step on the same inputs (reference selection)
    st = resident_setup(case, case["n_before"], kv_pair=kv_pair)
    ro = new_outputs(sh, sh.k)
    H.decode_step(case["q"], case["k_new"], case["v_new"], st["K"], st["V"], st["codes"], st["W"], n, sh.k,
                  n_max=sh.N, out=ro["out"], out_idx=ro["idx"], out_score=ro["score"], out_qcodes=ro["qc"])
    for rep in range(2):                                              # second launch: with the threshold hint
        H.decode_step_paged(case["q"], case["k_new"], case["v_new"], Kp, Vp, codes, case["W"].contiguous(), pt, n,
                            sh.k, n_max=sh.N, out=o["out"], out_idx=o["idx"], out_score=o["score"],
                            out_qcodes=o["qc"], workspace=ws)
        torch.cuda.synchronize()
        assert torch.equal(o["idx"], ro["idx"]) and torch.equal(o["score"], ro["score"])
        res = dict(K=_logical(Kp, pt, cap), V=_logical(Vp, pt, cap), codes=_logical(codes, pt, cap), out=o["out"],
                   idx=o["idx"], score=o["score"], qc=o["qc"], n=n)
        units = [(0, 0), (B - 1, Hkv - 1)] if B * Hkv > 8 else [(b, g) for b in range(B) for g in range(Hkv)]
        print(name, check_units(case, res, sh.k, units, code_rows_sample=8192))


def test_paged_validation():
    """Non-power-of-two pages, fp32 pools, n_max beyond the table -> errors, nothing launched."""
    sh = _shape("cfg2", N=256, k=16)
    case = synth.make_case(sh, seed=73, device="cuda")
    Kp, Vp, codes, pt = _paged(case, 64, True, seed=74)
    n = case["n_before"].cuda() + 1
    with pytest.raises(H.HataError):
        H.decode_step_paged(case["q"], case["k_new"], case["v_new"], Kp, Vp, codes, case["W"], pt, n, sh.k,
                            n_max=pt.shape[1] * 64 + 1)
    bad = Kp[:, :, :48]                                                 # 48-token pages
    with pytest.raises(H.HataError):
        H.decode_step_paged(case["q"], case["k_new"], case["v_new"], bad, Vp[:, :, :48], codes[:, :, :48],
                            case["W"], pt, n, sh.k, n_max=sh.N)
