"""HATA-off (§8(f) NEXT-4): the K and V caches live in
page-locked host memory (mapped into the device address space), the key codes
stay on the GPU; the fused decode step scores on the GPU, appends the new K/V
row into host memory and gathers only the selected rows over the host link.
Parity against the oracle exactly as for device-resident caches."""
import dataclasses

import pytest
import torch

import paper_2506_02572_b200 as H
import synth
from tests.hata_testutil import check_units, new_outputs

pytestmark = pytest.mark.gpu


def _shape(name, **kw):
    return dataclasses.replace(synth.CONFIGS[name], **kw)


@pytest.mark.parametrize("kv_pair", [True, False], ids=["pair", "split"])
@pytest.mark.parametrize("name,shape", [("g4_8k", _shape("cfg2", N=8192 + 37, k=256)),
                                        ("g5_r256_b2", _shape("cfg5", B=2, N=6000, k=200))], ids=["g4_8k", "g5_r256_b2"])
def test_hata_off_parity(name, shape, kv_pair):
    sh = shape
    case = synth.make_case(sh, seed=61, device="cuda")
    W = case["W"].contiguous()
    B, Hkv, cap, d = case["K"].shape
    # prefill on the GPU (keys hashed where they are produced), then offload K/V
    codes = torch.zeros(B, Hkv, cap, sh.rbits // 32, dtype=torch.int32, device="cuda")
    H.hash_keys(case["K"].contiguous(), W, codes, 0, sh.N - 1)
    if kv_pair:
        kv = torch.empty(B, Hkv, cap, 2, d, dtype=case["K"].dtype, pin_memory=True)
        kv[:, :, :, 0] = case["K"].cpu(); kv[:, :, :, 1] = case["V"].cpu()
        K, V = kv[:, :, :, 0], kv[:, :, :, 1]
    else:
        K = case["K"].cpu().pin_memory(); V = case["V"].cpu().pin_memory()
    assert not K.is_cuda and K.is_pinned()
    n = case["n_before"] + 1
    o = new_outputs(sh, sh.k)
    ws = torch.zeros(max(H.decode_workspace_size(B, sh.Hq, Hkv, d, sh.rbits, sh.N, sh.k), 1), dtype=torch.uint8,
                     device="cuda")
    for rep in range(2):
        H.decode_step(case["q"], case["k_new"], case["v_new"], K, V, codes, W, n, sh.k, n_max=sh.N, out=o["out"],
                      out_idx=o["idx"], out_score=o["score"], out_qcodes=o["qc"], workspace=ws)
        torch.cuda.synchronize()
        res = dict(K=K, V=V, codes=codes, out=o["out"], idx=o["idx"], score=o["score"], qc=o["qc"], n=n)
        print(name, check_units(case, res, sh.k, [(b, g) for b in range(B) for g in (0, Hkv - 1)]))
