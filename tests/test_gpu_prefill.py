"""NEXT-1 (Alg. 1): hata_prefill_write writes a prefilled
K/V chunk into the caches and hashes its keys in the same pass (K read once).
Rows [t0, t0+n) must hold the chunk, every other cache row and code row must
be untouched, and the codes must pass the parity protocol against the oracle."""
import dataclasses

import numpy as np
import pytest
import torch

import paper_2506_02572_b200 as H
import synth
from tests.hata_testutil import check_codes, codes_u32, to_np64

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rbits", [128, 256, 64])
@pytest.mark.parametrize("t0,n", [(0, 4096), (1000, 3777), (64, 100)])
def test_prefill_write(rbits, t0, n):
    B, Hkv, d, cap = 2, 4, 128, 6000
    g = torch.Generator(device="cuda").manual_seed(81)
    Ks = torch.randn(B, Hkv, n, d, generator=g, device="cuda").to(torch.bfloat16)
    Vs = torch.randn(B, Hkv, n, d, generator=g, device="cuda").to(torch.bfloat16)
    W = torch.randn(Hkv, d, rbits, generator=g, device="cuda").to(torch.bfloat16)
    kv = torch.full((B, Hkv, cap, 2, d), 7.0, dtype=torch.bfloat16, device="cuda")   # sentinel
    K, V = kv[:, :, :, 0], kv[:, :, :, 1]
    codes = torch.full((B, Hkv, cap, rbits // 32), 0x5A5A5A5A, dtype=torch.int32, device="cuda")
    H.prefill_write(Ks, Vs, W, K, V, codes, t0=t0)
    torch.cuda.synchronize()
    assert torch.equal(K[:, :, t0:t0 + n], Ks) and torch.equal(V[:, :, t0:t0 + n], Vs)
    outside = torch.ones(cap, dtype=torch.bool)
    outside[t0:t0 + n] = False
    assert torch.all(K[:, :, outside] == 7.0) and torch.all(V[:, :, outside] == 7.0)
    assert torch.all(codes[:, :, outside] == 0x5A5A5A5A)
    W64 = to_np64(W)
    for b in range(B):
        for h in range(Hkv):
            check_codes(codes_u32(codes[b, h, t0:t0 + n]), to_np64(Ks[b, h]), W64[h])
    # the same codes as the separate hash of the written cache
    c2 = torch.zeros_like(codes)
    H.hash_keys(K, W, c2, t0, n)
    torch.cuda.synchronize()
    assert torch.equal(c2[:, :, t0:t0 + n], codes[:, :, t0:t0 + n])
