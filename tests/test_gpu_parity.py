"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, following
the north_star protocol (codes bit-exact outside the near-zero band; given the
GPU's codes, D/S/index sets bit-exact; outputs within 2e-3 bf16 / 1e-5 fp32)."""
import dataclasses

import pytest
import torch

import synth
from tests.hata_testutil import check_decode, gpu_step

pytestmark = pytest.mark.gpu


def _shape(name, **kw):
    return dataclasses.replace(synth.CONFIGS[name], **kw)


SMALL = [
    ("cfg1", synth.CONFIGS["cfg1"], "planted"),
    ("g4_r128_8k", _shape("cfg2", N=8192 + 37, k=256), "planted"),
    ("g4_r128_ragged_tail", _shape("cfg2", N=5000, k=300, B=2), "planted"),
    ("g5_r256_small", _shape("cfg5", B=2, N=6000, k=200), "planted"),
    ("g1_r32", _shape("cfg1", dtype="bf16", rbits=32, N=3000, k=100), "planted"),
    ("g2_r64", _shape("cfg2", Hq=16, Hkv=8, rbits=64, N=4096, k=128), "planted"),
    ("g8_r128", _shape("cfg2", Hq=64, Hkv=8, N=4000, k=129), "planted"),
    ("f32_g4", _shape("cfg2", dtype="f32", N=3000, k=100), "plain"),
    ("tie_equal", _shape("cfg2", N=4096, k=500), "equal"),
    ("tie_pool8", _shape("cfg2", N=9000, k=700), "pool8"),
    ("tie_dup", _shape("cfg2", N=8192, k=333), "dup"),
    ("k_eq_n_dense", _shape("cfg2", N=2048, k=2048), "planted"),
    ("k_gt_n", _shape("cfg2", N=700, k=1024), "planted"),
    ("n_eq_1", _shape("cfg2", N=1, k=16), "plain"),
]


@pytest.mark.parametrize("name,shape,variant", SMALL, ids=[s[0] for s in SMALL])
@pytest.mark.parametrize("fused", [False, True], ids=["append+decode", "decode_step"])
def test_decode_parity_small(name, shape, variant, fused):
    case = synth.make_case(shape, seed=11, variant=variant)
    g = gpu_step(case, shape.k, fused=fused)
    st = check_decode(case, g, shape.k)
    print(name, st)


@pytest.mark.parametrize("fused", [False, True], ids=["append+decode", "decode_step"])
def test_decode_parity_ragged_batch(fused):
    shape = _shape("cfg2", B=3, N=6000, k=400)
    case = synth.make_case(shape, seed=5, cap=6000)
    nb = torch.tensor([5999, 4000, 17], dtype=torch.int64)
    case["n_before"] = nb
    g = gpu_step(case, shape.k, n_override=nb, fused=fused)
    st = check_decode(case, g, shape.k)
    print(st)


@pytest.mark.parametrize("name", ["cfg2", "cfg4"])
def test_decode_parity_full_size(name):
    """BASELINE sizes, bench launch configuration; codes sampled per head."""
    shape = synth.CONFIGS[name]
    case = synth.make_case(shape, seed=1)
    g = gpu_step(case, shape.k, fused=True)     # the launch bench.py times
    st = check_decode(case, g, shape.k, code_rows_sample=65536)
    print(name, st)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["cfg3", "cfg5"])
def test_decode_parity_full_size_batched(name):
    shape = synth.CONFIGS[name]
    case = synth.make_case(shape, seed=2)
    g = gpu_step(case, shape.k)
    st = check_decode(case, g, shape.k, code_rows_sample=4096)
    print(name, st)


def test_bf16_output_dtype():
    shape = _shape("cfg2", N=3000, k=100)
    case = synth.make_case(shape, seed=3)
    g32 = gpu_step(case, shape.k)
    g16 = gpu_step(case, shape.k, out_dtype=torch.bfloat16)
    assert torch.equal(g32["idx"], g16["idx"])
    assert (g16["out"].float() - g32["out"]).abs().max().item() <= 2 ** -8 * g32["out"].abs().max().item() + 1e-6


def _ws_for(shape, k):
    import paper_2506_02572_b200 as H
    dt = torch.bfloat16 if shape.dtype == "bf16" else torch.float32
    n = shape.N
    ws = H.decode_workspace_size(shape.B, shape.Hq, shape.Hkv, shape.d, shape.rbits, n, k, dt)
    return torch.zeros(max(ws, 1), dtype=torch.uint8, device="cuda")


HINTED = [
    ("g4_r128_8k", _shape("cfg2", N=8192 + 37, k=256), "planted"),
    ("g5_r256_small", _shape("cfg5", B=2, N=6000, k=200), "planted"),
    ("tie_pool8", _shape("cfg2", N=9000, k=700), "pool8"),
    ("tie_dup", _shape("cfg2", N=8192, k=333), "dup"),
    ("cfg2", synth.CONFIGS["cfg2"], "planted"),
    ("m1_b16", _shape("cfg3", N=4096, k=200), "planted"),          # one rank per unit (no exchange)
    ("m1_b16_pool8", _shape("cfg3", N=4096, k=300), "pool8"),
    ("m2_g5_r256_32k", _shape("cfg5", B=8, N=65536, k=1024), "planted"),   # CFG-5 layer: 2 ranks, 32K-token chunks
]


@pytest.mark.parametrize("name,shape,variant", HINTED, ids=[s[0] for s in HINTED])
def test_decode_parity_hinted(name, shape, variant):
    """A reused workspace holds the previous launch's threshold: the second
    launch takes the candidate-bitmap selection; results must not change."""
    ws = _ws_for(shape, shape.k)
    case = synth.make_case(shape, seed=13, variant=variant)
    for _ in range(3):
        g = gpu_step(case, shape.k, fused=True, workspace=ws)
        st = check_decode(case, g, shape.k)
    print(name, st)


@pytest.mark.parametrize("first,second", [("planted", "pool8"), ("pool8", "planted"), ("planted", "dup"),
                                          ("dup", "planted"), ("equal", "planted"), ("planted", "equal")])
@pytest.mark.parametrize("B", [1, 16], ids=["ranks", "one_rank"])
def test_decode_parity_stale_hint(first, second, B):
    """The hint comes from a different problem (higher or lower threshold):
    the selection falls back or scans extra candidates, never changes."""
    shape = _shape("cfg2", B=B, N=12000 if B == 1 else 3000, k=600 if B == 1 else 150)
    ws = _ws_for(shape, shape.k)
    a = synth.make_case(shape, seed=21, variant=first)
    gpu_step(a, shape.k, fused=True, workspace=ws)
    b = synth.make_case(shape, seed=22, variant=second)
    g = gpu_step(b, shape.k, fused=True, workspace=ws)
    st = check_decode(b, g, shape.k)
    print(first, second, st)


KVPAIR = [
    ("g4_r128_8k", _shape("cfg2", N=8192 + 37, k=256), "planted"),
    ("g5_r256_small", _shape("cfg5", B=2, N=6000, k=200), "planted"),
    ("g8_r128", _shape("cfg2", Hq=64, Hkv=8, N=4000, k=129), "planted"),
    ("tie_pool8", _shape("cfg2", N=9000, k=700), "pool8"),
    ("k_eq_n_dense", _shape("cfg2", N=2048, k=2048), "planted"),
    ("cfg4", synth.CONFIGS["cfg4"], "planted"),
]


@pytest.mark.parametrize("name,shape,variant", KVPAIR, ids=[s[0] for s in KVPAIR])
def test_decode_parity_kv_pair(name, shape, variant):
    """K and V rows of a token adjacent in HBM (the bench's cache layout): one
    512-byte bulk copy gathers both; results must not change."""
    case = synth.make_case(shape, seed=17, variant=variant)
    g = gpu_step(case, shape.k, fused=True, kv_pair=True)
    st = check_decode(case, g, shape.k, code_rows_sample=65536 if shape.N > 100000 else None)
    print(name, st)
