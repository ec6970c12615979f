"""GPU parity of decode-kernel paths the shape sweep in test_gpu_parity.py does
not reach: the global-workspace D spill, the
global rows list, n[b] == 0, the exact launch configuration bench.py times
(CUDA graph of PDL-chained fused steps on one reused workspace, a different q
every step), ragged batches with n_max > n on a reused workspace (hinted
selection on ranks whose chunk is only partly valid), and one workspace reused
while n_max (hence the rank count M) changes.  Large cases keep their inputs on
the GPU and check sampled (b, KV head) units one by one against the oracle."""
import dataclasses

import pytest
import torch

import paper_2506_02572_b200 as H
import synth
from tests.hata_testutil import check_units, new_outputs, resident_setup

pytestmark = pytest.mark.gpu


def _shape(name, **kw):
    return dataclasses.replace(synth.CONFIGS[name], **kw)


def _ws(sh, n_max, k):
    ws = H.decode_workspace_size(sh.B, sh.Hq, sh.Hkv, sh.d, sh.rbits, n_max, k, synth.torch_dtype(sh.dtype))
    return torch.zeros(max(ws, 1), dtype=torch.uint8, device="cuda"), ws


def _fused(case, st, o, n, k, n_max, ws, q=None, kn=None, vn=None):
    H.decode_step(case["q"] if q is None else q, case["k_new"] if kn is None else kn,
                  case["v_new"] if vn is None else vn, st["K"], st["V"], st["codes"], st["W"], n, k, n_max=n_max,
                  out=o["out"], out_idx=o["idx"], out_score=o["score"], out_qcodes=o["qc"], workspace=ws)


def _res(st, o, n):
    return dict(K=st["K"], V=st["V"], codes=st["codes"], out=o["out"], idx=o["idx"], score=o["score"], qc=o["qc"],
                n=n)


def test_global_D_spill():
    """One rank per unit with a 64K-token chunk: D does not fit in shared
    memory and lives in the workspace (the !d_smem path)."""
    sh = _shape("cfg3", N=65536, k=2048)                 # 128 units -> M = 1, chunk 65536
    assert H.decode_ranks(sh.B, sh.Hq, sh.Hkv, sh.d, sh.rbits, sh.N, sh.k) == 1
    ws, wsb = _ws(sh, sh.N, sh.k)
    assert wsb >= sh.B * sh.Hkv * sh.N * 2               # per-unit D arrays in the workspace
    case = synth.make_case(sh, seed=31, device="cuda")
    st = resident_setup(case, case["n_before"])
    o = new_outputs(sh, sh.k)
    n = st["nb"] + 1
    for rep in range(2):                                 # second launch: with the threshold hint
        _fused(case, st, o, n, sh.k, sh.N, ws)
        torch.cuda.synchronize()
        print(check_units(case, _res(st, o, n), sh.k, [(0, 0), (7, 3), (15, 7)], code_rows_sample=8192))


def test_global_rows_list():
    """k' larger than a rank's smem rows list (k = 8192 at CFG-4: up to 7296
    selected rows per rank) -> the rows list lives in the workspace."""
    sh = _shape("cfg4", k=8192)
    case = synth.make_case(sh, seed=32, device="cuda")
    st = resident_setup(case, case["n_before"], kv_pair=True)
    ws, _ = _ws(sh, sh.N, sh.k)
    o = new_outputs(sh, sh.k)
    n = st["nb"] + 1
    for rep in range(2):
        _fused(case, st, o, n, sh.k, sh.N, ws)
        torch.cuda.synchronize()
        print(check_units(case, _res(st, o, n), sh.k, [(0, g) for g in range(sh.Hkv)]))


@pytest.mark.parametrize("N", [3000, 40000], ids=["one_rank_chunks", "multi_rank"])
def test_n_zero_sequence(N):
    """n[b] == 0 (include/hata.h): zero output, out_idx all -1; the other
    sequences of the batch are unaffected."""
    sh = _shape("cfg2", B=3, N=N, k=256)
    case = synth.make_case(sh, seed=33, device="cuda")
    st = resident_setup(case, case["n_before"])
    H.append(case["k_new"], case["v_new"], st["W"], st["K"], st["V"], st["codes"], st["nb"])
    n = torch.tensor([0, N, N // 2], dtype=torch.int64, device="cuda")
    o = new_outputs(sh, sh.k)
    ws, _ = _ws(sh, N, sh.k)
    for rep in range(2):
        H.decode_topk_attn(case["q"], st["K"], st["V"], st["codes"], st["W"], n, sh.k, n_max=N, out=o["out"],
                           out_idx=o["idx"], out_score=o["score"], out_qcodes=o["qc"], workspace=ws)
        torch.cuda.synchronize()
        assert torch.all(o["idx"][0] == -1)
        assert torch.all(o["out"][0] == 0)
        # sequence 2 scores rows [0, N/2): its last row is a generator row
        ref = dict(case, k_new=case["k_new"].clone(), v_new=case["v_new"].clone())
        ref["k_new"][2] = case["K"][2, :, N // 2 - 1]
        ref["v_new"][2] = case["V"][2, :, N // 2 - 1]
        print(check_units(ref, _res(st, o, n), sh.k, [(1, 0), (1, 5), (2, 3)]))


@pytest.mark.parametrize("coop", [0, 1], ids=["plain", "cooperative"])
def test_bench_launch_configuration_varying_q(coop):
    """The exact configuration bench.py times: CFG-4, paired K/V layout, fused
    decode steps chained with programmatic dependent launch inside ONE CUDA
    graph, one workspace reused by every step (threshold hint on), and a
    different q / k_new / v_new every step (3 steps appending rows N-3, N-2,
    N-1).  Every step, on both replays, is checked against the oracle."""
    sh = synth.CONFIGS["cfg4"]
    S = 3
    case = synth.make_case(sh, seed=34, device="cuda")
    N = sh.N
    # steps append rows N-3 .. N-1: the prefill holds rows [0, N-3)
    gen = torch.Generator(device="cuda").manual_seed(340)
    dt = synth.torch_dtype(sh.dtype)
    qs = [(case["q"].float() + torch.randn(case["q"].shape, generator=gen, device="cuda")).to(dt) for _ in range(S)]
    kns = [case["K"][:, :, N - 3 + s].clone() for s in range(S - 1)] + [case["k_new"]]
    vns = [case["V"][:, :, N - 3 + s].clone() for s in range(S - 1)] + [case["v_new"]]
    nb0 = torch.full((sh.B,), N - 3, dtype=torch.int64, device="cuda")
    K0 = case["K"].clone(); V0 = case["V"].clone()
    K0[:, :, N - 3:] = 0; V0[:, :, N - 3:] = 0
    base = dict(case, K=K0, V=V0)
    st = resident_setup(base, nb0, kv_pair=True)
    ws, _ = _ws(sh, N, sh.k)
    outs = [new_outputs(sh, sh.k) for _ in range(S)]
    ns = [nb0 + 1 + s for s in range(S)]
    H.set_option("pdl", 1)
    H.set_option("selection_hint", 1)
    H.set_option("cooperative", coop)
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):                     # warm-up (plans, func attributes) outside capture
        _fused(base, st, outs[0], ns[0], sh.k, N, ws, qs[0], kns[0], vns[0])
    stream.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        for s in range(S):
            _fused(base, st, outs[s], ns[s], sh.k, N, ws, qs[s], kns[s], vns[s])
    for rep in range(2):
        graph.replay()
        torch.cuda.synchronize()
        for s in range(S):
            ref_case = dict(case, q=qs[s], k_new=kns[s], v_new=vns[s], K=K0, V=V0)
            # the oracle appends row n-1 itself; rows of earlier steps come from the generator
            ref_case["K"] = case["K"].clone(); ref_case["V"] = case["V"].clone()
            print(rep, s, check_units(ref_case, _res(st, outs[s], ns[s]), sh.k, [(0, g) for g in range(sh.Hkv)]))
    H.set_option("cooperative", 0)


@pytest.mark.parametrize("variant", ["planted", "pool8"])
def test_ragged_batch_nmax_above_n_reused_workspace(variant):
    """n[b] < n_max (trailing ranks hold partly valid or empty chunks) with
    the workspace reused, so the hinted selection runs on those ranks."""
    sh = _shape("cfg2", B=3, N=8192, k=400)
    case = synth.make_case(sh, seed=35, device="cuda", variant=variant)
    nb = torch.tensor([5999, 4000, 16], dtype=torch.int64, device="cuda")
    for b in range(sh.B):                                # rows >= nb are empty before the append
        case["K"][b, :, int(nb[b]):] = 0
        case["V"][b, :, int(nb[b]):] = 0
    st = resident_setup(case, nb)
    kn = torch.stack([case["k_new"][b] for b in range(sh.B)])
    n = nb + 1
    ws, _ = _ws(sh, sh.N, sh.k)
    o = new_outputs(sh, sh.k)
    for rep in range(3):
        _fused(case, st, o, n, sh.k, sh.N, ws, kn=kn)
        torch.cuda.synchronize()
        # the oracle's caches: generator rows with the new key at row n-1
        ref = dict(case)
        ref["K"] = case["K"].clone(); ref["V"] = case["V"].clone()
        print(check_units(ref, _res(st, o, n), sh.k, [(b, g) for b in range(sh.B) for g in (0, 7)]))


def test_workspace_reused_while_n_max_changes():
    """One workspace (sized for the largest n_max) serves launches whose n_max
    -- hence rank count M and workspace sections -- differ."""
    sh = _shape("cfg2", N=16384, k=300)
    case = synth.make_case(sh, seed=36, device="cuda")
    st = resident_setup(case, case["n_before"])
    H.append(case["k_new"], case["v_new"], st["W"], st["K"], st["V"], st["codes"], st["nb"])
    ws, _ = _ws(sh, sh.N, sh.k)
    Ms = set()
    for n_max in (4096, 16384, 2048, 16384, 8192, 4096):
        Ms.add(H.decode_ranks(sh.B, sh.Hq, sh.Hkv, sh.d, sh.rbits, n_max, sh.k))
        n = torch.full((sh.B,), n_max, dtype=torch.int64, device="cuda")
        o = new_outputs(sh, sh.k)
        H.decode_topk_attn(case["q"], st["K"], st["V"], st["codes"], st["W"], n, sh.k, n_max=n_max, out=o["out"],
                           out_idx=o["idx"], out_score=o["score"], out_qcodes=o["qc"], workspace=ws)
        torch.cuda.synchronize()
        ref = dict(case)
        ref["k_new"] = case["K"][:, :, n_max - 1].clone() if n_max < sh.N else case["k_new"]
        ref["v_new"] = case["V"][:, :, n_max - 1].clone() if n_max < sh.N else case["v_new"]
        print(n_max, check_units(ref, _res(st, o, n), sh.k, [(0, 0), (0, 4), (0, 7)]))
    assert len(Ms) >= 3


def test_noncontiguous_inputs_equal_contiguous():
    """Non-contiguous q / k_new / v_new (head slices of larger tensors) are
    copied by the binding; the copies must stay alive until the launch has
    read them (a freed temporary was once reused by the next copy, so the
    appended K row held v_new)."""
    sh = _shape("cfg2", B=2, N=4096, k=128)
    big = synth.make_case(_shape("cfg2", B=2, Hq=64, Hkv=16, N=4096, k=128), seed=37, device="cuda")
    case = dict(big, q=big["q"][:, 32:], k_new=big["k_new"][:, 8:], v_new=big["v_new"][:, 8:],
                K=big["K"][:, 8:].contiguous(), V=big["V"][:, 8:].contiguous(), W=big["W"][8:].contiguous(), shape=sh)
    assert not case["q"].is_contiguous() and not case["k_new"].is_contiguous()
    outs = []
    for contig in (False, True):
        c = dict(case)
        if contig:
            c.update(q=case["q"].contiguous(), k_new=case["k_new"].contiguous(), v_new=case["v_new"].contiguous())
        st = resident_setup(c, c["n_before"])
        o = new_outputs(sh, sh.k)
        _fused(c, st, o, st["nb"] + 1, sh.k, sh.N, None)
        torch.cuda.synchronize()
        assert torch.equal(st["K"][:, :, sh.N - 1], case["k_new"]) and torch.equal(st["V"][:, :, sh.N - 1], case["v_new"])
        outs.append((o["out"].clone(), o["idx"].clone()))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])


def test_epoch_wrap_keeps_results():
    """The workspace's per-unit epoch (the tag of the exchanged prefix counts
    and partials) is set just below its 32-bit wrap: the launches that wrap it
    (tag 0 is skipped: the zero-filled workspace carries tag 0) stay
    bit-exact in the selection and within tolerance in the output, with the
    threshold hint carried across the wrap."""
    sh = _shape("cfg2", N=16384, k=300)
    case = synth.make_case(sh, seed=37, device="cuda")
    st = resident_setup(case, case["n_before"])
    H.append(case["k_new"], case["v_new"], st["W"], st["K"], st["V"], st["codes"], st["nb"])
    ws, _ = _ws(sh, sh.N, sh.k)
    n = torch.full((sh.B,), sh.N, dtype=torch.int64, device="cuda")
    units = sh.B * sh.Hkv
    for rep in range(4):
        if rep == 1:
            words = ws[:32 * units].view(torch.int32).view(units, 8)
            words[:, 0] = -2                                      # epoch 0xFFFFFFFE: the next launches wrap
        o = new_outputs(sh, sh.k)
        H.decode_topk_attn(case["q"], st["K"], st["V"], st["codes"], st["W"], n, sh.k, n_max=sh.N, out=o["out"],
                           out_idx=o["idx"], out_score=o["score"], out_qcodes=o["qc"], workspace=ws)
        torch.cuda.synchronize()
        epochs = ws[:32 * units].view(torch.int32).view(units, 8)[:, 0].cpu().long() & 0xFFFFFFFF
        print(rep, epochs.tolist()[:2], check_units(case, _res(st, o, n), sh.k, [(0, 0), (0, 3), (0, 7)]))
    assert (epochs == 3).all()                                    # 0xFFFFFFFE -> 0xFFFFFFFF -> 2 -> 3
