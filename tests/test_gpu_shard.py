"""GPU parity of the sequence-sharded decode: P ranks are
simulated on one GPU (their exchanges become torch.stack), each rank holding
only its contiguous token slice.  The sharded result must equal the UNSHARDED
one: index sets and scores bit-exact (the oracle, fed the GPU's codes, decides),
outputs within the north_star tolerance."""
import dataclasses

import numpy as np
import pytest
import torch

import synth
from paper_2506_02572_b200.seqshard import SeqShardDecode, shard_range
from tests.hata_testutil import check_decode

pytestmark = pytest.mark.gpu


def _shape(name, **kw):
    return dataclasses.replace(synth.CONFIGS[name], **kw)


def sharded_step(case, k, P, nb=None, out_dtype=torch.float32):
    """Prefill-hash, split into P slices, run one sharded step with the append."""
    import paper_2506_02572_b200 as H
    sh = case["shape"]
    dev = "cuda"
    q = case["q"].to(dev)
    K = case["K"].to(dev).contiguous()
    V = case["V"].to(dev).contiguous()
    W = case["W"].to(dev).contiguous()
    kn, vn = case["k_new"].to(dev), case["v_new"].to(dev)
    nb = (case["n_before"] if nb is None else nb).to(dev)
    B, Hkv, cap, d = K.shape
    Wd = sh.rbits // 32
    codes = torch.zeros(B, Hkv, cap, Wd, dtype=torch.int32, device=dev)
    H.hash_keys(K, W, codes, 0, int(nb.max().item()))
    n = nb + 1
    n_max = int(n.max().item())
    # GPU query codes of the unsharded path (for the oracle's protocol step 2)
    qcodes = torch.zeros(B, sh.Hq, Wd, dtype=torch.int32, device=dev)
    Kf, Vf, cf = K.clone(), V.clone(), codes.clone()
    H.append(kn, vn, W, Kf, Vf, cf, nb)
    ref_idx = torch.full((B, Hkv, k), -7, dtype=torch.int32, device=dev)
    ref_out = H.decode_topk_attn(q, Kf, Vf, cf, W, n, k, n_max=n_max, out_idx=ref_idx, out_qcodes=qcodes)
    # the ranks
    C = (cap + P - 1) // P
    ranks = []
    for r in range(P):
        lo, hi = shard_range(cap, P, r)
        def sl(t):
            s = torch.zeros(B, Hkv, C, t.shape[3], dtype=t.dtype, device=dev)
            s[:, :, :hi - lo] = t[:, :, lo:hi]
            return s
        ranks.append(SeqShardDecode(sl(K), sl(V), sl(codes), W, sh.Hq, k, cap, r, P, out_dtype=out_dtype))
    cands = [rk.phase_local(q, n, n_max, kn, vn) for rk in ranks]
    all_D = torch.stack([c[0] for c in cands])
    all_idx = torch.stack([c[1] for c in cands])
    parts = torch.stack([rk.phase_select_attend(q, n, all_D, all_idx).clone() for rk in ranks])
    outs = [rk.phase_combine(parts).clone() for rk in ranks]
    torch.cuda.synchronize()
    for rk in ranks[1:]:
        assert torch.equal(rk.sel_idx, ranks[0].sel_idx), "ranks disagree on the global selection"
        assert torch.equal(rk.sel_score, ranks[0].sel_score)
    for o in outs[1:]:
        assert torch.equal(o, outs[0]), "ranks disagree on the combined output"
    if not torch.equal(ranks[0].sel_idx, ref_idx):
        bad = (ranks[0].sel_idx != ref_idx).any(-1).nonzero().tolist()
        b, g = bad[0]
        a, r = ranks[0].sel_idx[b, g].cpu().numpy(), ref_idx[b, g].cpu().numpy()
        print("DIFF units", bad, "sharded-only", np.setdiff1d(a, r)[:20], "ref-only", np.setdiff1d(r, a)[:20])
    assert torch.equal(ranks[0].sel_idx, ref_idx), "sharded selection != unsharded selection"
    # reassemble the caches the ranks hold (after the owner's append)
    Kc = torch.cat([rk.K[:, :, :shard_range(cap, P, r)[1] - shard_range(cap, P, r)[0]]
                    for r, rk in enumerate(ranks)], dim=2)
    Vc = torch.cat([rk.V[:, :, :shard_range(cap, P, r)[1] - shard_range(cap, P, r)[0]]
                    for r, rk in enumerate(ranks)], dim=2)
    cc = torch.cat([rk.codes[:, :, :shard_range(cap, P, r)[1] - shard_range(cap, P, r)[0]]
                    for r, rk in enumerate(ranks)], dim=2)
    g = dict(K=Kc.cpu(), V=Vc.cpu(), codes=cc.cpu(), out=outs[0].float().cpu(), idx=ranks[0].sel_idx.cpu(),
             score=ranks[0].sel_score.cpu(), qc=qcodes.cpu(), n=n.cpu())
    err_vs_unsharded = float((outs[0].float() - ref_out.float()).abs().max())
    return g, err_vs_unsharded


CASES = [
    ("g4_8k_P2", _shape("cfg2", N=8192 + 37, k=256), 2, "planted"),
    ("g4_8k_P3", _shape("cfg2", N=8192 + 37, k=256), 3, "planted"),
    ("g4_8k_P8", _shape("cfg2", N=8192 + 37, k=256), 8, "planted"),
    ("g5_r256_P4", _shape("cfg5", B=2, N=6000, k=200), 4, "planted"),
    ("f32_P2", _shape("cfg2", dtype="f32", N=3000, k=100), 2, "plain"),
    ("tie_equal_P4", _shape("cfg2", N=4096, k=500), 4, "equal"),
    ("tie_pool8_P3", _shape("cfg2", N=9000, k=700), 3, "pool8"),
    ("k_gt_local_P8", _shape("cfg2", N=2000, k=1024), 8, "planted"),
]


@pytest.mark.parametrize("name,shape,P,variant", CASES, ids=[c[0] for c in CASES])
def test_shard_parity(name, shape, P, variant):
    case = synth.make_case(shape, seed=21, variant=variant)
    g, e = sharded_step(case, shape.k, P)
    st = check_decode(case, g, shape.k)
    tol = 2e-3 if shape.dtype == "bf16" else 1e-5
    assert e <= tol
    print(name, st, "vs unsharded", e)


def test_shard_parity_ragged_batch():
    """Sequences of different length: some ranks own no token of a sequence."""
    shape = _shape("cfg2", B=3, N=6000, k=400)
    case = synth.make_case(shape, seed=5, cap=6000)
    nb = torch.tensor([5999, 2500, 17], dtype=torch.int64)
    case["n_before"] = nb
    g, e = sharded_step(case, shape.k, 4, nb=nb)
    check_decode(case, g, shape.k)
    assert e <= 2e-3


@pytest.mark.parametrize("P", [2, 8])
def test_shard_parity_cfg4(P):
    """CFG-4 (128K, k=2048) at the bench's shard counts; code rows sampled."""
    shape = synth.CONFIGS["cfg4"]
    case = synth.make_case(shape, seed=1)
    g, e = sharded_step(case, shape.k, P)
    st = check_decode(case, g, shape.k, code_rows_sample=65536)
    assert e <= 2e-3
    print(P, st, e)


def _nccl_worker(port, q):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK="0", WORLD_SIZE="1")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
    try:
        import paper_2506_02572_b200 as H
        from paper_2506_02572_b200.seqshard import SeqShardDecode
        shape = _shape("cfg2", N=8192, k=256)
        case = synth.make_case(shape, seed=23, device="cuda")
        K, V, W = case["K"].contiguous(), case["V"].contiguous(), case["W"].contiguous()
        codes = torch.zeros(1, shape.Hkv, shape.N, 4, dtype=torch.int32, device="cuda")
        H.hash_keys(K, W, codes, 0, shape.N - 1)
        Kf, Vf, cf = K.clone(), V.clone(), codes.clone()
        n = case["n_before"] + 1
        ref_idx = torch.full((1, shape.Hkv, shape.k), -7, dtype=torch.int32, device="cuda")
        ref = H.decode_step(case["q"], case["k_new"], case["v_new"], Kf, Vf, cf, W, n, shape.k, out_idx=ref_idx)
        rk = SeqShardDecode(K, V, codes, W, shape.Hq, shape.k, shape.N, 0, 1)
        # the collective path (NCCL all_gather_into_tensor), eager and captured in a CUDA graph
        out = rk.step(case["q"], n, shape.N, case["k_new"], case["v_new"]).clone()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            rk.step(case["q"], n, shape.N, case["k_new"], case["v_new"])
        torch.cuda.current_stream().wait_stream(s)
        with torch.cuda.graph(g):
            gout = rk.step(case["q"], n, shape.N, case["k_new"], case["v_new"])
        g.replay()
        torch.cuda.synchronize()
        q.put((bool(torch.equal(rk.sel_idx, ref_idx)), float((out - ref).abs().max()), float((gout - ref).abs().max())))
    finally:
        dist.destroy_process_group()


def test_seqshard_nccl_collective_path():
    """The NCCL branch of the exchange (all_gather_into_tensor of the packed
    candidates and of the partials), at world size 1 on one GPU, eagerly and
    inside a CUDA graph: equal to the unsharded fused step."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(port, q))
    p.start()
    same_idx, e_eager, e_graph = q.get(timeout=300)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert same_idx
    assert e_eager <= 2e-3 and e_graph <= 2e-3, (e_eager, e_graph)
