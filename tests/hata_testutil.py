"""Test helpers: run the CUDA path through the C ABI and compare with the
oracle following the north_star parity protocol.  (Tests only.)"""
from __future__ import annotations

import numpy as np
import torch

import oracle.hata_oracle as O

TOL = {"bf16": 2e-3, "f32": 1e-5}


def to_np64(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu", torch.float64).numpy()


def codes_u32(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy().view(np.uint32)


def gpu_step(case: dict, k: int, n_override=None, out_dtype=torch.float32, device="cuda", fused=False,
             workspace=None, kv_pair=False):
    """prefill-hash rows [0, N-1), append row n_before, decode; all via the C ABI.
    fused=True runs append + decode as one hata_decode_step launch.  A reused
    workspace carries the previous launch's threshold hint (fast selection)."""
    import paper_2506_02572_b200 as H
    sh = case["shape"]
    q = case["q"].to(device)
    K = case["K"].to(device).contiguous()
    V = case["V"].to(device).contiguous()
    if kv_pair:   # K and V rows of a token adjacent: [B, H_kv, cap, 2, d]
        kv = torch.stack((K, V), dim=3)
        K, V = kv[:, :, :, 0, :], kv[:, :, :, 1, :]
    W = case["W"].to(device).contiguous()
    kn, vn = case["k_new"].to(device), case["v_new"].to(device)
    nb = (case["n_before"] if n_override is None else n_override).to(device)
    B, Hkv, cap, d = K.shape
    Wd = sh.rbits // 32
    codes = torch.zeros(B, Hkv, cap, Wd, dtype=torch.int32, device=device)
    H.hash_keys(K, W, codes, 0, int(nb.max().item()))
    n = nb + 1
    n_max = int(n.max().item())
    out_idx = torch.full((B, Hkv, k), -7, dtype=torch.int32, device=device)
    out_score = torch.zeros(B, Hkv, k, dtype=torch.int32, device=device)
    qcodes = torch.zeros(B, sh.Hq, Wd, dtype=torch.int32, device=device)
    if fused:
        out = H.decode_step(q, kn, vn, K, V, codes, W, n, k, n_max=n_max, out_dtype=out_dtype, out_idx=out_idx,
                            out_score=out_score, out_qcodes=qcodes, workspace=workspace)
    else:
        H.append(kn, vn, W, K, V, codes, nb)
        out = H.decode_topk_attn(q, K, V, codes, W, n, k, n_max=n_max, out_dtype=out_dtype, out_idx=out_idx,
                                 out_score=out_score, out_qcodes=qcodes, workspace=workspace)
    torch.cuda.synchronize()
    return dict(K=K.cpu(), V=V.cpu(), codes=codes.cpu(), out=out.cpu(), idx=out_idx.cpu(),
                score=out_score.cpu(), qc=qcodes.cpu(), n=n.cpu())


def check_codes(gpu_codes: np.ndarray, K64: np.ndarray, W64: np.ndarray, rows=None):
    """Protocol step 1: GPU codes equal O1 except bits with |projection| < 1e-4.
    gpu_codes/K64 are [R, W] / [R, d] for one KV head.  Returns (mismatch, near_zero, bits)."""
    if rows is not None:
        gpu_codes, K64 = gpu_codes[rows], K64[rows]
    ref, nz = O.hash_encode(K64, W64)
    rbit = W64.shape[1]
    diff = O.bit_unpack(ref, rbit) != O.bit_unpack(gpu_codes, rbit)
    assert not np.any(diff & ~nz), f"{int((diff & ~nz).sum())} code bits differ outside the near-zero band"
    return int(diff.sum()), int(nz.sum()), diff.size


def check_decode(case: dict, g: dict, k: int, code_rows_sample: int | None = None, rng_seed: int = 0):
    """Full parity protocol on one decode step.  Returns stats dict."""
    sh = case["shape"]
    W64 = to_np64(case["W"])
    B, Hkv = sh.B, sh.Hkv
    G = sh.G
    n = g["n"].numpy()
    codes = codes_u32(g["codes"])
    # the oracle's own caches: generator inputs + oracle append (Alg. 3 lines 3-4)
    Wd = sh.rbits // 32
    K64, V64, _, _ = O.append(to_np64(case["K"]), to_np64(case["V"]),
                              np.zeros(case["K"].shape[:3] + (Wd,), np.uint32),
                              to_np64(case["k_new"]), to_np64(case["v_new"]), W64, n - 1)
    for b in range(B):
        nb = int(n[b])
        assert np.array_equal(to_np64(g["K"])[b, :, :nb], K64[b, :, :nb]), "K cache differs after append"
        assert np.array_equal(to_np64(g["V"])[b, :, :nb], V64[b, :, :nb]), "V cache differs after append"
    rng = np.random.default_rng(rng_seed)
    mism = nzc = bits = 0
    for b in range(B):
        for h in range(Hkv):
            nb = int(n[b])
            rows = None
            if code_rows_sample and nb > code_rows_sample:
                rows = np.sort(rng.choice(nb, size=code_rows_sample, replace=False))
                rows[-1] = nb - 1  # always include the appended token
            m, z, nbits = check_codes(codes[b, h, :nb], K64[b, h, :nb], W64[h], rows)
            mism += m; nzc += z; bits += nbits
    assert nzc < 1e-4 * bits, f"near-zero bits {nzc} of {bits}"
    # q codes (protocol step 1 for Q_H)
    q64 = to_np64(case["q"])
    qref, qnz = O.query_codes(q64, W64)
    qg = codes_u32(g["qc"])
    qdiff = O.bit_unpack(qref.reshape(-1, sh.rbits // 32), sh.rbits) != O.bit_unpack(qg.reshape(-1, sh.rbits // 32), sh.rbits)
    assert not np.any(qdiff & ~qnz.reshape(qdiff.shape)), "query code bits differ outside the near-zero band"
    # step 2: GPU codes into O3-O5 -> D, S, idx bit-exact
    res = O.decode(q64, K64, V64, codes, W64, n, k, qc=qg)
    idx = g["idx"].numpy()
    sc = g["score"].numpy()
    for b in range(B):
        kp = min(k, int(n[b]))
        for h in range(Hkv):
            assert np.array_equal(idx[b, h, :kp], res["idx"][b][h]), f"index set differs at b={b} g={h}"
            assert np.all(idx[b, h, kp:] == -1)
            assert np.array_equal(sc[b, h, :kp], res["S"][b][h]), f"scores differ at b={b} g={h}"
    # step 3: same indices -> outputs within tolerance
    err = float(np.max(np.abs(g["out"].double().numpy() - res["out"])))
    tol = TOL[sh.dtype]
    assert err <= tol, f"max abs err {err} > {tol}"
    return dict(code_bit_mismatch=mism, near_zero_bits=nzc, bits=bits, max_abs_err=err)


# ------------------------------------------------------------------------
# Large cases: inputs stay on the GPU; the oracle checks sampled (b, KV head)
# units one by one (north_star: "at full sizes ... sampled outputs the oracle
# can compute one by one").
def check_units(case: dict, res: dict, k: int, units, code_rows_sample: int | None = 65536, rng_seed: int = 0,
                n_dev=None):
    """Parity protocol on the (b, g) units listed.  ``case`` holds the
    generator inputs (any device); ``res`` the GPU results after the step:
    K, V, codes (caches), out, idx, score, qc (device tensors) and n [B]."""
    sh = case["shape"]
    G, Wd = sh.G, sh.rbits // 32
    n = res["n"].cpu().numpy()
    rng = np.random.default_rng(rng_seed)
    errs = []
    for (b, g) in units:
        nb = int(n[b])
        W64 = to_np64(case["W"][g])
        # oracle caches of this unit: generator rows + Alg. 3 line 3-4 append at nb-1
        K64 = to_np64(case["K"][b, g, :nb]); V64 = to_np64(case["V"][b, g, :nb])
        if nb >= 1:
            K64[nb - 1] = to_np64(case["k_new"][b, g]); V64[nb - 1] = to_np64(case["v_new"][b, g])
        assert np.array_equal(to_np64(res["K"][b, g, :nb]), K64), f"K cache differs at {(b, g)}"
        assert np.array_equal(to_np64(res["V"][b, g, :nb]), V64), f"V cache differs at {(b, g)}"
        codes = codes_u32(res["codes"][b, g, :nb])
        rows = None
        if code_rows_sample and nb > code_rows_sample:
            rows = np.sort(rng.choice(nb, size=code_rows_sample, replace=False))
            rows[-1] = nb - 1
        if nb:
            check_codes(codes, K64, W64, rows)
        q64 = to_np64(case["q"][b, g * G:(g + 1) * G])
        qg = codes_u32(res["qc"][b, g * G:(g + 1) * G])
        qref, qnz = O.hash_encode(q64, W64)
        qdiff = O.bit_unpack(qref, sh.rbits) != O.bit_unpack(qg, sh.rbits)
        assert not np.any(qdiff & ~qnz), f"query code bits differ outside the near-zero band at {(b, g)}"
        # protocol step 2 on this unit as a one-unit problem (B = 1, H_kv = 1)
        r1 = O.decode(q64[None], K64[None, None], V64[None, None], codes[None, None], W64[None], np.array([nb]), k,
                      qc=qg[None])
        kp = min(k, nb)
        idx = res["idx"][b, g].cpu().numpy()
        sc = res["score"][b, g].cpu().numpy()
        assert np.array_equal(idx[:kp], r1["idx"][0][0]), f"index set differs at {(b, g)}"
        assert np.all(idx[kp:] == -1)
        assert np.array_equal(sc[:kp], r1["S"][0][0]), f"scores differ at {(b, g)}"
        out = res["out"][b, g * G:(g + 1) * G].double().cpu().numpy()
        ref = r1["out"][0] if nb else np.zeros_like(out)
        err = float(np.max(np.abs(out - ref)))
        assert err <= TOL[sh.dtype], f"max abs err {err} at {(b, g)}"
        errs.append(err)
    return dict(units=len(units), max_abs_err=max(errs) if errs else 0.0)


def resident_setup(case: dict, n_before, kv_pair=False, device="cuda"):
    """Device caches for ``case`` (already on ``device``) with rows [0, n_before)
    hashed by hata_hash_keys; returns dict(K, V, codes, W, nb)."""
    import paper_2506_02572_b200 as H
    sh = case["shape"]
    K, V = case["K"].to(device), case["V"].to(device)
    if kv_pair:
        kv = torch.stack((K, V), dim=3)
        K, V = kv[:, :, :, 0, :], kv[:, :, :, 1, :]
    else:
        K, V = K.clone(), V.clone()
    W = case["W"].to(device).contiguous()
    B, Hkv, cap, d = K.shape
    codes = torch.zeros(B, Hkv, cap, sh.rbits // 32, dtype=torch.int32, device=device)
    nb = n_before.to(device)
    H.hash_keys(K, W, codes, 0, int(nb.max().item()))
    return dict(K=K, V=V, codes=codes, W=W, nb=nb)


def new_outputs(sh, k, device="cuda", out_dtype=torch.float32):
    return dict(out=torch.empty(sh.B, sh.Hq, sh.d, dtype=out_dtype, device=device),
                idx=torch.full((sh.B, sh.Hkv, k), -7, dtype=torch.int32, device=device),
                score=torch.zeros(sh.B, sh.Hkv, k, dtype=torch.int32, device=device),
                qc=torch.zeros(sh.B, sh.Hq, sh.rbits // 32, dtype=torch.int32, device=device))
