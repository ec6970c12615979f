"""Pins for the CPU oracle (oracle/hata_oracle.py) against things OTHER than
itself: the worked examples in tests/golden/ (SPEC-stated, cited), closed
forms, special cases, textbook identities, brute force on tiny inputs and an
independent library routine (torch SDPA in float64).  Each block names the
mistake it is there to catch.  CPU only.
"""
import itertools
import math
import os

import numpy as np
import pytest
import torch

import oracle.hata_oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
RNG = np.random.default_rng(12345)


def _read_golden(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append([c.strip() for c in line.split("|")])
    return rows


# ---------------------------------------------------------------- codec (O1)
def _golden_inputs(name, rbit):
    """Construct X, W realising each golden case (sign pattern is what is fixed)."""
    d = 8
    W = np.abs(RNG.standard_normal((d, rbit))) + 0.1  # strictly positive
    x = np.abs(RNG.standard_normal((1, d))) + 0.1      # strictly positive
    if name == "all_positive_projection":
        return x, W
    if name == "zero_input":
        return np.zeros((1, d)), RNG.standard_normal((d, rbit))
    if name == "all_negative":
        return -x, W
    if name in ("alternating_signs", "alternating_then_positive"):
        e0 = np.zeros((1, d)); e0[0, 0] = 1.0
        W2 = np.abs(RNG.standard_normal((d, rbit))) + 0.1
        for b in range(32):
            W2[0, b] = 1.0 if b % 2 == 0 else -1.0
        return e0, W2
    raise KeyError(name)


@pytest.mark.parametrize("row", _read_golden("codec_examples.txt"), ids=lambda r: r[0])
def test_codec_golden(row):
    """Catches: wrong bit order (MSB-first), wrong sign(0), wrong word order."""
    name, rbit, _, words = row
    rbit = int(rbit)
    X, W = _golden_inputs(name, rbit)
    codes, _ = O.hash_encode(X, W)
    assert [int(w) for w in codes[0]] == [int(h, 16) for h in words.split()]


def test_bitpack_single_bit_positions():
    """Bit b alone -> word b//32 == 2**(b%32).  Catches off-by-one / MSB-first."""
    rbit = 128
    for b in range(rbit):
        bits = np.zeros((1, rbit), dtype=np.uint8)
        bits[0, b] = 1
        w = O.bit_pack(bits)[0]
        expect = [0] * (rbit // 32)
        expect[b // 32] = 2 ** (b % 32)
        assert [int(v) for v in w] == expect


def test_bitpack_roundtrip():
    bits = RNG.integers(0, 2, size=(50, 256)).astype(np.uint8)
    assert np.array_equal(O.bit_unpack(O.bit_pack(bits), 256), bits)
    with pytest.raises(ValueError):
        O.bit_pack(np.zeros((1, 48), dtype=np.uint8))


def _brute_sign_bits(x, W):
    """Independent re-derivation: exact-rounded dot product (math.fsum) per bit."""
    d, r = W.shape
    out = []
    for b in range(r):
        p = math.fsum(float(x[j]) * float(W[j, b]) for j in range(d))
        out.append((1 if p >= 0 else 0, abs(p)))
    return out


def test_hash_encode_matches_bruteforce():
    """Catches: transposed W, wrong matmul operand, inverted sign test."""
    X = RNG.standard_normal((6, 16))
    W = RNG.standard_normal((16, 64))
    codes, nz = O.hash_encode(X, W)
    bits = O.bit_unpack(codes, 64)
    for i in range(6):
        ref = _brute_sign_bits(X[i], W)
        for b, (bit, mag) in enumerate(ref):
            if mag >= O.NEAR_ZERO:
                assert bits[i, b] == bit
            assert nz[i, b] == (mag < O.NEAR_ZERO)


def test_hash_encode_invariants():
    """Negation flips every bit outside the near-zero set; positive scaling of
    x or of any W column leaves codes unchanged; rows are independent."""
    X = RNG.standard_normal((20, 32))
    W = RNG.standard_normal((32, 128))
    c, nz = O.hash_encode(X, W)
    cn, _ = O.hash_encode(-X, W)
    b1, b2 = O.bit_unpack(c, 128), O.bit_unpack(cn, 128)
    assert np.all((b1 != b2) | nz)
    assert np.array_equal(O.hash_encode(3.5 * X, W)[0], c)
    Ws = W * (np.abs(RNG.standard_normal(128)) + 0.01)[None, :]
    assert np.array_equal(O.hash_encode(X, Ws)[0], c)
    for i in range(20):
        assert np.array_equal(O.hash_encode(X[i:i + 1], W)[0][0], c[i])


# -------------------------------------------------------------- scoring (O4)
def _naive_hamming(a, b, rbit):
    """Per-bit loop on python ints (not XOR/popcount of words)."""
    cnt = 0
    for bit in range(rbit):
        wa = int(a[bit // 32]) >> (bit % 32) & 1
        wb = int(b[bit // 32]) >> (bit % 32) & 1
        cnt += wa != wb
    return cnt


@pytest.mark.parametrize("rbit", [32, 64, 128, 256])
def test_hamming_equals_naive_bit_loop(rbit):
    a = RNG.integers(0, 2**32, size=(200, rbit // 32), dtype=np.uint64).astype(np.uint32)
    b = RNG.integers(0, 2**32, size=(200, rbit // 32), dtype=np.uint64).astype(np.uint32)
    h = O.hamming(a, b)
    for i in range(200):
        assert h[i] == _naive_hamming(a[i], b[i], rbit)


def test_hamming_special_cases():
    a = RNG.integers(0, 2**32, size=(4,), dtype=np.uint64).astype(np.uint32)
    assert O.hamming(a, a) == 0
    assert O.hamming(a, ~a) == 128
    for bit in (0, 5, 31, 32, 127):
        b = a.copy()
        b[bit // 32] ^= np.uint32(1 << (bit % 32))
        assert O.hamming(a, b) == 1


def test_hamming_exhaustive_rbit32_pool():
    """All pairs of a small pool at rbit=32, vs bin().count."""
    pool = [0, 0xFFFFFFFF, 0x55555555, 0xAAAAAAAA, 1, 0x80000000] + \
        [int(v) for v in RNG.integers(0, 2**32, size=26, dtype=np.uint64)]
    arr = np.array(pool, dtype=np.uint32)[:, None]
    for i, x in enumerate(pool):
        h = O.hamming(arr[i:i + 1], arr)
        for j, y in enumerate(pool):
            assert h[j] == bin(x ^ y).count("1")


def _pm1(codes, rbit):
    return 2.0 * O.bit_unpack(codes, rbit).astype(np.float64) - 1.0


@pytest.mark.parametrize("G,rbit", [(1, 128), (4, 128), (5, 256), (2, 64)])
def test_score_pm1_inner_product_identity(G, rbit):
    """sum_h <h(q_h), h(k_t)> = G*rbit - 2*D  (textbook; h in {-1,1}^r).
    Catches: dropped head in the GQA sum, wrong head->group map, per-word bug."""
    Hkv, N, B = 2, 300, 2
    W = rbit // 32
    qc = RNG.integers(0, 2**32, size=(B, Hkv * G, W), dtype=np.uint64).astype(np.uint32)
    codes = RNG.integers(0, 2**32, size=(B, Hkv, N, W), dtype=np.uint64).astype(np.uint32)
    n = np.array([N, N - 17])
    Dl = O.score(qc, codes, n, G)
    for b in range(B):
        for g in range(Hkv):
            kp = _pm1(codes[b, g, :n[b]], rbit)
            ip = sum(kp @ _pm1(qc[b, h][None], rbit)[0] for h in range(g * G, (g + 1) * G))
            assert np.array_equal(O.similarity(Dl[b][g], G, rbit), ip.astype(np.int64))


def test_score_aggregation_properties():
    """Single head -> plain hamming; duplicated heads -> doubled; permuting the
    query heads inside a group leaves D unchanged."""
    rbit, N = 128, 64
    codes = RNG.integers(0, 2**32, size=(1, 1, N, 4), dtype=np.uint64).astype(np.uint32)
    q1 = RNG.integers(0, 2**32, size=(1, 1, 4), dtype=np.uint64).astype(np.uint32)
    D1 = O.score(q1, codes, [N], 1)[0][0]
    assert np.array_equal(D1, np.array([_naive_hamming(q1[0, 0], codes[0, 0, t], rbit) for t in range(N)]))
    q2 = np.concatenate([q1, q1], axis=1)
    assert np.array_equal(O.score(q2, codes, [N], 2)[0][0], 2 * D1)
    q4 = RNG.integers(0, 2**32, size=(1, 4, 4), dtype=np.uint64).astype(np.uint32)
    Da = O.score(q4, codes, [N], 4)[0][0]
    Db = O.score(q4[:, [2, 0, 3, 1]], codes, [N], 4)[0][0]
    assert np.array_equal(Da, Db)


# ---------------------------------------------------------------- top-k (O5)
@pytest.mark.parametrize("row", _read_golden("topk_examples.txt"), ids=lambda r: r[0] + "|" + r[1])
def test_topk_golden(row):
    sims = np.array([int(v) for v in row[0].split()])
    k = int(row[1])
    expect = [int(v) for v in row[2].split()]
    D = sims.max() - sims  # distance; monotone decreasing in similarity (R2)
    assert O.topk(D, k).tolist() == expect


def _brute_topk(D, k):
    """Among ALL subsets of size k', the unique one where every selected (D,t)
    precedes every unselected (D,t) lexicographically."""
    N = len(D)
    kp = min(k, N)
    hits = []
    for S in itertools.combinations(range(N), kp):
        s = set(S)
        rest = [j for j in range(N) if j not in s]
        if all((D[i], i) < (D[j], j) for i in S for j in rest):
            hits.append(list(S))
    assert len(hits) == 1
    return hits[0]


def test_topk_bruteforce_tiny():
    """Catches: tie toward higher index, largest-instead-of-smallest D,
    unsorted output, wrong clamp."""
    for trial in range(300):
        N = int(RNG.integers(1, 9))
        D = RNG.integers(0, 4, size=N)  # heavy ties
        for k in range(1, N + 2):
            assert O.topk(D, k).tolist() == _brute_topk(list(D), k)


def test_topk_properties():
    D = RNG.integers(100, 140, size=5000)
    for k in (1, 64, 1000, 4999, 5000, 7000):
        idx = O.topk(D, k)
        kp = min(k, 5000)
        assert len(idx) == kp and np.all(np.diff(idx) > 0)
        mask = np.zeros(5000, bool); mask[idx] = True
        if kp < 5000:
            T = D[mask].max()
            assert T <= D[~mask].min()                    # min(selected) >= max(rest) in S
            tied_out = np.where(~mask & (D == T))[0]
            tied_in = np.where(mask & (D == T))[0]
            if len(tied_out):
                assert tied_in.max() < tied_out.min()     # lowest index wins
        assert np.array_equal(O.topk(D + 17, k), idx)     # shift invariance
    assert O.topk(np.full(100, 7), 10).tolist() == list(range(10))
    with pytest.raises(ValueError):
        O.topk(D, 0)


def test_topk_chunked_quota_model_equals_sort():
    """Tie-order invariance (north_star): a chunked counting select that visits
    tokens in any chunking (as a GPU/cluster/shard decomposition does) --
    threshold T from the histogram, then per-chunk tie quotas in chunk order --
    yields exactly the sort-based set."""
    for trial in range(50):
        N = int(RNG.integers(50, 3000))
        D = RNG.integers(0, 12, size=N)
        k = int(RNG.integers(1, N + 1))
        ref = O.topk(D, k)
        for nchunks in (1, 3, 7, 16):
            bounds = np.linspace(0, N, nchunks + 1).astype(int)
            hist = np.bincount(D, minlength=13)
            cum = np.cumsum(hist)
            T = int(np.searchsorted(cum, min(k, N)))
            need = min(k, N) - (cum[T - 1] if T > 0 else 0)
            sel = []
            for c in range(nchunks):
                lo, hi = bounds[c], bounds[c + 1]
                ties = np.where(D[lo:hi] == T)[0]
                quota = max(0, min(need, len(ties)))
                need -= quota
                for t in range(lo, hi):
                    if D[t] < T:
                        sel.append(t)
                sel.extend((lo + ties[:quota]).tolist())
            assert sorted(sel) == ref.tolist()


# ------------------------------------------------------------ attention (O6)
def _sdpa64(q, K, V, scale):
    """Library cross-check: torch SDPA in float64."""
    qt = torch.tensor(q, dtype=torch.float64)[None, None, None, :]
    Kt = torch.tensor(K, dtype=torch.float64)[None, None]
    Vt = torch.tensor(V, dtype=torch.float64)[None, None]
    return torch.nn.functional.scaled_dot_product_attention(qt, Kt, Vt, scale=scale)[0, 0, 0].numpy()


def test_attention_special_cases():
    d = 16
    K = RNG.standard_normal((10, d)); V = RNG.standard_normal((10, d)); q = RNG.standard_normal(d)
    assert np.allclose(O.sparse_attention(q, K, V, np.array([0])), V[0], atol=0, rtol=0)  # singleton
    assert np.allclose(O.sparse_attention(q, K, V, np.array([7])), V[7], atol=0, rtol=0)
    Kid = np.repeat(K[:1], 10, axis=0)
    assert np.allclose(O.dense_attention(q, Kid, V), V.mean(0), atol=1e-14)   # identical keys -> mean
    assert np.allclose(O.dense_attention(np.zeros(d), K, V), V.mean(0), atol=1e-14)  # q = 0 -> mean


def test_attention_two_token_closed_form():
    """o = (e^{z0} v0 + e^{z1} v1) / (e^{z0} + e^{z1}), z = q.k / sqrt(d).
    Catches: missing 1/sqrt(d) (Eq. 1), missing max-subtraction bugs."""
    d = 4
    q = np.array([1.0, -2.0, 0.5, 3.0]); K = np.array([[1, 0, 2, 1.], [0, 1, -1, 2.]])
    V = np.array([[1, 2, 3, 4.], [-1, 0, 1, 5.]])
    z0 = (1 * 1 + 0 + 0.5 * 2 + 3 * 1) / 2.0
    z1 = (0 - 2 * 1 - 0.5 + 3 * 2) / 2.0
    w0 = math.exp(z0) / (math.exp(z0) + math.exp(z1))
    expect = w0 * V[0] + (1 - w0) * V[1]
    assert np.allclose(O.dense_attention(q, K, V), expect, atol=1e-14)


def test_attention_vs_sdpa_and_convex_hull():
    d, N = 128, 500
    K = RNG.standard_normal((N, d)); V = RNG.standard_normal((N, d)); q = RNG.standard_normal(d) * 2
    idx = np.sort(RNG.choice(N, size=37, replace=False))
    o = O.sparse_attention(q, K, V, idx)
    assert np.allclose(o, _sdpa64(q, K[idx], V[idx], 1 / math.sqrt(d)), atol=1e-12)
    assert np.all(o <= V[idx].max(0) + 1e-12) and np.all(o >= V[idx].min(0) - 1e-12)
    assert np.allclose(O.sparse_attention(q, K, V, np.arange(N)), _sdpa64(q, K, V, 1 / math.sqrt(d)), atol=1e-12)
    perm = RNG.permutation(N)
    assert np.allclose(O.dense_attention(q, K[perm], V[perm]), O.dense_attention(q, K, V), atol=1e-12)


# ------------------------------------------------------- end to end (Alg. 3)
def _small_case(B=2, Hq=8, Hkv=2, d=32, rbit=64, N=200, seed=0):
    r = np.random.default_rng(seed)
    cap = N + 4
    K = r.standard_normal((B, Hkv, cap, d)); V = r.standard_normal((B, Hkv, cap, d))
    W = r.standard_normal((Hkv, d, rbit)); q = r.standard_normal((B, Hq, d))
    kn = r.standard_normal((B, Hkv, d)); vn = r.standard_normal((B, Hkv, d))
    codes, _ = O.hash_keys(K, W)
    return q, kn, vn, K, V, codes, W


def test_decode_full_budget_equals_dense():
    """k >= N -> output equals dense attention (north_star), per head,
    checked against torch SDPA float64 on the whole cache."""
    q, kn, vn, K, V, codes, W = _small_case()
    nb = np.array([150, 199])
    res = O.decode_step(q, kn, vn, K, V, codes, W, nb, k=10_000)
    G = q.shape[1] // W.shape[0]
    for b in range(2):
        n = nb[b] + 1
        for h in range(q.shape[1]):
            g = h // G
            ref = _sdpa64(q[b, h], res["K"][b, g, :n], res["V"][b, g, :n], 1 / math.sqrt(q.shape[2]))
            assert np.allclose(res["out"][b, h], ref, atol=1e-12)
            assert res["idx"][b][g].tolist() == list(range(n))


def test_decode_first_step_returns_v():
    """First decode on an empty cache -> output == v."""
    q, kn, vn, K, V, codes, W = _small_case()
    res = O.decode_step(q, kn, vn, K, V, codes, W, np.array([0, 0]), k=5)
    G = q.shape[1] // W.shape[0]
    for b in range(2):
        for h in range(q.shape[1]):
            assert np.allclose(res["out"][b, h], vn[b, h // G], atol=0)


def test_decode_appended_token_is_scored_and_codes_consistent():
    """The new key's code is written at row n_before (Alg. 3 line 9) and equals
    HashEncode of the new key; selected sims are the top of the full S."""
    q, kn, vn, K, V, codes, W = _small_case(seed=3)
    nb = np.array([120, 50])
    res = O.decode_step(q, kn, vn, K, V, codes, W, nb, k=16)
    for b in range(2):
        for g in range(W.shape[0]):
            assert np.array_equal(res["codes"][b, g, nb[b]], O.hash_encode(kn[b, g][None], W[g])[0][0])
            D = res["D"][b][g]
            assert len(D) == nb[b] + 1
            sel = res["idx"][b][g]
            rest = np.setdiff1d(np.arange(len(D)), sel)
            assert D[sel].max() <= D[rest].min()


def test_q_w_per_kv_head_mapping():
    """Query head h uses W[h // G] (R4/R5): swapping W of KV head 1 changes only
    the codes of query heads G..2G-1.  Catches h % H_kv style mappings."""
    q, kn, vn, K, V, codes, W = _small_case()
    qc1, _ = O.query_codes(q, W)
    W2 = W.copy(); W2[1] = np.random.default_rng(9).standard_normal(W2[1].shape)
    qc2, _ = O.query_codes(q, W2)
    G = q.shape[1] // W.shape[0]
    assert np.array_equal(qc1[:, :G], qc2[:, :G])
    assert not np.array_equal(qc1[:, G:], qc2[:, G:])


def test_prefill_overhead_and_bytes():
    """HashEncode / attention complexity ratio < 1% at 32K (0.003876)."""
    assert abs(O.prefill_overhead_ratio(32768, 128, 128) - 0.003876) < 1e-6
    assert abs(O.prefill_overhead_ratio(4096, 128, 128) - 0.031008) < 1e-6
    # SURVEY §8(d) table, derived independently of this code.
    assert O.algorithmic_bytes(1, 32, 8, 128, 128, 131072, 2048, 2) == 25_174_016
    assert O.algorithmic_bytes(1, 32, 8, 128, 128, 32768, 1024, 2) == 8_396_800
    assert O.algorithmic_bytes(1, 1, 1, 128, 128, 1024, 64, 4) == 82_432


# --------------------------------------- pins added in round 2 (VERDICT weak #1)
def test_hash_keys_per_kv_head_weights_bruteforce():
    """Alg. 1 lines 2-5 with reading R4 (one W per KV head):
    codes[b, g, t] must equal the sign bits of K[b, g, t] . W[g], re-derived by
    an exact-rounded per-bit dot product (math.fsum), and changing W[1] must
    change only head 1's codes.  Catches: W[0] used for every head, heads
    transposed with batches, a wrong row written."""
    r = np.random.default_rng(21)
    B, Hkv, N, d, rbit = 2, 3, 5, 16, 64
    K = r.standard_normal((B, Hkv, N, d))
    W = r.standard_normal((Hkv, d, rbit))
    codes, nz = O.hash_keys(K, W)
    for b in range(B):
        for g in range(Hkv):
            bits = O.bit_unpack(codes[b, g], rbit)
            for t in range(N):
                for bb, (bit, mag) in enumerate(_brute_sign_bits(K[b, g, t], W[g])):
                    assert nz[b, g, t, bb] == (mag < O.NEAR_ZERO)
                    if mag >= O.NEAR_ZERO:
                        assert bits[t, bb] == bit, (b, g, t, bb)
    W2 = W.copy()
    W2[1] = r.standard_normal(W2[1].shape)
    codes2, _ = O.hash_keys(K, W2)
    assert np.array_equal(codes2[:, [0, 2]], codes[:, [0, 2]])
    assert not np.array_equal(codes2[:, 1], codes[:, 1])


def test_append_writes_exactly_row_pos():
    """Alg. 3 lines 3-4, 7-9: after append, row pos[b] of every
    (b, g) holds k_new / v_new and the brute-force code of k_new under W[g];
    every other row of K, V and codes is unchanged.  Catches: an off-by-one
    row (pos + 1), K and V swapped, the code of the wrong head."""
    r = np.random.default_rng(22)
    B, Hkv, cap, d, rbit = 2, 2, 9, 16, 64
    K = r.standard_normal((B, Hkv, cap, d)); V = r.standard_normal((B, Hkv, cap, d))
    W = r.standard_normal((Hkv, d, rbit))
    codes = r.integers(0, 2**32, size=(B, Hkv, cap, rbit // 32), dtype=np.uint64).astype(np.uint32)
    kn = r.standard_normal((B, Hkv, d)); vn = r.standard_normal((B, Hkv, d))
    pos = np.array([4, 0])
    K2, V2, c2, _ = O.append(K, V, codes, kn, vn, W, pos)
    for b in range(B):
        p = int(pos[b])
        others = [t for t in range(cap) if t != p]
        for g in range(Hkv):
            assert np.array_equal(K2[b, g, p], kn[b, g]) and np.array_equal(V2[b, g, p], vn[b, g])
            assert np.array_equal(K2[b, g, others], K[b, g, others])
            assert np.array_equal(V2[b, g, others], V[b, g, others])
            assert np.array_equal(c2[b, g, others], codes[b, g, others])
            bits = O.bit_unpack(c2[b, g, p][None], rbit)[0]
            for bb, (bit, mag) in enumerate(_brute_sign_bits(kn[b, g], W[g])):
                if mag >= O.NEAR_ZERO:
                    assert bits[bb] == bit


@pytest.mark.parametrize("G,rbit", [(4, 64), (5, 32)])
def test_decode_S_is_group_pm1_inner_product(G, rbit):
    """north_star / R2: the reported S of each selected token is the +-1 inner
    product of its key code with the G query codes of its group, summed over
    the group (P:138 h in {-1,1}^r; P:255 aggregation).  Computed here from
    the unpacked +-1 vectors, not from D.  Catches: S reported with G = 1, a
    missing factor 2, the wrong head range."""
    q, kn, vn, K, V, codes, W = _small_case(Hq=2 * G, Hkv=2, rbit=rbit, seed=5)
    nb = np.array([120, 77])
    res = O.decode_step(q, kn, vn, K, V, codes, W, nb, k=24)
    qc = res["qc"]
    for b in range(2):
        for g in range(2):
            idx = res["idx"][b][g]
            kp = _pm1(res["codes"][b, g, idx], rbit)
            ip = sum(kp @ _pm1(qc[b, h][None], rbit)[0] for h in range(g * G, (g + 1) * G))
            assert np.array_equal(res["S"][b][g], ip.astype(np.int64))
