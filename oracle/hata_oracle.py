"""HATA decode hot path -- plain, slow, obviously-correct CPU oracle (fp64).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product path (``paper_2506_02572_b200``) never imports it and
shares no code with it (no kernels, helpers, tables or constants).

Citation format: ``P:n`` = /root/reference/PAPER.md line n (HATA, arXiv
2506.02572), ``S:n`` = SPEC.md line n.  Every function follows the paper's
algorithm step by step, in the paper's order and notation; where the paper is
silent the reading taken is the one listed in DESIGN.md "Readings" (R-numbers
below refer to that table).

All floating point is fp64 on exactly-upcast inputs (bf16 -> fp64 and
fp32 -> fp64 are exact).  A library primitive (numpy matmul, a stable sort,
numpy popcount) serves as a single step where noted; there is no blocking,
fusion or reordering beyond the definition.

Layouts (same as the C-ABI):
  q      [B, H_q, d]
  K, V   [B, H_kv, N, d]        (N = cached tokens incl. the appended one)
  W      [H_kv, d, rbits]       (one hash weight per KV head, R4)
  codes  [B, H_kv, N, rbits/32] uint32, LSB-first (R7)
  qc     [B, H_q, rbits/32]     uint32

Parity pinning: every function here is pinned by tests/test_oracle_pins.py
(special cases, closed forms, brute force, library cross-checks).  The only
part with no pin against the *paper itself* is the end-to-end composition:
the paper prints no worked numeric example (P:376, P:389, P:666 are figure
placeholders) -- "parity unpinned vs the paper" for decode_step as a whole;
it is pinned by invariants and degenerate cases only.
"""
from __future__ import annotations

import numpy as np

NEAR_ZERO = 1e-4  # |projection| band whose sign bit may differ (north_star)


# ---------------------------------------------------------------------------
# O1  HashEncode  (Alg. 2)
# ---------------------------------------------------------------------------
def projection(X: np.ndarray, W_H: np.ndarray) -> np.ndarray:
    """MatMul(V, W_H) of Alg. 2 line 5, in fp64.

    X: [s, d], W_H: [d, rbit]  ->  [s, rbit] fp64.
    """
    X = np.asarray(X, dtype=np.float64)
    W_H = np.asarray(W_H, dtype=np.float64)
    return X @ W_H  # library primitive: one matmul


def sign_bits(P: np.ndarray) -> np.ndarray:
    """Sign(...) of Alg. 2 line 5 as {0,1} bits: bit = 1 iff p >= 0.

    h(x) = sign(x W_H) in {-1,+1}^r; +1 <-> bit 1, -1 <-> bit 0;
    sign(0) -> +1 (reading R6).
    """
    return (np.asarray(P) >= 0.0).astype(np.uint8)


def bit_pack(bits: np.ndarray) -> np.ndarray:
    """BitPack of Alg. 2 line 7: [s, rbit] {0,1} -> [s, rbit/32] uint32.

    Bit b lands in word b // 32 at position b % 32 (LSB-first, words in
    ascending bit order; reading R7).  rbit must be a multiple of 32
    ("N^{s x rbit/32}").
    """
    bits = np.asarray(bits, dtype=np.uint64)
    s, r = bits.shape
    if r % 32 != 0:
        raise ValueError("rbit must be a multiple of 32 (P:214)")
    out = np.zeros((s, r // 32), dtype=np.uint64)
    for b in range(r):  # plain loop over bit positions, written out
        out[:, b // 32] |= bits[:, b] << np.uint64(b % 32)
    return out.astype(np.uint32)


def bit_unpack(codes: np.ndarray, rbit: int) -> np.ndarray:
    """Inverse of bit_pack: [s, rbit/32] uint32 -> [s, rbit] {0,1}."""
    codes = np.asarray(codes, dtype=np.uint64)
    s = codes.shape[0]
    bits = np.zeros((s, rbit), dtype=np.uint8)
    for b in range(rbit):
        bits[:, b] = ((codes[:, b // 32] >> np.uint64(b % 32)) & np.uint64(1)).astype(np.uint8)
    return bits


def hash_encode(X: np.ndarray, W_H: np.ndarray):
    """HashEncode (Alg. 2): V_H = BitPack(Sign(MatMul(V, W_H))).

    Returns (codes [s, rbit/32] uint32, near_zero [s, rbit] bool) where
    near_zero marks bits whose |projection| < 1e-4 (north_star: such bits are
    counted and excluded from the bit-exact comparison).
    """
    P = projection(X, W_H)
    codes = bit_pack(sign_bits(P))
    return codes, np.abs(P) < NEAR_ZERO


# ---------------------------------------------------------------------------
# a1 / Alg. 1 lines 2-5  hash the keys of a prefilled cache
# ---------------------------------------------------------------------------
def hash_keys(K: np.ndarray, W: np.ndarray):
    """Alg. 1 lines 2-5: K_H <- HashEncode(K); fill the code cache.

    K: [B, H_kv, N, d], W: [H_kv, d, rbit] -> codes [B, H_kv, N, rbit/32],
    near_zero [B, H_kv, N, rbit].  Key head g uses W[g] (reading R4).
    """
    B, Hkv, N, d = K.shape
    rbit = W.shape[2]
    codes = np.zeros((B, Hkv, N, rbit // 32), dtype=np.uint32)
    nz = np.zeros((B, Hkv, N, rbit), dtype=bool)
    for b in range(B):
        for g in range(Hkv):
            codes[b, g], nz[b, g] = hash_encode(K[b, g], W[g])
    return codes, nz


# ---------------------------------------------------------------------------
# O2  Append  (Alg. 3 lines 2-9)
# ---------------------------------------------------------------------------
def append(K, V, codes, k_new, v_new, W, pos):
    """Alg. 3 lines 3-4 and 7-9: write k_new, v_new and HashEncode(k_new) at
    row pos[b] of every (b, g).  Returns new (K, V, codes) copies plus the
    near-zero mask of the appended codes [B, H_kv, rbit].

    K, V: [B, H_kv, cap, d]; codes: [B, H_kv, cap, rbit/32];
    k_new, v_new: [B, H_kv, d]; pos: [B] int.
    """
    K = np.array(K, copy=True)
    V = np.array(V, copy=True)
    codes = np.array(codes, copy=True)
    B, Hkv = k_new.shape[:2]
    rbit = W.shape[2]
    nz = np.zeros((B, Hkv, rbit), dtype=bool)
    for b in range(B):
        p = int(pos[b])
        for g in range(Hkv):
            K[b, g, p] = k_new[b, g]                       # line 3
            V[b, g, p] = v_new[b, g]                       # line 4
            c, z = hash_encode(k_new[b, g][None, :], W[g])  # line 7
            codes[b, g, p] = c[0]                          # line 9
            nz[b, g] = z[0]
    return K, V, codes, nz


# ---------------------------------------------------------------------------
# O3  Query codes  (Alg. 3 line 6)
# ---------------------------------------------------------------------------
def kv_head_of(h: int, G: int) -> int:
    """Query head h reads KV head floor(h / G) (reading R5)."""
    return h // G


def query_codes(q: np.ndarray, W: np.ndarray):
    """Q_H <- HashEncode(Q) (Alg. 3 line 6), per query head with the
    W of its KV head.  q: [B, H_q, d] -> (qc [B, H_q, rbit/32], near_zero
    [B, H_q, rbit])."""
    B, Hq, d = q.shape
    Hkv, _, rbit = W.shape
    G = Hq // Hkv
    qc = np.zeros((B, Hq, rbit // 32), dtype=np.uint32)
    nz = np.zeros((B, Hq, rbit), dtype=bool)
    for b in range(B):
        for h in range(Hq):
            c, z = hash_encode(q[b, h][None, :], W[kv_head_of(h, G)])
            qc[b, h], nz[b, h] = c[0], z[0]
    return qc, nz


# ---------------------------------------------------------------------------
# O4  Hamming score + GQA aggregation  (Alg. 3 lines 10-11)
# ---------------------------------------------------------------------------
def hamming(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """bitcount(bitwise_xor(a, b)) (Alg. 3 line 11): the
    number of differing bits, word-wise popcount of XOR, summed over words.
    a, b broadcastable [..., rbit/32] uint32 -> [...] int64."""
    x = np.bitwise_xor(np.asarray(a, dtype=np.uint32), np.asarray(b, dtype=np.uint32))
    return np.bitwise_count(x).astype(np.int64).sum(axis=-1)  # library popcount


def score(qc: np.ndarray, codes: np.ndarray, n: np.ndarray, G: int):
    """D[b, g, t] = sum_{h : h // G == g} hamming(qc[b, h], codes[b, g, t])
    for t < n[b] (P:238 per head; "aggregate the scores S for shared
    KVCache" = sum over the G query heads, reading R3; "including the current
    K_H", R11).

    Returns a list over b of int64 arrays [H_kv, n[b]].  The reported
    similarity is S = G*rbit - 2*D (north_star; R2), see similarity().
    """
    B, Hkv = codes.shape[:2]
    out = []
    for b in range(B):
        nb = int(n[b])
        D = np.zeros((Hkv, nb), dtype=np.int64)
        for g in range(Hkv):
            for h in range(g * G, (g + 1) * G):
                D[g] += hamming(qc[b, h][None, :], codes[b, g, :nb])
        out.append(D)
    return out


def similarity(D: np.ndarray, G: int, rbit: int) -> np.ndarray:
    """S = G*rbit - 2*D: the summed +-1 inner product of the hash codes
    (north_star "rbits minus twice the differing sign bits", per head)."""
    return G * rbit - 2 * np.asarray(D, dtype=np.int64)


# ---------------------------------------------------------------------------
# O5  Top-k  (Alg. 3 lines 12-13)
# ---------------------------------------------------------------------------
def topk(D: np.ndarray, k: int) -> np.ndarray:
    """Idx <- TopK(S, k) on one (b, g) row of distances D [N].

    Reading R1: the k most *similar* keys = smallest D.  R8: ties go to the
    lowest index.  R10: k' = min(k, N); k < 1 is an error.  R9: the result is
    returned sorted ascending.

    Step by step: stable-sort t in [0, N) by the key (D[t] asc, t asc), take
    the first k', sort ascending.
    """
    if k < 1:
        raise ValueError("empty selection (k < 1)")
    D = np.asarray(D, dtype=np.int64)
    N = D.shape[0]
    kp = min(k, N)
    t = np.arange(N)
    order = np.lexsort((t, D))  # primary key D, secondary key t (library sort)
    return np.sort(order[:kp]).astype(np.int64)


# ---------------------------------------------------------------------------
# O6  Sparse attention  (Alg. 3 lines 14-17; Eq. 1-2)
# ---------------------------------------------------------------------------
def sparse_attention(q_h: np.ndarray, K: np.ndarray, V: np.ndarray, idx: np.ndarray,
                     scale: float | None = None) -> np.ndarray:
    """O = Attention(Q, K^sparse, V^sparse) with K^sparse = Gather(K, Idx)
    (P:241-244), Attention = Softmax(q K^T / sqrt(d)) V (Eq. 1; R12).

    q_h: [d]; K, V: [N, d]; idx: [k'] -> [d] fp64.
    """
    q_h = np.asarray(q_h, dtype=np.float64)
    Ks = np.asarray(K, dtype=np.float64)[idx]   # Gather(K^cache, Idx)
    Vs = np.asarray(V, dtype=np.float64)[idx]   # Gather(V^cache, Idx)
    d = q_h.shape[0]
    if scale is None:
        scale = 1.0 / np.sqrt(d)
    z = scale * (Ks @ q_h)                       # q K^T / sqrt(d)
    m = z.max()
    p = np.exp(z - m)                            # softmax numerator (max-subtracted)
    return (p @ Vs) / p.sum()


def dense_attention(q_h, K, V, scale=None):
    """O7: Eq. 1 over the whole cache: sparse_attention with Idx = [0, N)."""
    return sparse_attention(q_h, K, V, np.arange(np.asarray(K).shape[0]), scale)


# ---------------------------------------------------------------------------
# Alg. 3 lines 10-17 for a whole batch (the decode hot path after append)
# ---------------------------------------------------------------------------
def decode(q, K, V, codes, W, n, k, scale=None, qc=None):
    """HATA decode (Alg. 3 lines 6, 10-17) over caches
    that already hold the appended token (n[b] = tokens incl. the new one).

    If ``qc`` is given it is used as Q_H (parity protocol step 2: feed the
    GPU's codes, north_star); otherwise Q_H = HashEncode(q).

    Returns dict(out [B, H_q, d] fp64, idx list over b of [H_kv, k'] int64,
    D list over b of [H_kv, n[b]], S = similarity of the selected tokens,
    qc [B, H_q, W]).
    """
    q = np.asarray(q)
    B, Hq, d = q.shape
    Hkv, _, rbit = W.shape
    G = Hq // Hkv
    if qc is None:
        qc, _ = query_codes(q, W)                                  # line 6
    Dl = score(qc, codes, n, G)                                     # lines 10-11
    out = np.zeros((B, Hq, d), dtype=np.float64)
    idx_all, S_all = [], []
    for b in range(B):
        nb = int(n[b])
        idx_b = np.zeros((Hkv, min(k, nb)), dtype=np.int64)
        S_b = np.zeros_like(idx_b)
        for g in range(Hkv):
            idx = topk(Dl[b][g], k)                                 # lines 12-13
            idx_b[g] = idx
            S_b[g] = similarity(Dl[b][g][idx], G, rbit)
            for h in range(g * G, (g + 1) * G):                     # lines 14-17
                out[b, h] = sparse_attention(q[b, h], K[b, g, :nb], V[b, g, :nb], idx, scale)
        idx_all.append(idx_b)
        S_all.append(S_b)
    return dict(out=out, idx=idx_all, D=Dl, S=S_all, qc=qc)


def decode_step(q, k_new, v_new, K, V, codes, W, n_before, k, scale=None):
    """Alg. 3 in full: append (lines 2-9) then decode
    (lines 10-17).  n_before[b] = tokens cached before this step; the new
    token lands at row n_before[b] and is scored (R11)."""
    pos = np.asarray(n_before, dtype=np.int64)
    K2, V2, c2, _ = append(K, V, codes, k_new, v_new, W, pos)
    res = decode(q, K2, V2, c2, W, pos + 1, k, scale)
    res.update(K=K2, V=V2, codes=c2)
    return res


# ---------------------------------------------------------------------------
# Algorithmic bytes (north_star roofline definition)
# ---------------------------------------------------------------------------
def algorithmic_bytes(B, Hq, Hkv, d, rbit, N, k, elem_bytes):
    """codes + k' selected K and V rows + q, per decode step."""
    kp = min(k, N)
    return B * Hkv * N * rbit // 8 + B * Hkv * kp * 2 * d * elem_bytes + B * Hq * d * elem_bytes


def prefill_overhead_ratio(s, d, rbit):
    """HashEncode O(s*d*rbit) vs attention O(s^2 d + s^2)."""
    return (s * d * rbit) / (s * s * d + s * s)
