"""NEXT-3: learning-to-hash (Eq. 9; App. A).  CPU
checks of the loss terms against a direct re-derivation, of the data
sampling rule, and that a short training run lowers the loss."""
import math

import torch

import synth
from paper_2506_02572_b200 import hashtrain as HT


def test_hash_loss_terms_match_definition():
    """Eq. 9 written out with explicit loops over queries, keys and bits."""
    g = torch.Generator().manual_seed(0)
    d, r = 6, 4
    W = torch.randn(d, r, generator=g, dtype=torch.float64)
    trip = [(torch.randn(d, generator=g, dtype=torch.float64), torch.randn(5, d, generator=g, dtype=torch.float64),
             torch.tensor([20.0, 10.5, 1.0, -1.0, -1.0], dtype=torch.float64)),
            (torch.randn(d, generator=g, dtype=torch.float64), torch.randn(3, d, generator=g, dtype=torch.float64),
             torch.tensor([20.0, -1.0, -1.0], dtype=torch.float64))]
    sigma, eps, lam, eta = 0.1, 0.01, 1.0, 2.0

    def h(x):
        return [2.0 / (1.0 + math.exp(-sigma * sum(x[a] * W[a, b] for a in range(d)))) - 1.0 for b in range(r)]
    sim = bal = 0.0
    for q, keys, s in trip:
        hq = h(q.tolist())
        colsum = [0.0] * r
        for i in range(keys.shape[0]):
            hk = h(keys[i].tolist())
            sim += float(s[i]) * sum((hq[b] - hk[b]) ** 2 for b in range(r))
            colsum = [colsum[b] + hk[b] for b in range(r)]
        bal += sum(v * v for v in colsum)
    WtW = [[sum(W[a, i] * W[a, j] for a in range(d)) - (1.0 if i == j else 0.0) for j in range(r)] for i in range(r)]
    unc = math.sqrt(sum(v * v for row in WtW for v in row))
    loss, parts = HT.hash_loss([(q.float(), k.float(), s.float()) for q, k, s in trip], W.float(), sigma, eps, lam, eta,
                               normalize=False)
    assert abs(parts["sim"] - sim) < 1e-3 * max(1, abs(sim))
    assert abs(parts["bal"] - bal) < 1e-3 * max(1, abs(bal))
    assert abs(parts["unc"] - unc) < 1e-4 * max(1, unc)
    assert abs(float(loss) - (eps * sim + eta * bal + lam * unc)) < 1e-3 * max(1, abs(float(loss)))


def test_sampling_rule():
    """App. A.1: m in [n/2, n), keys k_1..k_m, top 10 % labelled 20 -> 1 (linear), the rest -1."""
    Q, K = synth.make_training_sequence(200, 8, 2, seed=1)
    trip = HT.sample_triplets(Q[:, 0], K, 5, torch.Generator().manual_seed(3))
    for q, keys, s in trip:
        m = keys.shape[0]
        assert 100 <= m - 1 < 200
        npos = max(1, int(0.1 * m))
        assert int((s > 0).sum()) == npos and bool(torch.all(s[s < 0] == -1))
        top = torch.argsort(keys @ q, descending=True)[:npos]
        assert torch.allclose(s[top], torch.linspace(20.0, 1.0, npos))


def test_short_training_lowers_loss():
    seqs = [synth.make_training_sequence(256, 16, 2, seed=s) for s in range(2)]
    seqs = [(Q.reshape(-1, 16)[::2], K) for Q, K in seqs]
    W, hist = HT.train_hash_weights(seqs, 16, 32, epochs=4, iters=6, queries_per_epoch=4, device="cpu")
    assert hist[-1]["bal"] < hist[0]["bal"]
    assert hist[-1]["loss"] < hist[0]["loss"]
