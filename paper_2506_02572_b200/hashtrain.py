"""Learning-to-hash for HATA: train the hash weights W_H
of one KV head on synthetic query/key data, and measure the recall of the
product decode kernel's top-k selection against exact top-k attention scores.

PAPER: §3.1 -- the relaxed objective Eq. 9

    min  eps * sum_j sum_i s_ji ||h(q_j) - h(k_ji)||^2
       + eta * sum_j ||sum_i h(k_ji)||^2            (bit balance, Eq. 5 relaxed)
       + lam * ||W_H^T W_H - I_r||                   (uncorrelation, Eq. 6 relaxed)
    h(x) = 2 Sigmoid(sigma x W_H) - 1

with the data sampling of App. A.1 (one query q_m, m in [n/2, n),
its causal keys k_1..k_m, the top 10 % of q_m k_i scores labelled linearly
from 20 down to 1, the rest -1) and the settings of App. A.2 (P:721-747:
sigma 0.1, eps 0.01, lam 1.0, eta 2.0, SGD lr 0.1, momentum 0.9, weight decay
1e-6, 15 epochs x 20 iterations), with the loss terms normalised per pair /
per query and SGD lr 0.01 (reading R21).  One W_H per KV head (R4); a GQA group's
query heads all contribute queries.  Training runs once per layer, offline
(P:170); it is PyTorch autograd on the GPU -- the decode hot path never
touches it.  Training on real LLM activations stays out of scope (needs model
weights and LongBench); the data here come from synth.make_training_sequence.
"""
from __future__ import annotations

import torch


def sample_triplets(Q: torch.Tensor, K: torch.Tensor, n_queries: int, gen: torch.Generator):
    """App. A.1 on one sequence: Q [n, d] (the queries of the
    group's heads, concatenated per position), K [n, d].  Returns the list of
    (q_m [d], keys [m, d], labels [m]) for n_queries sampled positions m in
    [n/2, n); labels: top 10 % of q_m . k_i linearly 20 -> 1, others -1."""
    n = K.shape[0]
    out = []
    for _ in range(n_queries):
        m = int(torch.randint(n // 2, n, (1,), generator=gen, device="cpu"))
        q = Q[m]
        keys = K[:m + 1]                                  # causal: k_1 .. k_m (inclusive of the current token)
        score = keys.float() @ q.float()
        order = torch.argsort(score, descending=True)
        npos = max(1, int(0.1 * keys.shape[0]))
        labels = torch.full((keys.shape[0],), -1.0, device=K.device)
        labels[order[:npos]] = torch.linspace(20.0, 1.0, npos, device=K.device)
        out.append((q, keys, labels))
    return out


def relaxed_hash(x: torch.Tensor, W: torch.Tensor, sigma: float) -> torch.Tensor:
    """h(x) = 2 Sigmoid(sigma x W_H) - 1."""
    return 2.0 * torch.sigmoid(sigma * (x.float() @ W)) - 1.0


def hash_loss(triplets, W: torch.Tensor, sigma=0.1, eps=0.01, lam=1.0, eta=2.0, normalize=False):
    """Eq. 9 over the sampled queries j.

    normalize=False: the sums exactly as printed.  normalize=True (reading
    R21; the paper does not state how its batches are scaled):
    the similarity term averaged over the pairs and each query's balance term
    divided by its key count m_j, then averaged over the queries -- so that
    balanced bits contribute O(r) and no term grows with the sequence length
    (the printed sums put ||sum_i h(k_i)||^2 = O(m^2 r) against O(m r)).
    """
    r = W.shape[1]
    sim = 0.0
    bal = 0.0
    npairs = 0
    for q, keys, s in triplets:
        hq = relaxed_hash(q[None], W, sigma)             # [1, r]
        hk = relaxed_hash(keys, W, sigma)                # [m, r]
        sim = sim + (s * ((hq - hk) ** 2).sum(-1)).sum()
        b = (hk.sum(0) ** 2).sum()
        bal = bal + (b / keys.shape[0] if normalize else b)
        npairs += keys.shape[0]
    if normalize:
        sim = sim / npairs
        bal = bal / len(triplets)
    unc = torch.linalg.matrix_norm(W.t() @ W - torch.eye(r, device=W.device, dtype=W.dtype))
    val = lambda t: float(torch.as_tensor(t).detach())  # noqa: E731
    return eps * sim + eta * bal + lam * unc, dict(sim=val(sim), bal=val(bal), unc=val(unc))


def train_hash_weights(sequences, d: int, rbits: int, epochs=15, iters=20, queries_per_epoch=8, sigma=0.1,
                       eps=0.01, lam=1.0, eta=2.0, lr=0.01, momentum=0.9, weight_decay=1e-6, seed=0, W0=None,
                       device="cuda", normalize=True):
    """Train one KV head's W_H [d, rbits] (App. A.2; lr 0.01 instead of the
    table's 0.1 -- reading R21: with the synthetic activations' norms the
    table's rate oscillates between the balance and uncorrelation terms and
    the columns of W_H blow up, measured in tools/hashtrain_diag.py).  sequences: list of
    (Q [n, d], K [n, d]) tensors; each epoch samples fresh triplets (the
    paper loads a few 32K chunks per epoch) and runs `iters` SGD iterations on
    them.  Returns (W, history of loss terms)."""
    gen = torch.Generator().manual_seed(seed)
    if W0 is None:
        W0 = torch.randn(d, rbits, generator=gen) / d ** 0.5
    W = W0.clone().to(device).float().requires_grad_(True)
    opt = torch.optim.SGD([W], lr=lr, momentum=momentum, weight_decay=weight_decay)
    hist = []
    for ep in range(epochs):
        trip = []
        for Qs, Ks in sequences:
            trip += sample_triplets(Qs.to(device), Ks.to(device), queries_per_epoch, gen)
        for it in range(iters):
            opt.zero_grad()
            loss, parts = hash_loss(trip, W, sigma, eps, lam, eta, normalize)
            loss.backward()
            opt.step()
        hist.append(dict(epoch=ep, loss=float(loss), **parts))
    return W.detach(), hist


def exact_topk(q_group: torch.Tensor, K: torch.Tensor, n: int, k: int) -> torch.Tensor:
    """Ground truth for the recall metric: the k tokens of largest summed
    attention logit over the group's query heads, sum_h q_h . k_t (the exact
    top-k attention of Eq. 2, aggregated like P:255).  Ascending."""
    s = (K[:n].float() @ q_group.float().t()).sum(-1)
    return torch.sort(torch.topk(s, min(k, n)).indices).values


def recall_at_k(sel: torch.Tensor, ref: torch.Tensor) -> float:
    """|selected ∩ exact| / |exact| for index sets."""
    a = set(sel[sel >= 0].tolist())
    b = set(ref.tolist())
    return len(a & b) / max(1, len(b))
