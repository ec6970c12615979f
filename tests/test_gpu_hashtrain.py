"""NEXT-3 recall harness: hash weights trained with Eq. 9 on
synthetic anisotropic activations vs random projections, recall@k of the
PRODUCT decode kernel's selection against exact top-k attention scores on
held-out sequences."""
import pytest
import torch

import paper_2506_02572_b200 as H
import synth
from paper_2506_02572_b200 import hashtrain as HT

pytestmark = pytest.mark.gpu


def recall_eval(W, seeds, n=8192, G=4, k=256, d=128):
    """Mean recall@k of hata_decode_topk_attn's selection (W [d, rbits])."""
    rbits = W.shape[1]
    rec = []
    for s in seeds:
        Q, K = synth.make_training_sequence(n, d, G, seed=s, device="cuda")
        Kc = K.to(torch.bfloat16)[None, None].contiguous()              # [1, 1, n, d]
        V = torch.randn_like(Kc)
        Wb = W.to(torch.bfloat16)[None].contiguous()
        codes = torch.zeros(1, 1, n, rbits // 32, dtype=torch.int32, device="cuda")
        H.hash_keys(Kc, Wb, codes)
        q = Q[n - 1].to(torch.bfloat16)[None]                           # [1, G, d]: the last position's heads
        nn_ = torch.tensor([n], dtype=torch.int64, device="cuda")
        idx = torch.full((1, 1, k), -1, dtype=torch.int32, device="cuda")
        H.decode_topk_attn(q, Kc, V, codes, Wb, nn_, k, out_idx=idx)
        ref = HT.exact_topk(q[0].float(), Kc[0, 0].float(), n, k)
        rec.append(HT.recall_at_k(idx[0, 0].cpu(), ref.cpu()))
    return sum(rec) / len(rec)


def test_trained_hash_beats_random_projection():
    d, G, rbits = 128, 4, 128
    train = []
    for s in range(4):
        Q, K = synth.make_training_sequence(4096, d, G, seed=100 + s, device="cuda")
        train.append((Q.reshape(-1, d)[::G].contiguous(), K))            # one query head per position (rotating below)
    W, hist = HT.train_hash_weights(train, d, rbits, epochs=15, iters=20, queries_per_epoch=8, device="cuda")
    held = list(range(500, 508))
    r_trained = recall_eval(W, held)
    W_rand = torch.randn(d, rbits, generator=torch.Generator().manual_seed(9)).cuda()
    r_random = recall_eval(W_rand, held)
    print("recall@256 trained", r_trained, "random", r_random, "loss", hist[0]["loss"], "->", hist[-1]["loss"])
    assert hist[-1]["loss"] < hist[0]["loss"]
    assert r_trained > r_random
