"""Dev diagnostic for NEXT-3: loss terms and recall@k over training (GPU)."""
import sys
import torch
sys.path.insert(0, ".")
import synth
from paper_2506_02572_b200 import hashtrain as HT
from tests.test_gpu_hashtrain import recall_eval

d, G, rbits = 128, 4, 128
train = []
for s in range(4):
    Q, K = synth.make_training_sequence(4096, d, G, seed=100 + s, device="cuda")
    train.append((Q.reshape(-1, d)[::G].contiguous(), K))
held = list(range(500, 504))
W_rand = torch.randn(d, rbits, generator=torch.Generator().manual_seed(9)).cuda()
print("random", recall_eval(W_rand, held))
for name, kw in [("lr0.01", dict(lr=0.01)), ("lr0.003", dict(lr=0.003)), ("lr0.01_eta0.2", dict(lr=0.01, eta=0.2))]:
    W = None
    for stage in range(3):
        W, hist = HT.train_hash_weights(train, d, rbits, epochs=5, iters=20, queries_per_epoch=8, W0=None if W is None else W.cpu(),
                                        device="cuda", seed=stage, **kw)
        print(name, stage, {k: round(v, 4) for k, v in hist[-1].items()}, "recall", recall_eval(W, held),
              "colnorm", float(W.norm(dim=0).mean()))
