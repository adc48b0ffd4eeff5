"""NEXT-4: train the memory estimator MLP of Eq.7.

The paper trains M_max = MLP(n_gpus, n_layers, n_hiddens, n_heads, tp, pp, dp, bs_micro,
bs_mini, bs_global) -- five layers of 200 -- on memory PROFILED on up to four nodes
(32 GPUs) and validates it up to 128 GPUs.  Its profiles and weights are unpublished, so
the "profiled" memory here is the analytic estimator of reading R11 (oracle/), for every
configuration of a family of GPT shapes on 1..4 nodes x 8 GPUs; the extrapolation is
checked on 8..32 nodes.  This script calls only oracle/ and torch (CPU); it writes the
parameters (float64) to paper_2405_18093_b200/data/mem_mlp.json in the flat layout of
pipette_set_memory_model (include/pipette.h).

    python tools/train_mem_mlp.py [iterations]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

H = 200
SHAPES = [(24, 1024, 16), (24, 2048, 16), (32, 2560, 32), (32, 4096, 32), (40, 5120, 40), (48, 8192, 64),
          (16, 1536, 16), (36, 3072, 24), (44, 6144, 48)]
BATCHES = [64, 128, 256, 512, 1024, 1536]


def samples(nodes, seq=2048):
    X, Y = [], []
    for n in nodes:
        for (L, h, a) in SHAPES:
            for bs in BATCHES:
                cl = O.make_cluster(n, 8)
                mo = O.make_model(L, h, a, seq, 50257)
                for c in O.enumerate_configs(cl, mo, bs):
                    X.append([n * 8, L, h, a, c.tp, c.pp, c.dp, c.mb, bs // c.dp, bs])
                    Y.append(float(c.mem_bytes) / 1e9)
    return np.asarray(X, dtype=np.float64), np.asarray(Y, dtype=np.float64)


def main(iters=20000):
    torch.manual_seed(0)
    Xtr, Ytr = samples([1, 2, 3, 4])
    Xte, Yte = samples([8, 16, 32])
    # log features and target (R23): memory spans four orders of magnitude
    Ltr, Lte, ly = np.log(Xtr), np.log(Xte), np.log(Ytr)
    mean, std = Ltr.mean(0), Ltr.std(0) + 1e-9
    ym, ys = ly.mean(), ly.std()
    xt = torch.tensor((Ltr - mean) / std, dtype=torch.float64)
    yt = torch.tensor((ly - ym) / ys, dtype=torch.float64).unsqueeze(1)
    net = torch.nn.Sequential(torch.nn.Linear(10, H), torch.nn.ReLU(), torch.nn.Linear(H, H), torch.nn.ReLU(),
                              torch.nn.Linear(H, H), torch.nn.ReLU(), torch.nn.Linear(H, H), torch.nn.ReLU(),
                              torch.nn.Linear(H, 1)).double()
    opt = torch.optim.Adam(net.parameters(), lr=1e-3)
    sched = torch.optim.lr_scheduler.CosineAnnealingLR(opt, iters)
    for it in range(iters):
        idx = torch.randint(0, len(xt), (256,))
        loss = torch.mean((net(xt[idx]) - yt[idx]) ** 2)
        opt.zero_grad()
        loss.backward()
        opt.step()
        sched.step()

    def mape(X, Y):
        with torch.no_grad():
            p = np.exp(net(torch.tensor((np.log(X) - mean) / std)).squeeze(1).numpy() * ys + ym)
        return float(np.mean(np.abs(p - Y) / Y))

    lin = [m for m in net if isinstance(m, torch.nn.Linear)]
    params = list(mean) + list(std)
    for m in lin:
        params += m.weight.detach().numpy().ravel().tolist() + m.bias.detach().numpy().ravel().tolist()
    params += [ys, ym]
    out = {"cite": "PAPER.md P:357-371 (Eq.7); trained by tools/train_mem_mlp.py on the analytic memory of reading R11",
           "features": ["n_gpus", "n_layers", "hidden", "heads", "tp", "pp", "dp", "bs_micro", "bs_mini", "bs_global"],
           "layers": [10, H, H, H, H, 1], "iterations": iters,
           "train": {"samples": len(Xtr), "clusters_gpus": [8, 16, 24, 32], "mape": mape(Xtr, Ytr)},
           "extrapolation": {"samples": len(Xte), "clusters_gpus": [64, 128, 256], "mape": mape(Xte, Yte)},
           "params": params}
    path = os.path.join(ROOT, "paper_2405_18093_b200", "data", "mem_mlp.json")
    json.dump(out, open(path, "w"))
    print(json.dumps({k: v for k, v in out.items() if k != "params"}))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 20000)
