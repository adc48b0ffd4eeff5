"""NEXT-2 sweep (a Fig.5a analog): T_Pipette (Eq.3) and T_prev (Eq.1) against the
1F1B discrete-event simulation on random plans of every feasible configuration, all on
the GPU (pipette_eval_models).  Prints one JSON line: MAPE of both closed forms vs the
DES (overall and by pipeline depth) and the kernel's candidates/s.

    python tools/models_sweep.py [C2] [n_per_config]
"""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2405_18093_b200 import Model, Pipette  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
per = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
w = W.WORKLOADS[name]
B, prof = W.workload_inputs(w)
m = w.model
pip = Pipette(w.n_nodes, w.gpus_per_node, B, prof, w.cap_bytes, w.margin_permille)
model = Model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
cfgs, nmb, mem, feas = pip.enumerate(model, w.bs_global)
fi = [i for i in range(len(feas)) if feas[i]]
rows = np.repeat(np.asarray(fi), per)
cf = torch.from_numpy(cfgs[rows].astype(np.int16)).cuda().contiguous()
Ns = (cfgs[rows, 0] * cfgs[rows, 2]).astype(np.int64)
stride = int(((Ns.max() + 7) // 8) * 8)
g = torch.Generator(device="cuda").manual_seed(1)
keys = torch.rand((len(rows), stride), device="cuda", generator=g)
col = torch.arange(stride, device="cuda").unsqueeze(0)
Nt = torch.from_numpy(Ns).cuda().unsqueeze(1)
keys = torch.where(col < Nt, keys, 2.0 + col.to(keys.dtype))
perm = torch.argsort(keys, dim=1).to(torch.int16).contiguous()
for _ in range(2):
    out = pip.eval_models(model, w.bs_global, cf, perm)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
out = pip.eval_models(model, w.bs_global, cf, perm)
b.record()
torch.cuda.synchronize()
t = a.elapsed_time(b) / 1e3
tp, tprev, tdes, st = (x.cpu().numpy() for x in out)
ok = (st == 0) | (st == 1)
ep = np.abs(tp - tdes) / tdes
eprev = np.abs(tprev - tdes) / tdes
by = collections.defaultdict(lambda: [[], []])
for i in np.nonzero(ok)[0]:
    by[int(cfgs[rows[i], 0])][0].append(ep[i])
    by[int(cfgs[rows[i], 0])][1].append(eprev[i])
res = {"workload": name, "candidates": int(len(rows)), "configs": len(fi),
       "mape_pipette_vs_des": float(np.mean(ep[ok])), "mape_prev_vs_des": float(np.mean(eprev[ok])),
       "by_pp": {str(k): {"n": len(v[0]), "mape_pipette": float(np.mean(v[0])), "mape_prev": float(np.mean(v[1]))}
                 for k, v in sorted(by.items())},
       "k_models_candidates_per_s": len(rows) / t, "k_models_ms": t * 1e3,
       "note": "DES: 1F1B with f = C'/3, b = 2C'/3, directed one-way hops (R22); MAPE = mean |model - DES| / DES"}
print(json.dumps(res))
