"""pipette_eval on one 2^22 batch (homogeneous largest-N config, or mixed) for profiling."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import workloads as W  # noqa: E402
from paper_2405_18093_b200 import Model, Pipette  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "homogeneous"
name = sys.argv[2] if len(sys.argv) > 2 else "C2"
w = W.WORKLOADS[name]
B, prof = W.workload_inputs(w)
m = w.model
pip = Pipette(w.n_nodes, w.gpus_per_node, B, prof, w.cap_bytes, w.margin_permille)
model = Model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
cfgs, nmb, mem, feas = pip.enumerate(model, w.bs_global)
fi = [i for i in range(len(feas)) if feas[i]]
n = 1 << 22
if mode == "homogeneous":
    idx = max(fi, key=lambda i: (cfgs[i][0] * cfgs[i][2], -i))
    if len(sys.argv) > 3:
        idx = int(sys.argv[3])
    rows = np.full(n, idx)
else:
    rows = np.asarray([fi[k % len(fi)] for k in range(n)])
    np.random.default_rng(3).shuffle(rows)
cf = torch.from_numpy(cfgs[rows].astype(np.int16)).cuda().contiguous()
Ns = torch.from_numpy((cfgs[rows, 0] * cfgs[rows, 2]).astype(np.int64)).cuda()
stride = int(((Ns.max().item() + 7) // 8) * 8)
perm = bench._perms(n, Ns, stride, 5)
t, _ = bench._eval_time(pip, model, w, cf, perm)
print(f"{mode} {name}: {n / t:.3e} candidates/s  ({t * 1e3:.3f} ms)")
