"""Why some searches after an L2 flush are slow: per-search task timeline summary."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2405_18093_b200 import Model, Pipette  # noqa: E402

w = W.WORKLOADS["C2"]
B, prof = W.workload_inputs(w)
m = w.model
pip = Pipette(w.n_nodes, w.gpus_per_node, B, prof, w.cap_bytes, w.margin_permille)
model = Model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    pip.search(model, w.bs_global, w.chains, w.iterations, w.seed)
for k in range(12):
    flush.fill_(k)
    torch.cuda.synchronize()
    r = pip.search(model, w.bs_global, w.chains, w.iterations, w.seed)
    tp = pip.last_task_profile().astype(np.int64)
    t0 = tp[:, 0].min()
    st, en = (tp[:, 0] - t0) / 1e6, (tp[:, 1] - t0) / 1e6
    dur = en - st
    sm = tp[:, 2]
    per_sm_end = np.zeros(200)
    np.maximum.at(per_sm_end, sm, en)
    late = np.argsort(-en)[:3]
    print(f"sa {r['plan'].timings_ms['sa']:.2f} span {en.max():.2f} first-wave start max {np.sort(st)[1775]:.3f} "
          f"dur p50 {np.median(dur):.2f} max {dur.max():.2f} | latest tasks: " +
          ", ".join(f"cfg {tp[i,3]} sm {tp[i,2]} start {st[i]:.2f} dur {dur[i]:.2f}" for i in late))
