"""Per-config SA task durations of one pipette_search (load-balance diagnostics)."""
import collections
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402
from paper_2405_18093_b200 import Model, Pipette  # noqa: E402


def main(name="C2", chains=None, iters=None):
    chains = int(chains) if chains else None
    iters = int(iters) if iters else None
    w = W.WORKLOADS[name]
    B, prof = W.workload_inputs(w)
    m = w.model
    pip = Pipette(w.n_nodes, w.gpus_per_node, B, prof, w.cap_bytes, w.margin_permille)
    model = Model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
    chains = chains or w.chains
    iters = iters or w.iterations
    for _ in range(2):
        res = pip.search(model, w.bs_global, chains, iters, w.seed)
    tp = pip.last_task_profile().astype(np.int64)
    cfgs, nmb, mem, feas = pip.enumerate(model, w.bs_global)
    t0 = tp[:, 0].min()
    dur = (tp[:, 1] - tp[:, 0]) / 1e6
    by = collections.defaultdict(list)
    for (s, e, sm, c), d in zip(tp, dur):
        by[int(c)].append((d, (s - t0) / 1e6, (e - t0) / 1e6))
    print(f"kernel span {(tp[:, 1].max() - t0) / 1e6:.2f} ms, tasks {len(tp)}, sa_ms {res['plan'].timings_ms['sa']:.2f}")
    print(f"{'e':>4} {'pp':>3} {'tp':>3} {'dp':>3} {'mb':>3} {'N':>4} {'tasks':>5} {'mean ms':>8} {'max ms':>8} {'first start':>11} {'last end':>9}")
    for c, v in sorted(by.items(), key=lambda x: -np.mean([a[0] for a in x[1]])):
        pp, tpp, dp, mb = cfgs[c]
        print(f"{c:4d} {pp:3d} {tpp:3d} {dp:3d} {mb:3d} {pp*dp:4d} {len(v):5d} {np.mean([a[0] for a in v]):8.3f} "
              f"{max(a[0] for a in v):8.3f} {min(a[1] for a in v):11.3f} {max(a[2] for a in v):9.3f}")
    # concurrency timeline
    ts = np.linspace(0, (tp[:, 1].max() - t0), 20)
    act = [int(np.sum((tp[:, 0] - t0 <= t) & (tp[:, 1] - t0 > t))) for t in ts]
    print("active warps over time:", act)
    # chunk barrier waste: the warps of one block chunk start together on one SM; the early
    # finishers idle until the chunk's last warp ends (the block's next fetch is collective)
    groups = collections.defaultdict(list)
    for s, e, sm, c in tp:
        groups[(int(sm), int(s) // 20000)].append(int(e))   # same SM, starts within 20 us
    idle = sum(max(es) - e for es in groups.values() for e in es)
    busy = float(np.sum(tp[:, 1] - tp[:, 0]))
    print(f"chunk barrier idle: {idle / 1e6:.1f} warp-ms = {100 * idle / busy:.1f}% of busy warp time "
          f"({len(groups)} chunks)")


if __name__ == "__main__":
    main(*(sys.argv[1:4] or ["C2"]))
