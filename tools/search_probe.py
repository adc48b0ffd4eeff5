"""Time pipette_search on a BASELINE workload (optionally fewer chains/iterations)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2405_18093_b200 import Model, Pipette  # noqa: E402

name = sys.argv[1]
w = W.WORKLOADS[name]
chains = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else w.chains
iters = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "-" else w.iterations
moves = {"w_migrate": 683, "w_reverse": 682} if len(sys.argv) > 4 and sys.argv[4] == "full" else {}
B, prof = W.workload_inputs(w)
m = w.model
pip = Pipette(w.n_nodes, w.gpus_per_node, B, prof, w.cap_bytes, w.margin_permille)
model = Model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
res = pip.search(model, w.bs_global, chains, iters, w.seed, **moves)
torch.cuda.synchronize()
t0 = time.perf_counter()
res = pip.search(model, w.bs_global, chains, iters, w.seed, **moves)
dt = time.perf_counter() - t0
p = res["plan"]
print(f"{name}{' full moves' if moves else ''}: chains {chains} iters {iters} F={p.configs_enumerated - p.configs_rejected_oom} "
      f"steps {p.sa_steps:.3e} wall {dt * 1e3:.1f} ms sa {p.timings_ms['sa']:.1f} ms -> {p.sa_steps / dt:.3e} evals/s; "
      f"plan {p.cfg} T={p.latency_s:.6f}")
