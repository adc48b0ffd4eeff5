"""torchrun worker: per-rank timing breakdown of repeated pipette_search calls (host wall,
device step, phases).  torchrun --nproc-per-node W tools/mp_timing.py [C2] [reps]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import workloads as W  # noqa: E402
from paper_2405_18093_b200 import Model, Pipette  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
local = int(os.environ.get("LOCAL_RANK", "0"))
world = int(os.environ.get("WORLD_SIZE", "1"))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
w = W.WORKLOADS[name]
B, prof = W.workload_inputs(w)
m = w.model
kw = dict(mem_capacity_bytes=w.cap_bytes, mem_margin_permille=w.margin_permille)
pip = (Pipette.from_torch_distributed(w.n_nodes, w.gpus_per_node, B, prof, device=local, **kw) if world > 1
       else Pipette(w.n_nodes, w.gpus_per_node, B, prof, device=local, **kw))
model = Model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
chains = w.chains * world
for _ in range(2):
    pip.search(model, w.bs_global, chains, w.iterations, w.seed)
rows = []
s = torch.cuda.current_stream()
for _ in range(reps):
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record(s)
    r = pip.search(model, w.bs_global, chains, w.iterations, w.seed)
    b.record(s)
    torch.cuda.synchronize()
    rows.append({"wall_ms": (time.perf_counter() - t0) * 1e3, "dev_ms": a.elapsed_time(b), **r["plan"].timings_ms})
out = [None] * world
if world > 1:
    dist.all_gather_object(out, {"rank": local, "rows": rows})
else:
    out = [{"rank": 0, "rows": rows}]
if local == 0:
    for o in out:
        med = {k: sorted(x[k] for x in o["rows"])[len(o["rows"]) // 2] for k in o["rows"][0]}
        print(json.dumps({"rank": o["rank"], **{k: round(v, 3) for k, v in med.items()}}))
if world > 1:
    dist.destroy_process_group()
