"""torchrun worker: pipette_search over NCCL on W GPUs; rank 0 writes the plan as JSON.
Usage: torchrun --nproc-per-node W tests/helpers/mp_search.py OUT.json WORKLOAD CHAINS ITERS [W_MIGRATE W_REVERSE]
With PIPETTE_TRANSPORT=host the process group is gloo and the combine runs through the
library's host transport (pipette_dist.host_allreduce); ranks share GPU (rank mod #GPUs)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import workloads as W  # noqa: E402
from paper_2405_18093_b200 import Model, Pipette  # noqa: E402


def main(out, name, chains, iters, w_migrate=0, w_reverse=0):
    transport = os.environ.get("PIPETTE_TRANSPORT", "nccl")
    local = int(os.environ["LOCAL_RANK"]) % (torch.cuda.device_count() if transport == "host" else 1 << 30)
    torch.cuda.set_device(local)
    if transport == "host":
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = W.WORKLOADS[name]
    B, prof = W.workload_inputs(w)
    m = w.model
    pip = Pipette.from_torch_distributed(w.n_nodes, w.gpus_per_node, B, prof, device=local, transport=transport,
                                         mem_capacity_bytes=w.cap_bytes, mem_margin_permille=w.margin_permille)
    res = pip.search(Model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab), w.bs_global, chains, iters, w.seed,
                     per_config=True, w_migrate=w_migrate, w_reverse=w_reverse)
    p = res["plan"]
    rec = {"rank": dist.get_rank(), "world": dist.get_world_size(), "latency": p.latency_s.hex(),
           "cfg_index": p.cfg_index, "chain": p.chain, "best_step": p.best_step, "perm": p.perm.tolist(), "transport": transport,
           "t_pp": p.t_pp.hex(), "t_dp": p.t_dp.hex(), "sa_steps": p.sa_steps, "sa_accepted": p.sa_accepted,
           "per_config": [(q.cfg_index, q.latency_s.hex(), q.chain, q.perm.tolist()) for q in res["per_config"]]}
    recs = [None] * dist.get_world_size()
    dist.all_gather_object(recs, rec)
    if dist.get_rank() == 0:
        json.dump(recs, open(out, "w"))
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), *[int(x) for x in sys.argv[5:7]])
