"""NEXT-3: profile this box's GPU-to-GPU bandwidth matrix (pipette_profile_bandwidth) and
plan a GPT-345M run on it (one GPU per "node", tp = 1).  Prints one JSON line.
    python tools/netprof.py [bytes_MiB]"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2405_18093_b200 import Model, Pipette, profile_bandwidth  # noqa: E402

mib = int(sys.argv[1]) if len(sys.argv) > 1 else 256
n = torch.cuda.device_count()
B, ms = profile_bandwidth(list(range(n)), bytes_per_copy=mib << 20, reps=5)
prof = W.profile_entries(W.GPT_345M, 1, 8 * n)
pip = Pipette(n, 1, B, prof, 80_000_000_000, 100)
res = pip.search(Model(24, 1024, 16, 1024), 8 * n, 256, 2000, 1)
p = res["plan"]
off = B[~np.eye(n, dtype=bool)] if n > 1 else np.array([np.nan])
print(json.dumps({"gpus": n, "bytes": mib << 20, "bw_GBps": (B / 1e9).round(1).tolist(),
                  "intra_GBps_median": float(np.median(np.diag(B)) / 1e9),
                  "peer_GBps_min": float(off.min() / 1e9), "peer_GBps_median": float(np.median(off) / 1e9),
                  "plan": {"cfg": list(p.cfg), "latency_s": p.latency_s, "perm": p.perm.tolist()}}))
