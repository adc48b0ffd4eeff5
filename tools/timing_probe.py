"""Probe: time pipette_search under different conditions (flush / clock sampling)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import workloads as W  # noqa: E402
from paper_2405_18093_b200 import Model, Pipette  # noqa: E402

w = W.WORKLOADS["C2"]
B, prof = W.workload_inputs(w)
m = w.model
pip = Pipette(w.n_nodes, w.gpus_per_node, B, prof, w.cap_bytes, w.margin_permille)
model = Model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()


def run(tag, n=4, do_flush=False, sampler=False, sleep=0.0, flush_fn=None):
    out = []
    ctx = bench.ClockSampler(0) if sampler else None
    if ctx:
        ctx.__enter__()
    for k in range(n):
        if do_flush:
            flush.fill_(k)
        if flush_fn:
            flush_fn(k)
        if sleep:
            torch.cuda.synchronize(); time.sleep(sleep)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        r = pip.search(model, w.bs_global, w.chains, w.iterations, w.seed)
        b.record(s)
        torch.cuda.synchronize()
        out.append((round(a.elapsed_time(b), 2), round(r["plan"].timings_ms["sa"], 2)))
    if ctx:
        ctx.__exit__()
        print(tag, out, ctx.summary())
    else:
        print(tag, out)




def tiny(k):
    flush.fill_(k)
    pip.search(model, w.bs_global, 1, 10, w.seed)

run("plain")
run("flush256", do_flush=True)
for mb in (48, 96, 128, 192):
    buf = torch.empty(mb << 20, dtype=torch.uint8, device="cuda")
    run(f"fill{mb}MB", flush_fn=lambda k, b=buf: b.fill_(k))
    del buf
run("flush256+tinysearch", flush_fn=tiny)
run("plain again")
