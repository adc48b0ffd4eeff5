"""Reduced parity workload for compute-sanitizer (memcheck / racecheck / synccheck), one tool
per run: small searches on every K3 variant (MODE 0 n <= 8 and n <= 16, MODE 1 direct and
list witnesses with and without the pipeline-sum cache, MODE 2, the full move set, the
self-calibrated T0), the eval stream (K2 thread- and warp-per-candidate, edge cases) and
eval_models.  Exits non-zero if a result disagrees with the oracle on the sampled checks.

    compute-sanitizer --tool racecheck python tools/sanitize_suite.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import workloads as W  # noqa: E402
from paper_2405_18093_b200 import Model, Pipette  # noqa: E402


def ctx(w):
    B, prof = W.workload_inputs(w)
    m = w.model
    pip = Pipette(w.n_nodes, w.gpus_per_node, B, prof, w.cap_bytes, w.margin_permille)
    return pip, Model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab), B, prof


def check_plan(w, chains, iters, **kw):
    pip, model, B, prof = ctx(w)
    res = pip.search(model, w.bs_global, chains, iters, w.seed, **kw)
    m = w.model
    cl = O.make_cluster(w.n_nodes, w.gpus_per_node, w.cap_bytes, w.margin_permille)
    mo = O.make_model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
    ref = O.search(cl, B, O.make_profile(prof), mo, w.bs_global, chains, iters, w.seed,
                   t0=kw.get("t0", 0.0), w_migrate=kw.get("w_migrate", 0), w_reverse=kw.get("w_reverse", 0))
    p = res["plan"]
    ok = p.latency_s == ref.latency and np.array_equal(p.perm, ref.perm)
    print(f"{w.name} chains={chains} iters={iters} {kw}: plan {p.cfg} T={p.latency_s:.9f} "
          f"stats {pip.last_search_stats()} {'OK' if ok else 'MISMATCH'}", flush=True)
    return ok


def check_eval(w, n=600):
    pip, model, B, prof = ctx(w)
    cfgs, nmb, mem, feas = pip.enumerate(model, w.bs_global)
    fi = [i for i in range(len(feas)) if feas[i]]
    rng = np.random.default_rng(7)
    rows = rng.choice(fi, size=n)
    Ns = cfgs[rows, 0] * cfgs[rows, 2]
    stride = int(Ns.max())
    perm = np.zeros((n, stride), dtype=np.uint16)
    for i, N in enumerate(Ns):
        perm[i, :N] = rng.permutation(N)
    perm[0, :2] = perm[0, 1], perm[0, 1]                # a duplicate: status 3
    cf = torch.tensor(cfgs[rows].astype(np.int16), device="cuda")
    lat, memo, st = pip.eval(model, w.bs_global, cf, torch.from_numpy(perm.view(np.int16)).cuda())
    tp, tprev, tdes, st2 = pip.eval_models(model, w.bs_global, cf, torch.from_numpy(perm.view(np.int16)).cuda())
    torch.cuda.synchronize()
    m = w.model
    cl = O.make_cluster(w.n_nodes, w.gpus_per_node, w.cap_bytes, w.margin_permille)
    mo = O.make_model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
    P = O.make_profile(prof)
    by = {c.e: c for c in O.enumerate_configs(cl, mo, w.bs_global, P)}
    R = O.inverse_bandwidth(B)
    lat = lat.cpu().numpy()
    ok = int(st[0].item()) == 3
    for i in range(1, n, 37):
        K = O.constants(cl, mo, by[int(rows[i])], P)
        ok = ok and lat[i] == O.latency(K, R, perm[i, :Ns[i]]).T
    print(f"{w.name} eval n={n}: {'OK' if ok else 'MISMATCH'}", flush=True)
    return ok


def main():
    ok = True
    ok &= check_plan(W.WORKLOADS["C1"], 2, 200)
    ok &= check_plan(W.WORKLOADS["C2"], 32, 150)
    ok &= check_plan(W.WORKLOADS["C3"], 32, 100)
    ok &= check_plan(W.WORKLOADS["C4"], 32, 150)
    ok &= check_plan(W.WORKLOADS["C5"], 32, 60)
    ok &= check_plan(W.WORKLOADS["C2"], 32, 100, w_migrate=683, w_reverse=682)
    ok &= check_plan(W.WORKLOADS["C4"], 32, 100, t0=-1.0)
    ok &= check_plan(W.Workload("C0", 40, 8, W.GPT_345M, 320, 80_000_000_000, 100, 8, 600, 0.2, 0.2, 11), 8, 60)
    for name in ("C1", "C2", "C4", "C5"):
        ok &= check_eval(W.WORKLOADS[name])
    print("SANITIZE SUITE", "OK" if ok else "MISMATCH")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
