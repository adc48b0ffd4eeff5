"""Multi-GPU pipette_search over NCCL (one process per GPU, torchrun): every rank gets the
identical plan, bit-identical to the 1-GPU search and to the oracle (R18)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _ngpu():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("world,chains,moves,name,iters", [
    (2, 8, (0, 0), "C1", 1000), (2, 7, (0, 0), "C1", 1000), (4, 8, (0, 0), "C1", 1000), (4, 5, (0, 0), "C1", 1000),
    (8, 8, (0, 0), "C1", 1000), (2, 6, (683, 682), "C1", 1000), (4, 5, (683, 682), "C1", 1000),
    # the headline shape: 128 nodes, MODE 1 (shared R table, S1M witnesses), NCCL combine
    (2, 8, (0, 0), "C5", 150), (4, 9, (0, 0), "C5", 150), (8, 8, (0, 0), "C5", 150)])
def test_multi_gpu_plan_bit_identical(world, chains, moves, name, iters, tmp_path):
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    _run_and_check(world, chains, moves, name, iters, tmp_path, "nccl")


# the same protocol through the library's host transport (pipette_dist.host_allreduce over a
# gloo group): runs on a 1-GPU box too, the W ranks sharing the device
@pytest.mark.parametrize("world,chains,moves,name,iters", [
    (2, 8, (0, 0), "C1", 1000), (3, 7, (683, 682), "C1", 1000), (2, 6, (0, 0), "C3", 300), (3, 8, (0, 0), "C5", 150)])
def test_host_transport_plan_bit_identical(world, chains, moves, name, iters, tmp_path):
    _run_and_check(world, chains, moves, name, iters, tmp_path, "host")


def _run_and_check(world, chains, moves, name, iters, tmp_path, transport):
    out = tmp_path / "plan.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(HERE, "helpers", "mp_search.py"),
           str(out), name, str(chains), str(iters), str(moves[0]), str(moves[1])]
    subprocess.run(cmd, check=True, timeout=600, env={**os.environ, "PIPETTE_TRANSPORT": transport})
    recs = json.load(open(out))
    w = W.WORKLOADS[name]
    B, prof = W.workload_inputs(w)
    m = w.model
    cl = O.make_cluster(w.n_nodes, w.gpus_per_node, w.cap_bytes, w.margin_permille)
    mo = O.make_model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
    ref = O.search(cl, B, O.make_profile(prof), mo, w.bs_global, chains, iters, w.seed,
                   w_migrate=moves[0], w_reverse=moves[1])
    assert len(recs) == world
    for r in recs:
        assert r == {**recs[0], "rank": r["rank"]}                      # identical on every rank
        assert r["transport"] == transport and r["world"] == world
        assert float.fromhex(r["latency"]) == ref.latency
        assert (r["cfg_index"], r["chain"], r["best_step"]) == (ref.cfg_index, ref.chain, ref.best_step)
        assert r["perm"] == ref.perm.tolist()
        assert float.fromhex(r["t_pp"]) == ref.t_pp and float.fromhex(r["t_dp"]) == ref.t_dp
        assert (r["sa_steps"], r["sa_accepted"]) == (ref.sa_steps, ref.sa_accepted)
        assert sorted(float.fromhex(q[1]) for q in r["per_config"]) == sorted(ref.per_config_best.tolist())


def test_profile_bandwidth_feeds_the_search():
    # NEXT-3: Alg.1 l.1 on this box; the measured matrix drives pipette_init / the oracle alike
    import torch

    import oracle as O
    import workloads as W
    from paper_2405_18093_b200 import Model, Pipette, profile_bandwidth
    n = torch.cuda.device_count()
    B, ms = profile_bandwidth(list(range(n)), bytes_per_copy=64 << 20, reps=3)
    assert B.shape == (n, n) and np.all(np.isfinite(B)) and np.all(B > 0)
    assert np.all(np.diag(B) > 5e11)                  # an HBM-to-HBM copy moves > 0.5 TB/s
    if n > 1:
        off = B[~np.eye(n, dtype=bool)]
        assert np.all(off > 1e11)                     # NVLink 5 through NVSwitch: > 100 GB/s per pair
    prof = W.profile_entries(W.GPT_345M, 1, 8 * n)
    pip = Pipette(n, 1, B, prof, 80_000_000_000, 100)
    model = Model(24, 1024, 16, 1024)
    res = pip.search(model, 8 * n, 4, 300, 5)
    cl = O.make_cluster(n, 1)
    mo = O.make_model(24, 1024, 16, 1024, 50257)
    ref = O.search(cl, B, O.make_profile(prof), mo, 8 * n, 4, 300, 5)
    p = res["plan"]
    assert (p.latency_s, p.cfg_index, p.chain) == (ref.latency, ref.cfg_index, ref.chain)


def test_host_transport_rank0_of_two_in_one_process():
    """Product combine path at W = 2 in ONE process: rank 0's context with a host transport
    that stands in for an absent peer (min/sum of one contribution = identity).  The plan is
    then rank 0's shard (items j = f*chains + c with j even, R18), which the oracle computes
    chain by chain; a failing transport surfaces as E_NCCL."""
    from paper_2405_18093_b200 import Model, Pipette, PipetteError
    w = W.WORKLOADS["C1"]
    B, prof = W.workload_inputs(w)
    m = w.model
    calls = []

    def identity(user, buf, count, op):
        calls.append((int(count), int(op)))
        return 0

    pip = Pipette(w.n_nodes, w.gpus_per_node, B, prof, w.cap_bytes, w.margin_permille, rank=0, world=2,
                  host_allreduce=identity)
    chains, iters = 5, 400
    model = Model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
    res = pip.search(model, w.bs_global, chains, iters, w.seed)
    assert [op for _, op in calls] == [0, 0, 1]          # min bits, min items, sum of plan rows
    cl = O.make_cluster(w.n_nodes, w.gpus_per_node, w.cap_bytes, w.margin_permille)
    mo = O.make_model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
    P = O.make_profile(prof)
    R = O.inverse_bandwidth(B)
    feas = [c for c in O.enumerate_configs(cl, mo, w.bs_global, P) if c.feasible]
    best = None
    for j in range(0, len(feas) * chains, 2):
        f, c = divmod(j, chains)
        K = O.constants(cl, mo, feas[f], P)
        r = O.sa_chain(K, R, iters, w.seed, c, feas[f].e)
        if best is None or r.best < best[0]:
            best = (r.best, f, c, r.best_perm)
    p = res["plan"]
    assert p.latency_s == best[0] and p.chain == best[2] and p.perm.tolist() == best[3].tolist()

    def failing(user, buf, count, op):
        return 7

    bad = Pipette(w.n_nodes, w.gpus_per_node, B, prof, w.cap_bytes, w.margin_permille, rank=1, world=2,
                  host_allreduce=failing)
    with pytest.raises(PipetteError) as ei:
        bad.search(model, w.bs_global, chains, iters, w.seed)
    assert ei.value.status == 5 and "host allreduce" in str(ei.value)
