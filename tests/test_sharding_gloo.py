"""N>1 path on CPU (world_size 2, gloo): the product's sharding (pipette_shard_items, R18)
covers every SA item exactly once, and the two-step combine -- allreduce(min) of the
per-config best latency bits, then allreduce(min) of the item ids attaining it, then
the owners' plans by an allreduce(sum) of owner-only rows -- reproduces the single-rank
search of the oracle bit for bit.  The per-rank SA work is done by the oracle here (no
GPU); on the GPU the same protocol runs in pipette_search over NCCL or over the library's
host transport, which the last test here drives through the binding's gloo callback
(tests/test_gpu_multi.py runs both end to end)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs():
    w = W.WORKLOADS["C1"]
    m = w.model
    cl = O.make_cluster(w.n_nodes, w.gpus_per_node, w.cap_bytes, w.margin_permille)
    mo = O.make_model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
    B, prof = W.workload_inputs(w)
    return w, cl, mo, B, O.make_profile(prof)


def _worker(rank, world, port, chains, iters, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2405_18093_b200 import shard_items
    w, cl, mo, B, P = _inputs()
    R = O.inverse_bandwidth(B)
    feas = [c for c in O.enumerate_configs(cl, mo, w.bs_global, P) if c.feasible]
    F = len(feas)
    items = shard_items(F * chains, rank, world)
    best = np.full(F, np.inf)
    chain = np.full(F, -1, dtype=np.int64)
    perms = {}
    acc = 0
    for j in items.tolist():
        f, c = divmod(j, chains)
        K = O.constants(cl, mo, feas[f], P)
        r = O.sa_chain(K, R, iters, w.seed, c, feas[f].e)
        acc += r.accepted
        if r.best < best[f] or (r.best == best[f] and c < chain[f]):
            best[f], chain[f], perms[f] = r.best, c, r.best_perm
    # step 1: min of the latency bits (non-negative doubles order as integers)
    bits = torch.from_numpy(best.view(np.int64).copy())
    dist.all_reduce(bits, op=dist.ReduceOp.MIN)
    # step 2: min item id among the ranks attaining it
    mine = torch.tensor([f * chains + chain[f] if chain[f] >= 0 and best.view(np.int64)[f] == bits[f].item()
                         else np.iinfo(np.int64).max for f in range(F)], dtype=torch.int64)
    dist.all_reduce(mine, op=dist.ReduceOp.MIN)
    # step 3: owners contribute their plans, every other rank zeros
    Nmax = max(c.pp * c.dp for c in feas)
    rows = torch.zeros((F, Nmax + 1), dtype=torch.int64)
    for f in range(F):
        if int(mine[f]) == f * chains + chain[f]:
            rows[f, :len(perms[f])] = torch.from_numpy(perms[f].astype(np.int64))
            rows[f, Nmax] = 1
    dist.all_reduce(rows, op=dist.ReduceOp.SUM)
    a = torch.tensor([acc], dtype=torch.int64)
    dist.all_reduce(a, op=dist.ReduceOp.SUM)
    gbest = bits.numpy().view(np.float64)
    fw = int(np.argmin(gbest))
    out_q.put((rank, float(gbest[fw]), int(mine[fw]), rows[fw, :feas[fw].pp * feas[fw].dp].numpy().tolist(),
               int(rows[:, Nmax].sum()), int(a.item()), len(items)))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_two_step_combine_matches_single_rank(world):
    import __graft_entry__
    __graft_entry__.build()
    chains, iters = 3, 300
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, chains, iters, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w, cl, mo, B, P = _inputs()
    ref = O.search(cl, B, P, mo, w.bs_global, chains, iters, w.seed)
    F = ref.F
    assert sum(r[6] for r in res) == F * chains                       # every item exactly once
    for (rank, lat, item, perm, owners, acc, _) in res:
        assert lat == ref.latency                                      # bit-identical on every rank
        assert divmod(item, chains)[1] == ref.chain
        assert perm == ref.perm.tolist()
        assert owners == F                                             # exactly one owner per config
        assert acc == ref.sa_accepted


def _ar_worker(rank, world, port, out_q):
    import ctypes as C
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2405_18093_b200 import _abi, torch_host_allreduce
    fn = _abi.HOST_ALLREDUCE(torch_host_allreduce())     # exactly what pipette_init receives
    vals = [[~0 & (2**64 - 1), 5, 2**63 + 7, 2**63 - 1], [3, 2**64 - 2, 2**63 + 1, 2**63]]
    outs = []
    for op in (0, 1):
        buf = (C.c_uint64 * 4)(*vals[rank % 2])
        assert fn(None, buf, 4, op) == 0
        outs.append(list(buf))
    out_q.put((rank, outs))
    dist.destroy_process_group()


def test_torch_host_allreduce_is_uint64_min_and_wrapping_sum():
    # the host transport of the combine (pipette_dist.host_allreduce): uint64 order for min
    # (no-owner items are ~0), sum modulo 2^64, on every rank
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ar_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = [2**64 - 1, 5, 2**63 + 7, 2**63 - 1], [3, 2**64 - 2, 2**63 + 1, 2**63]
    for r in (0, 1):
        assert res[r][0] == [min(x, y) for x, y in zip(a, b)]
        assert res[r][1] == [(x + y) % 2**64 for x, y in zip(a, b)]
