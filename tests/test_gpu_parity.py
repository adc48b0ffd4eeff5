"""GPU vs oracle parity through the C ABI (SURVEY 8(c) acceptance):
  * K1: enumeration order, memory bytes and verdicts bit-exact;
  * K2: eval-stream latencies bit-exact (bar: 1e-12 relative), memory and status exact,
        on random candidates of every feasible config of C1-C5 plus edge cases;
  * K3/K4: per-chain best latency, best step, accepted count and best mapping bit-exact,
        accepted-swap traces bit-exact, the plan bit-exact -- full on C1, sampled on C2
        at BASELINE size in the bench's launch configuration.
"""
import numpy as np
import pytest

import oracle as O
import workloads as W

pytestmark = pytest.mark.gpu
REL = 1e-12


def _ctx(w, B=None, prof=None, **kw):
    from paper_2405_18093_b200 import Pipette
    B0, prof0 = W.workload_inputs(w)
    B = B0 if B is None else B
    prof = prof0 if prof is None else prof
    return Pipette(w.n_nodes, w.gpus_per_node, B, prof, w.cap_bytes, w.margin_permille, **kw), B, prof


def _models(w):
    from paper_2405_18093_b200 import Model
    m = w.model
    return (Model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab),
            O.make_model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab),
            O.make_cluster(w.n_nodes, w.gpus_per_node, w.cap_bytes, w.margin_permille))


def _assert_close(got, want):
    got, want = np.asarray(got, dtype=np.float64), np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape
    rel = np.abs(got - want) / np.maximum(np.abs(want), 1e-300)
    assert float(rel.max(initial=0.0)) <= REL
    return int(np.sum(got.view(np.uint64) != want.view(np.uint64)))


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_enumeration_and_memory_filter_bit_exact(name):
    w = W.WORKLOADS[name]
    pip, B, prof = _ctx(w)
    model, mo, cl = _models(w)
    cfgs, nmb, mem, feas = pip.enumerate(model, w.bs_global)
    ref = O.enumerate_configs(cl, mo, w.bs_global, O.make_profile(prof))
    assert len(ref) == len(cfgs)
    assert [tuple(c) for c in cfgs.tolist()] == [(c.pp, c.tp, c.dp, c.mb) for c in ref]
    assert nmb.tolist() == [c.n_mb for c in ref]
    assert [int(x) for x in mem] == [int(c.mem_bytes) for c in ref]
    assert feas.tolist() == [bool(c.feasible) for c in ref]


def _eval_batch(pip, model, bs, cfg_rows, perms):
    import torch
    cfg = torch.tensor(np.asarray(cfg_rows, dtype=np.int16), device="cuda")
    p = torch.from_numpy(np.ascontiguousarray(perms).astype(np.uint16).view(np.int16)).cuda()
    lat, mem, st = pip.eval(model, bs, cfg, p)
    torch.cuda.synchronize()
    return lat.cpu().numpy(), mem.cpu().numpy().view(np.uint64), st.cpu().numpy()


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_eval_stream_random_candidates(name):
    w = W.WORKLOADS[name]
    pip, B, prof = _ctx(w)
    model, mo, cl = _models(w)
    P = O.make_profile(prof)
    R = O.inverse_bandwidth(B)
    ref = O.enumerate_configs(cl, mo, w.bs_global, P)
    rng = np.random.default_rng(hash(name) & 0xFFFF)
    chosen = [c for c in ref if c.feasible] + [c for c in ref if not c.feasible][:8]
    per = 40 if name != "C5" else 12
    Nmax = max(c.pp * c.dp for c in chosen)
    stride = ((Nmax + 7) // 8) * 8
    rows, perms, want_lat, want_mem, want_st = [], [], [], [], []
    for c in chosen:
        K = O.constants(cl, mo, c, P)
        ps = W.random_perms(K.N, per, int(rng.integers(1 << 30)))
        ps[0] = np.arange(K.N)                       # identity included
        for p in ps:
            row = np.zeros(stride, dtype=np.uint16)
            row[:K.N] = p
            rows.append((c.pp, c.tp, c.dp, c.mb)); perms.append(row)
            want_lat.append(O.latency(K, R, p).T); want_mem.append(int(c.mem_bytes))
            want_st.append(0 if c.feasible else 1)
    lat, mem, st = _eval_batch(pip, model, w.bs_global, rows, np.stack(perms))
    assert st.tolist() == want_st
    assert [int(x) for x in mem] == want_mem
    nbits = _assert_close(lat, want_lat)
    assert nbits == 0, f"{nbits} latencies not bit-identical"


def test_eval_stream_edge_cases():
    w = W.WORKLOADS["C1"]
    model, mo, cl = _models(w)
    B, prof = W.workload_inputs(w)
    prof_missing = [e for e in prof if not (e[0] == 2 and e[1] == 4)]
    pip, _, _ = _ctx(w, B=B, prof=prof_missing)
    P = O.make_profile(prof_missing)
    R = O.inverse_bandwidth(B)
    ref = {(c.pp, c.tp, c.dp, c.mb): c for c in O.enumerate_configs(cl, mo, w.bs_global, P)}
    stride = 17                                        # odd stride: scalar (unaligned) path
    rows, perms, want = [], [], []

    def add(cfg, perm, st, lat=None):
        row = np.zeros(stride, dtype=np.uint16)
        row[:len(perm)] = perm
        rows.append(cfg); perms.append(row); want.append((st, lat))

    c = ref[(4, 2, 2, 1)]
    K = O.constants(cl, mo, c, P)
    good = np.random.default_rng(0).permutation(8)
    add((4, 2, 2, 1), good, 0, O.latency(K, R, good).T)
    add((4, 2, 2, 1), [0, 1, 2, 3, 4, 5, 6, 6], 3)     # duplicate slot
    add((4, 2, 2, 1), [0, 1, 2, 3, 4, 5, 6, 9], 3)     # out of range
    add((3, 2, 2, 1), good, 2)                         # pp*tp*dp != G
    add((4, 2, 2, 3), good, 2)                         # mb does not divide bs_mini
    add((32, 1, 1, 1), np.arange(16), 2)               # pp > n_layers
    add((4, 2, 2, 4), good, 4)                         # profile entry removed
    add((1, 8, 2, 32), [1, 0], 0 if ref[(1, 8, 2, 32)].feasible else 1,
        O.latency(O.constants(cl, mo, ref[(1, 8, 2, 32)], P), R, [1, 0]).T)
    for extra in range(300):                           # ragged tail across blocks
        add((4, 2, 2, 1), good, 0, O.latency(K, R, good).T)
    lat, mem, st = _eval_batch(pip, model, w.bs_global, rows, np.stack(perms))
    for i, (s, l) in enumerate(want):
        assert st[i] == s, (i, rows[i], st[i], s)
        if l is None:
            assert np.isnan(lat[i])
        else:
            assert lat[i] == l
    assert mem[3] == 0 and mem[1] == ref[(4, 2, 2, 1)].mem_bytes


@pytest.mark.parametrize("name,n_cand", [("C1", 4099), ("C2", 6001), ("C3", 5003), ("C4", 2085)])
def test_eval_stream_homogeneous_tiles(name, n_cand):
    """Batches of ONE configuration (the bench's homogeneous stream): whole tiles of one
    config take the contiguous staging path.  Invalid rows (duplicates, ids >= N, 0xffff)
    sit inside those tiles; the batch ends in a ragged tail.  Every latency is compared."""
    w = W.WORKLOADS[name]
    pip, B, prof = _ctx(w)
    model, mo, cl = _models(w)
    P = O.make_profile(prof)
    R = O.inverse_bandwidth(B)
    feas = [c for c in O.enumerate_configs(cl, mo, w.bs_global, P) if c.feasible]
    for c in (max(feas, key=lambda c: (c.pp * c.dp, -c.e)), feas[len(feas) // 2]):
        K = O.constants(cl, mo, c, P)
        stride = ((K.N + 7) // 8) * 8
        rng = np.random.default_rng(K.N * 7 + n_cand)
        ps = W.random_perms(K.N, n_cand, int(rng.integers(1 << 30)))
        rows = np.zeros((n_cand, stride), dtype=np.uint16)
        rows[:, :K.N] = ps
        bad = rng.choice(n_cand, size=min(60, n_cand // 20), replace=False)
        for j, i in enumerate(bad):
            if K.N < 2:
                rows[i, 0] = [1, 0xFFFF, K.N][j % 3]
                continue
            a, b = rng.choice(K.N, size=2, replace=False)
            rows[i, a] = [rows[i, b], K.N, 0xFFFF, min(K.N + 64, 0xFFFF)][j % 4]
        lat, mem, st = _eval_batch(pip, model, w.bs_global, [(c.pp, c.tp, c.dp, c.mb)] * n_cand, rows)
        want_st = np.full(n_cand, 0 if c.feasible else 1)
        want_st[bad] = 3
        assert st.tolist() == want_st.tolist()
        assert np.all(mem == c.mem_bytes)
        ok = want_st != 3
        assert np.all(np.isnan(lat[~ok]))
        want = [O.latency(K, R, rows[i, :K.N]).T for i in np.flatnonzero(ok)]
        assert _assert_close(lat[ok], want) == 0


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_eval_stream_homogeneous_tiles_every_depth(name):
    """Single-configuration tiles of one configuration per pipeline depth present (K2 MODE 1
    takes a compile-time-depth path there, pp = 1..32): a full tile plus a ragged tail,
    duplicates and out-of-range ids inside, every latency compared bit for bit."""
    w = W.WORKLOADS[name]
    pip, B, prof = _ctx(w)
    model, mo, cl = _models(w)
    P = O.make_profile(prof)
    R = O.inverse_bandwidth(B)
    feas = [c for c in O.enumerate_configs(cl, mo, w.bs_global, P) if c.feasible]
    by_pp = {}
    for c in feas:
        by_pp.setdefault(c.pp, c)
    assert len(by_pp) >= 5
    n_cand = 2048 + 301
    for pp, c in sorted(by_pp.items()):
        K = O.constants(cl, mo, c, P)
        stride = ((K.N + 7) // 8) * 8
        rng = np.random.default_rng(K.N * 31 + pp)
        rows = np.zeros((n_cand, stride), dtype=np.uint16)
        rows[:, :K.N] = W.random_perms(K.N, n_cand, int(rng.integers(1 << 30)))
        bad = rng.choice(n_cand, size=40, replace=False)
        for j, i in enumerate(bad):
            a, b = rng.choice(K.N, size=2, replace=False)
            rows[i, a] = [rows[i, b], K.N, 0xFFFF][j % 3]
        lat, mem, st = _eval_batch(pip, model, w.bs_global, [(c.pp, c.tp, c.dp, c.mb)] * n_cand, rows)
        want_st = np.zeros(n_cand, dtype=np.int64)
        want_st[bad] = 3
        assert st.tolist() == want_st.tolist(), pp
        ok = want_st == 0
        want = [O.latency(K, R, rows[i, :K.N]).T for i in np.flatnonzero(ok)]
        assert _assert_close(lat[ok], want) == 0, pp


def test_eval_single_gpu_cluster_and_empty_batch():
    import torch
    from paper_2405_18093_b200 import Model, Pipette
    prof = W.profile_entries(W.GPT_345M, 1, 4)
    pip = Pipette(1, 1, np.array([[2e11]]), prof, 80_000_000_000, 100)
    model = Model(24, 1024, 16, 1024)
    lat, mem, st = _eval_batch(pip, model, 4, [(1, 1, 1, 2)], np.zeros((1, 8), dtype=np.uint16))
    mo = O.make_model(24, 1024, 16, 1024, 50257)
    cl = O.make_cluster(1, 1)
    c = [c for c in O.enumerate_configs(cl, mo, 4, O.make_profile(prof)) if c.mb == 2][0]
    K = O.constants(cl, mo, c, O.make_profile(prof))
    assert lat[0] == O.latency(K, O.inverse_bandwidth(np.array([[2e11]])), [0]).T == c.n_mb * K.S
    e = torch.empty((0, 4), dtype=torch.int16, device="cuda")
    out = pip.eval(model, 4, e, torch.empty((0, 8), dtype=torch.int16, device="cuda"))
    assert out[0].numel() == 0


def _oracle_chain(cl, mo, P, R, cfg_by_e, e, chain, iters, seed, trace=False, **kw):
    K = O.constants(cl, mo, cfg_by_e[e], P)
    return O.sa_chain(K, R, iters, seed, chain, e, trace=trace, **kw)


def test_search_c1_every_chain_bit_exact():
    w = W.WORKLOADS["C1"]
    pip, B, prof = _ctx(w)
    model, mo, cl = _models(w)
    P = O.make_profile(prof)
    R = O.inverse_bandwidth(B)
    chains, iters = 3, 1000
    res = pip.search(model, w.bs_global, chains, iters, w.seed, per_config=True, chain_results=True)
    by_e = {c.e: c for c in O.enumerate_configs(cl, mo, w.bs_global, P)}
    assert len(res["chains"]) == 78 * chains
    for r in res["chains"]:
        o = _oracle_chain(cl, mo, P, R, by_e, r["cfg_index"], r["chain"], iters, w.seed)
        assert r["L0"] == o.L0
        assert (r["best"], r["best_step"], r["accepted"]) == (o.best, o.best_step, o.accepted), r["item"]
        assert (r["best_t_pp"], r["best_t_dp"]) == (o.best_t_pp, o.best_t_dp)
        assert np.array_equal(r["perm"], o.best_perm)
    ref = O.search(cl, B, P, mo, w.bs_global, chains, iters, w.seed)
    plan = res["plan"]
    assert (plan.latency_s, plan.cfg_index, plan.chain, plan.best_step) == \
        (ref.latency, ref.cfg_index, ref.chain, ref.best_step)
    assert np.array_equal(plan.perm, ref.perm)
    assert (plan.t_pp, plan.t_dp, plan.t_bubble, plan.t_straggler) == (ref.t_pp, ref.t_dp, ref.t_bubble, ref.t_straggler)
    assert (plan.sa_steps, plan.sa_accepted) == (ref.sa_steps, ref.sa_accepted)
    assert plan.configs_enumerated == 78 and plan.configs_rejected_oom == 0
    pcs = res["per_config"]
    assert [p.latency_s for p in pcs] == sorted(ref.per_config_best.tolist())


def test_search_traces_bit_exact():
    w = W.WORKLOADS["C2"]
    pip, B, prof = _ctx(w)
    model, mo, cl = _models(w)
    P = O.make_profile(prof)
    R = O.inverse_bandwidth(B)
    chains, iters = 64, 2000
    feas = [c for c in O.enumerate_configs(cl, mo, w.bs_global, P) if c.feasible]
    items = [f * chains + c for f, c in [(0, 0), (5, 17), (17, 63), (30, 1), (44, 40), (len(feas) - 1, 33)]]
    res = pip.search(model, w.bs_global, chains, iters, w.seed, trace_items=items, trace_cap=iters)
    by_e = {c.e: c for c in feas}
    for t, j in enumerate(items):
        f, c = divmod(j, chains)
        o = _oracle_chain(cl, mo, P, R, by_e, feas[f].e, c, iters, w.seed, trace=True)
        got = res["trace"][t]
        assert len(o.trace) == iters
        for a, b in zip(got, o.trace):
            assert a == b, (j, a, b)


def test_search_c2_full_size_sampled_chains():
    # BASELINE size (1024 chains x 10k swaps on all 62 feasible configs), launch config of bench.py
    w = W.WORKLOADS["C2"]
    pip, B, prof = _ctx(w)
    model, mo, cl = _models(w)
    P = O.make_profile(prof)
    R = O.inverse_bandwidth(B)
    res = pip.search(model, w.bs_global, w.chains, w.iterations, w.seed, chain_results=True, per_config=True)
    rows = res["chains"]
    feas = [c for c in O.enumerate_configs(cl, mo, w.bs_global, P) if c.feasible]
    assert len(rows) == len(feas) * w.chains
    by_e = {c.e: c for c in feas}
    rng = np.random.default_rng(1)
    sample = rng.choice(len(rows), size=48, replace=False).tolist()
    winners = {p.cfg_index: p for p in res["per_config"]}
    for j in sample + [r["item"] for r in rows if r["cfg_index"] == res["plan"].cfg_index and r["chain"] == res["plan"].chain]:
        r = rows[j]
        o = _oracle_chain(cl, mo, P, R, by_e, r["cfg_index"], r["chain"], w.iterations, w.seed)
        assert (r["best"], r["best_step"], r["accepted"]) == (o.best, o.best_step, o.accepted), j
        assert np.array_equal(r["perm"], o.best_perm)
    # properties at full size: every best mapping is a permutation whose latency is its best value
    for p in res["per_config"]:
        K = O.constants(cl, mo, by_e[p.cfg_index], P)
        assert O.is_permutation(p.perm)
        assert O.latency(K, R, p.perm).T == p.latency_s
        assert p.latency_s <= O.latency(K, R, np.arange(K.N)).T
    best = min(rows, key=lambda r: (r["best"], r["item"]))
    assert res["plan"].latency_s == best["best"] and res["plan"].chain == best["chain"]
    assert res["plan"].sa_steps == sum(w.chains * w.iterations for c in feas if c.pp * c.dp >= 2)
    assert winners[res["plan"].cfg_index].latency_s == res["plan"].latency_s


def test_search_degenerates_and_errors():
    from paper_2405_18093_b200 import Model, Pipette, PipetteError
    prof = W.profile_entries(W.GPT_345M, 1, 4)
    pip = Pipette(1, 1, np.array([[2e11]]), prof, 80_000_000_000, 100)
    res = pip.search(Model(24, 1024, 16, 1024), 4, 4, 200, 3)
    p = res["plan"]
    assert p.cfg[:3] == (1, 1, 1) and p.perm.tolist() == [0] and p.best_step == -1
    assert p.sa_steps == 0 and p.sa_accepted == 0
    w = W.WORKLOADS["C1"]
    model, _, _ = _models(w)
    tiny, _, _ = _ctx(w)
    B, prof = W.workload_inputs(w)
    oom = Pipette(w.n_nodes, w.gpus_per_node, B, prof, 1 << 20, 100)
    with pytest.raises(PipetteError) as ei:
        oom.search(model, w.bs_global, 1, 10, 1)
    assert ei.value.status == 1
    noprof = Pipette(w.n_nodes, w.gpus_per_node, B, prof[:3], w.cap_bytes, 100)
    with pytest.raises(PipetteError) as ei:
        noprof.search(model, w.bs_global, 1, 10, 1)
    assert ei.value.status == 3
    with pytest.raises(PipetteError) as ei:
        tiny.search(Model(24, 1000, 16, 1024), w.bs_global, 1, 10, 1)     # hidden % heads != 0
    assert ei.value.status == 2


def test_search_is_deterministic_and_bandwidth_update_matters():
    w = W.WORKLOADS["C2"]
    pip, B, prof = _ctx(w)
    model, _, _ = _models(w)
    a = pip.search(model, w.bs_global, 64, 1000, 11)["plan"]
    b = pip.search(model, w.bs_global, 64, 1000, 11)["plan"]
    assert (a.latency_s, a.cfg_index, a.chain) == (b.latency_s, b.cfg_index, b.chain)
    assert np.array_equal(a.perm, b.perm)
    pip.set_bandwidth(B * 0.5)
    c = pip.search(model, w.bs_global, 64, 1000, 11)["plan"]
    assert c.latency_s > a.latency_s


def _sampled_chain_parity(w, chains, iters, n_sample, seed=2, trace_n=3, stats=None, **moves):
    pip, B, prof = _ctx(w)
    model, mo, cl = _models(w)
    P = O.make_profile(prof)
    R = O.inverse_bandwidth(B)
    feas = [c for c in O.enumerate_configs(cl, mo, w.bs_global, P) if c.feasible]
    rng = np.random.default_rng(seed)
    items = rng.choice(len(feas) * chains, size=trace_n, replace=False).tolist()
    res = pip.search(model, w.bs_global, chains, iters, w.seed, chain_results=True, per_config=True,
                     trace_items=items, trace_cap=iters, **moves)
    if stats is not None:
        stats.update(pip.last_search_stats())
    rows = res["chains"]
    assert len(rows) == len(feas) * chains
    by_e = {c.e: c for c in feas}
    for j in rng.choice(len(rows), size=n_sample, replace=False).tolist():
        r = rows[j]
        o = _oracle_chain(cl, mo, P, R, by_e, r["cfg_index"], r["chain"], iters, w.seed, **moves)
        assert r["L0"] == o.L0
        assert (r["best"], r["best_step"], r["accepted"]) == (o.best, o.best_step, o.accepted), (j, r["cfg_index"])
        assert (r["best_t_pp"], r["best_t_dp"]) == (o.best_t_pp, o.best_t_dp)
        assert np.array_equal(r["perm"], o.best_perm)
    for t, j in enumerate(items):
        f, c = divmod(j, chains)
        o = _oracle_chain(cl, mo, P, R, by_e, feas[f].e, c, iters, w.seed, trace=True, **moves)
        assert res["trace"][t] == o.trace, j
    ref_best = min(rows, key=lambda r: (r["best"], r["item"]))
    assert res["plan"].latency_s == ref_best["best"] and res["plan"].chain == ref_best["chain"]
    return res


def test_search_mode0_c3_sixteen_nodes_sampled_chains_and_traces():
    # 16 nodes: MODE 0 with the 256-code m2*R table and four rank words (the n <= 16 kernel
    # instantiation, not C2's n <= 8 one), every pipeline depth of C3 (pp = 1 .. 32)
    res = _sampled_chain_parity(W.WORKLOADS["C3"], chains=64, iters=2000, n_sample=48)
    assert {p.cfg[0] for p in res["per_config"]} >= {1, 2, 4, 8, 16, 32}


def test_full_moves_mode0_c3_sixteen_nodes():
    _sampled_chain_parity(W.WORKLOADS["C3"], chains=32, iters=1000, n_sample=32, trace_n=2,
                          w_migrate=683, w_reverse=682)


def test_search_mode1_c4_sampled_chains_and_traces():
    # 32 nodes: packed positions, sorted-table stage-1 state (S1Large), R through L1
    _sampled_chain_parity(W.WORKLOADS["C4"], chains=64, iters=2000, n_sample=40)


def test_search_mode1_c5_sampled_chains_and_traces():
    # 128 nodes, N up to 256
    _sampled_chain_parity(W.WORKLOADS["C5"], chains=32, iters=1000, n_sample=24, trace_n=2)


def test_search_mode1_byte_counts_16_gpus_per_node():
    # 16 nodes x 16 GPUs: g > 15 takes MODE 1; with tp = 1 a node holds 16 slots, so a
    # stage-1 count can reach 16 and the counts stay bytes (no nibble plane)
    w = W.Workload("C0", 16, 16, W.GPT_345M, 256, 80_000_000_000, 100, 4, 400, 0.2, 0.2, 13)
    res = _sampled_chain_parity(w, chains=4, iters=400, n_sample=40, trace_n=3)
    assert any(p.cfg[1] == 1 and p.cfg[2] >= 16 for p in res["per_config"])


def test_search_mode2_wide_positions():
    # N > 256 (tp = 1 on 40 nodes x 8 GPUs) takes the 32-bit position layout
    w = W.Workload("C0", 40, 8, W.GPT_345M, 320, 80_000_000_000, 100, 8, 600, 0.2, 0.2, 11)
    res = _sampled_chain_parity(w, chains=8, iters=600, n_sample=24, trace_n=2)
    assert any(p.cfg[0] * p.cfg[2] > 256 for p in res["per_config"])


def test_search_zero_iterations_and_odd_chain_counts():
    w = W.WORKLOADS["C1"]
    pip, B, prof = _ctx(w)
    model, mo, cl = _models(w)
    P = O.make_profile(prof)
    # iterations = 0: the plan is the best identity mapping; every chain keeps L0
    res = pip.search(model, w.bs_global, 5, 0, w.seed, chain_results=True)
    assert all(r["best_step"] == -1 and r["accepted"] == 0 and r["best"] == r["L0"] for r in res["chains"])
    ref = O.search(cl, B, P, mo, w.bs_global, 5, 0, w.seed)
    assert res["plan"].latency_s == ref.latency and res["plan"].sa_steps == 0
    # 33 and 65 chains: partial warps at the end of every config
    for chains in (33, 65):
        res = pip.search(model, w.bs_global, chains, 200, w.seed)
        ref = O.search(cl, B, P, mo, w.bs_global, chains, 200, w.seed)
        p = res["plan"]
        assert (p.latency_s, p.cfg_index, p.chain, p.best_step) == (ref.latency, ref.cfg_index, ref.chain, ref.best_step)
        assert np.array_equal(p.perm, ref.perm) and p.sa_accepted == ref.sa_accepted


def test_search_custom_temperature_and_alpha():
    w = W.WORKLOADS["C1"]
    pip, B, prof = _ctx(w)
    model, mo, cl = _models(w)
    P = O.make_profile(prof)
    for kw in ({"alpha": 0.99, "tau": 0.3}, {"alpha": 1.0, "t0": 1e-3}):
        res = pip.search(model, w.bs_global, 4, 500, 77, **kw)
        ref = O.search(cl, B, P, mo, w.bs_global, 4, 500, 77, **kw)
        p = res["plan"]
        assert (p.latency_s, p.cfg_index, p.chain, p.best_step) == (ref.latency, ref.cfg_index, ref.chain, ref.best_step)
        assert p.sa_accepted == ref.sa_accepted


# ------------------------------------------------------------------ full move set (NEXT-1, R21)
UNIFORM = {"w_migrate": 683, "w_reverse": 682}


def test_full_moves_c1_every_chain_and_plan_bit_exact():
    w = W.WORKLOADS["C1"]
    pip, B, prof = _ctx(w)
    model, mo, cl = _models(w)
    P = O.make_profile(prof)
    R = O.inverse_bandwidth(B)
    chains, iters = 3, 800
    res = pip.search(model, w.bs_global, chains, iters, w.seed, chain_results=True, **UNIFORM)
    by_e = {c.e: c for c in O.enumerate_configs(cl, mo, w.bs_global, P)}
    for r in res["chains"]:
        o = _oracle_chain(cl, mo, P, R, by_e, r["cfg_index"], r["chain"], iters, w.seed, **UNIFORM)
        assert (r["L0"], r["best"], r["best_step"], r["accepted"]) == (o.L0, o.best, o.best_step, o.accepted), r["item"]
        assert (r["best_t_pp"], r["best_t_dp"]) == (o.best_t_pp, o.best_t_dp)
        assert np.array_equal(r["perm"], o.best_perm)
    ref = O.search(cl, B, P, mo, w.bs_global, chains, iters, w.seed, **UNIFORM)
    p = res["plan"]
    assert (p.latency_s, p.cfg_index, p.chain, p.best_step) == (ref.latency, ref.cfg_index, ref.chain, ref.best_step)
    assert np.array_equal(p.perm, ref.perm) and p.sa_accepted == ref.sa_accepted


@pytest.mark.parametrize("moves", [UNIFORM, {"w_migrate": 2048, "w_reverse": 0}, {"w_migrate": 0, "w_reverse": 2048}],
                         ids=["uniform", "migrate", "reverse"])
def test_full_moves_c2_sampled_chains_and_traces(moves):
    _sampled_chain_parity(W.WORKLOADS["C2"], chains=32, iters=600, n_sample=32, trace_n=3, **moves)


def test_full_moves_mode1_c4_and_c5():
    _sampled_chain_parity(W.WORKLOADS["C4"], chains=32, iters=400, n_sample=24, trace_n=2, **UNIFORM)
    _sampled_chain_parity(W.WORKLOADS["C5"], chains=8, iters=200, n_sample=12, trace_n=2, **UNIFORM)


def test_full_moves_unsupported_above_256_positions_and_bad_weights():
    from paper_2405_18093_b200 import PipetteError
    w = W.Workload("C0", 40, 8, W.GPT_345M, 320, 80_000_000_000, 100, 8, 600, 0.2, 0.2, 11)
    pip, _, _ = _ctx(w)
    model, _, _ = _models(w)
    with pytest.raises(PipetteError) as ei:
        pip.search(model, w.bs_global, 2, 10, 1, **UNIFORM)
    assert ei.value.status == 6
    w1 = W.WORKLOADS["C1"]
    pip1, _, _ = _ctx(w1)
    with pytest.raises(PipetteError) as ei:
        pip1.search(_models(w1)[0], w1.bs_global, 2, 10, 1, w_migrate=2000, w_reverse=100)
    assert ei.value.status == 2


# ------------------------------------------------------------------ NEXT-2: Eq.1 and the 1F1B DES (R22)
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_eval_models_bit_exact(name):
    import torch
    w = W.WORKLOADS[name]
    pip, B, prof = _ctx(w)
    model, mo, cl = _models(w)
    P = O.make_profile(prof)
    R = O.inverse_bandwidth(B)
    feas = [c for c in O.enumerate_configs(cl, mo, w.bs_global, P) if c.feasible]
    rng = np.random.default_rng(11)
    per = {"C4": 3, "C5": 4}.get(name, 6)     # (C5: pp up to 32, n_mb up to 384)
    Nmax = max(c.pp * c.dp for c in feas)
    stride = ((Nmax + 7) // 8) * 8
    rows, perms, want = [], [], []
    for c in feas:
        K = O.constants(cl, mo, c, P)
        for p in W.random_perms(K.N, per, int(rng.integers(1 << 30))):
            row = np.zeros(stride, dtype=np.uint16)
            row[:K.N] = p
            rows.append((c.pp, c.tp, c.dp, c.mb)); perms.append(row)
            want.append(O.models(K, R, p))
    bad = np.zeros(stride, dtype=np.uint16)                    # duplicate slot -> status 3
    rows.append(rows[0]); perms.append(bad)
    rows.append((3, 1, 1, 1)); perms.append(perms[0])          # not enumerated -> status 2
    cfg = torch.tensor(np.asarray(rows, dtype=np.int16), device="cuda")
    pr = torch.from_numpy(np.stack(perms).view(np.int16)).cuda()
    tp, tprev, tdes, st = (x.cpu().numpy() for x in pip.eval_models(model, w.bs_global, cfg, pr))
    n = len(want)
    want = np.asarray(want)
    assert st[n] == 3 and st[n + 1] == 2 and np.isnan(tp[n]) and np.isnan(tdes[n + 1])
    for col, got in enumerate((tp[:n], tprev[:n], tdes[:n])):
        assert _assert_close(got, want[:, col]) == 0, f"model {col}: not bit-identical"
    # the same T_Pipette as the eval stream
    lat, _, _ = _eval_batch(pip, model, w.bs_global, rows[:n], np.stack(perms[:n]))
    assert np.array_equal(lat, tp[:n])


# ------------------------------------------------------------------ non-power-of-two shapes
# pp in {3, 6, 9, 18, ...} takes the runtime pipeline-depth paths, spn in {6, 3} the
# divide-by-magic node ids (MODE 0: 3 nodes x 6 GPUs; 20 nodes x 6 GPUs: the swap search
# takes MODE 2 -- the MODE 1 swap kernel maps slots to nodes by shifts, so it needs a
# power-of-two gpus_per_node -- and the full move set MODE 1's general node map)
ODD0 = W.Workload("C0", 3, 6, W.GPT_345M, 72, 80_000_000_000, 100, 8, 600, 0.3, 0.3, 21)
ODD1 = W.Workload("C0", 20, 6, W.GPT_345M, 120, 80_000_000_000, 100, 4, 400, 0.3, 0.3, 22)


@pytest.mark.parametrize("w", [ODD0, ODD1], ids=["mode0", "mode1"])
def test_non_power_of_two_shapes_swap_and_full_moves(w):
    res = _sampled_chain_parity(w, chains=w.chains, iters=w.iterations, n_sample=32, trace_n=3)
    assert any(p.cfg[0] not in (1, 2, 4, 8, 16, 32) for p in res["per_config"])
    _sampled_chain_parity(w, chains=w.chains, iters=w.iterations // 2, n_sample=24, trace_n=2, **UNIFORM)


@pytest.mark.parametrize("w", [ODD0, ODD1], ids=["mode0", "mode1"])
def test_non_power_of_two_eval_stream(w):
    pip, B, prof = _ctx(w)
    model, mo, cl = _models(w)
    P = O.make_profile(prof)
    R = O.inverse_bandwidth(B)
    feas = [c for c in O.enumerate_configs(cl, mo, w.bs_global, P) if c.feasible]
    rng = np.random.default_rng(4)
    Nmax = max(c.pp * c.dp for c in feas)
    stride = ((Nmax + 7) // 8) * 8
    rows, perms, want = [], [], []
    for c in feas:
        K = O.constants(cl, mo, c, P)
        for p in W.random_perms(K.N, 8, int(rng.integers(1 << 30))):
            row = np.zeros(stride, dtype=np.uint16)
            row[:K.N] = p
            rows.append((c.pp, c.tp, c.dp, c.mb)); perms.append(row); want.append(O.latency(K, R, p).T)
    lat, mem, st = _eval_batch(pip, model, w.bs_global, rows, np.stack(perms))
    assert np.all((st == 0) | (st == 1))
    assert _assert_close(lat, want) == 0


# ------------------------------------------------------------------ NEXT-4: Eq.7's MLP (R23)
@pytest.mark.parametrize("name", ["C1", "C2", "C4"])
def test_memory_mlp_filter_bit_exact(name):
    from paper_2405_18093_b200 import load_memory_mlp
    params = np.asarray(load_memory_mlp()["params"], dtype=np.float64)
    w = W.WORKLOADS[name]
    pip, B, prof = _ctx(w)
    model, mo, cl = _models(w)
    P = O.make_profile(prof)
    pip.set_memory_model(params)
    cfgs, nmb, mem, feas = pip.enumerate(model, w.bs_global)
    O.set_memory_model(params)
    try:
        ref = O.enumerate_configs(cl, mo, w.bs_global, P)
        assert [int(x) for x in mem] == [int(c.mem_bytes) for c in ref]
        assert feas.tolist() == [bool(c.feasible) for c in ref]
        if name != "C4":
            res = pip.search(model, w.bs_global, 2, 300, w.seed)
            o = O.search(cl, B, P, mo, w.bs_global, 2, 300, w.seed)
            p = res["plan"]
            assert (p.latency_s, p.cfg_index, p.chain, p.mem_bytes) == (o.latency, o.cfg_index, o.chain, o.mem_bytes)
            assert p.configs_rejected_oom == o.E - o.F
    finally:
        O.set_memory_model(None)
    pip.set_memory_model(None)
    _, _, mem2, _ = pip.enumerate(model, w.bs_global)
    assert [int(x) for x in mem2] == [int(O.memory(mo, c.pp, c.tp, c.mb, c.n_mb)) for c in ref]


@pytest.mark.parametrize("name,chains,iters,moves", [
    ("C1", 2, 600, {}),
    ("C2", 16, 1000, {"w_migrate": 683, "w_reverse": 682}),
    ("C4", 32, 1000, {}),
    ("C5", 8, 600, {}),
])
def test_search_self_calibrated_t0(name, chains, iters, moves):
    # t0 < 0: SPEC S:448's self-calibrated initial temperature (R24, k_t0_calibrate) --
    # sampled chains, traces and the plan bit-exact against the oracle's calibration
    _sampled_chain_parity(W.WORKLOADS[name], chains=chains, iters=iters, n_sample=min(24, chains * 8), trace_n=2,
                          t0=-1.0, **moves)


# ---- full-size launch paths: more block chunks than resident blocks, so blocks take a
# second (and later) chunk of another configuration -- table rebuilds (MODE 0), per-warp
# region re-layout (MODE 1) and warp-state reuse are exercised -- in every kernel variant

@pytest.mark.parametrize("name,chains,iters,mode", [("C3", 2048, 2000, 0), ("C4", 2048, 2000, 1), ("C5", 2560, 1000, 1)])
def test_search_more_chunks_than_resident_blocks(name, chains, iters, mode):
    st = {}
    res = _sampled_chain_parity(W.WORKLOADS[name], chains=chains, iters=iters, n_sample=32, trace_n=2, stats=st)
    assert st["mode"] == mode
    assert st["chunks"] > st["grid"], st          # blocks run >= 2 chunks
    assert res["plan"].sa_steps == sum(chains * iters for p in res["per_config"] if len(p.perm) >= 2)


def test_search_mode2_more_chunks_than_resident_blocks():
    # N > 256 (tp = 1 on 40 nodes x 8 GPUs): 32-bit positions, with enough chains that blocks
    # take several chunks
    w = W.Workload("C0", 40, 8, W.GPT_345M, 320, 80_000_000_000, 100, 8, 600, 0.2, 0.2, 11)
    st = {}
    res = _sampled_chain_parity(w, chains=1024, iters=300, n_sample=16, trace_n=2, stats=st)
    assert st["mode"] == 2 and st["chunks"] > st["grid"], st
    assert any(p.cfg[0] * p.cfg[2] > 256 for p in res["per_config"])


def test_search_mode1_c4_ten_thousand_iterations():
    # the cold end of the 10k-step schedule (beta x e^10) in MODE 1
    st = {}
    _sampled_chain_parity(W.WORKLOADS["C4"], chains=64, iters=10000, n_sample=24, trace_n=2, stats=st)
    assert st["mode"] == 1


@pytest.mark.parametrize("name,stride_pad,force", [("C4", 0, "0"), ("C4", 3, "0"), ("C5", 5, "0"), ("C5", 0, "1")])
def test_eval_both_k2_paths_any_stride(name, stride_pad, force, monkeypatch):
    # PIPETTE_EVAL_THREAD forces K2's path: the warp-per-candidate kernel on C4 (k <= 16 member
    # pairs and the sorted-list T_ex), the thread path on C5; an odd stride takes the unaligned
    # row reads (no uint4 prefetch); plus invalid rows (duplicate, id >= N) and unknown configs
    monkeypatch.setenv("PIPETTE_EVAL_THREAD", force)
    w = W.WORKLOADS[name]
    pip, B, prof = _ctx(w)
    model, mo, cl = _models(w)
    P = O.make_profile(prof)
    R = O.inverse_bandwidth(B)
    feas = [c for c in O.enumerate_configs(cl, mo, w.bs_global, P) if c.feasible]
    rng = np.random.default_rng(17)
    stride = max(c.pp * c.dp for c in feas) + stride_pad
    rows, perms, want, st_want = [], [], [], []
    for c in feas:
        K = O.constants(cl, mo, c, P)
        for p in W.random_perms(K.N, 10, int(rng.integers(1 << 30))):
            row = np.zeros(stride, dtype=np.uint16)
            row[:K.N] = p
            rows.append((c.pp, c.tp, c.dp, c.mb)); perms.append(row); want.append(O.latency(K, R, p).T); st_want.append(0)
    c = feas[0]
    bad = np.zeros(stride, dtype=np.uint16); bad[:c.pp * c.dp] = np.arange(c.pp * c.dp); bad[1] = bad[0]
    big = np.zeros(stride, dtype=np.uint16); big[:c.pp * c.dp] = np.arange(c.pp * c.dp); big[2] = c.pp * c.dp
    for r_ in (bad, big):
        rows.append((c.pp, c.tp, c.dp, c.mb)); perms.append(r_); want.append(np.nan); st_want.append(3)
    rows.append((c.pp + 1000, c.tp, c.dp, c.mb)); perms.append(bad); want.append(np.nan); st_want.append(2)
    lat, mem, st = _eval_batch(pip, model, w.bs_global, rows, np.stack(perms))
    assert st.tolist() == st_want
    ok = np.array(st_want) == 0
    assert _assert_close(lat[ok], np.array(want)[ok]) == 0
    assert np.all(np.isnan(lat[~ok]))
