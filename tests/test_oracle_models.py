"""Pins of NEXT-2: the 1F1B discrete-event simulation (P:107-111,
P:132-138, hidden critical paths P:269-271) and the prior-work closed form Eq.1
 beside Eq.3-6, reading R22 of DESIGN.md."""
import json
import os

import numpy as np
import pytest

import oracle as O
import workloads as W
from des import simulate

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def close(a, b, rel=1e-12):
    return abs(a - b) <= rel * max(abs(a), abs(b), 1e-300)


def test_des_matches_the_independent_python_simulator():
    # tests/des.py (dict-based, op lists) vs the oracle's array-based event loop
    rng = np.random.default_rng(0)
    for _ in range(400):
        pp, n_mb = int(rng.integers(1, 10)), int(rng.integers(1, 30))
        f, b = float(rng.random()), float(2 * rng.random())
        h = rng.random(max(pp - 1, 0)).tolist()
        want, _ = simulate(pp, n_mb, f, b, h)
        assert O.des_1f1b(pp, n_mb, f, b, h) == want, (pp, n_mb)


def test_des_golden_table():
    for row in json.load(open(os.path.join(GOLD, "des_1f1b_uniform_hops.json")))["rows"]:
        pp = row["pp"]
        assert O.des_1f1b(pp, row["n_mb"], 1.0, 1.0, [1.0] * (pp - 1)) == row["des"]


@pytest.mark.parametrize("pp", [1, 2, 3, 5, 8])
def test_des_without_hops_is_the_textbook_1f1b_time(pp):
    # (n_mb + pp - 1)(f + b): Narayanan et al. SC'21 1F1B without communication
    for n_mb in (1, 2, pp, 3 * pp + 1):
        assert O.des_1f1b(pp, n_mb, 0.25, 0.5, [0.0] * (pp - 1)) == (n_mb + pp - 1) * 0.75


def test_des_uses_each_direction_and_is_monotone():
    pp, n_mb = 4, 8
    base = O.des_1f1b(pp, n_mb, 1.0, 2.0, [0.1] * 3, [0.1] * 3)
    slow_f = O.des_1f1b(pp, n_mb, 1.0, 2.0, [0.1, 2.0, 0.1], [0.1] * 3)
    slow_b = O.des_1f1b(pp, n_mb, 1.0, 2.0, [0.1] * 3, [0.1, 2.0, 0.1])
    assert slow_f > base and slow_b > base
    rng = np.random.default_rng(3)
    # the backward hops are their own (directed B, R5): they change the makespan
    assert any(O.des_1f1b(pp, n_mb, 1.0, 2.0, hf, hb) != O.des_1f1b(pp, n_mb, 1.0, 2.0, hf, hf)
               for hf, hb in (rng.random((2, 3)) for _ in range(20)))
    for _ in range(100):
        hf, hb = rng.random(3), rng.random(3)
        t = O.des_1f1b(pp, n_mb, 1.0, 2.0, hf, hb)
        i = int(rng.integers(3))
        hf2 = hf.copy(); hf2[i] += 0.5
        assert O.des_1f1b(pp, n_mb, 1.0, 2.0, hf2, hb) >= t


def _plan(name, rng):
    w = W.WORKLOADS[name]
    B, prof = W.workload_inputs(w)
    m = w.model
    cl = O.make_cluster(w.n_nodes, w.gpus_per_node, w.cap_bytes, w.margin_permille)
    mo = O.make_model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
    P = O.make_profile(prof)
    feas = [c for c in O.enumerate_configs(cl, mo, w.bs_global, P) if c.feasible]
    return cl, mo, P, O.inverse_bandwidth(B), feas


def test_models_relations_on_real_plans():
    rng = np.random.default_rng(5)
    cl, mo, P, R, feas = _plan("C2", rng)
    for c in feas[::3]:
        K = O.constants(cl, mo, c, P)
        perm = rng.permutation(K.N)
        tp, tprev, tdes = O.models(K, R, perm)
        bd = O.latency(K, R, perm)
        assert tp == bd.T
        # Eq.3 - Eq.1 = the (n_mb/pp - 1) hidden critical paths of T_PP
        assert close(tp - tprev, bd.t_pp * (c.n_mb / c.pp - 1.0), 1e-9) or abs(tp - tprev - bd.t_pp * (c.n_mb / c.pp - 1.0)) < 1e-12 * tp
        if c.pp == 1:
            assert tdes == tp == tprev or close(tdes, tp)


def test_zero_hops_all_three_models_agree():
    # homogeneous, hop-free cluster: one pipeline per config, T_DP = 0 (dp = 1)
    K = O.raw_consts(4, 1, 1, 4, 12, 0.75, 0.0, 0.0)
    R = O.inverse_bandwidth(W.uniform_bandwidth(4, 1e10, 1e11))
    tp, tprev, tdes = O.models(K, R, [0, 1, 2, 3])
    assert close(tp, (12 + 4 - 1) * 0.75) and close(tprev, tp) and close(tdes, tp)


def test_pipette_closer_to_des_than_eq1_when_microbatches_outnumber_stages():
    # the paper's claim (Fig.5a): Eq.1 misses the hidden critical paths
    rng = np.random.default_rng(9)
    cl, mo, P, R, feas = _plan("C2", rng)
    ep, eprev = [], []
    for c in feas:
        if c.pp < 2 or c.n_mb < 2 * c.pp:
            continue
        K = O.constants(cl, mo, c, P)
        for _ in range(3):
            tp, tprev, tdes = O.models(K, R, rng.permutation(K.N))
            ep.append(abs(tp - tdes) / tdes)
            eprev.append(abs(tprev - tdes) / tdes)
    assert len(ep) > 20 and np.mean(ep) < np.mean(eprev)


def _op_positions(pp, n_mb):
    """Megatron 1F1B op order per stage s: w = min(pp-s-1, n_mb) warm-up
    forwards, then F/B pairs, then the cool-down backwards; positions of F(m) and B(m)."""
    pos = []
    for s in range(pp):
        w = min(pp - s - 1, n_mb)
        ops = [("F", m) for m in range(w)]
        for j in range(n_mb - w):
            ops += [("F", w + j), ("B", j)]
        ops += [("B", m) for m in range(n_mb - w, n_mb)]
        assert len(ops) == 2 * n_mb
        pos.append({op: k for k, op in enumerate(ops)})
    return pos


def _closed_positions(pp, n_mb):
    s = np.arange(pp)[:, None]
    m = np.arange(n_mb)[None, :]
    w = np.minimum(pp - s - 1, n_mb)
    f = np.where(m < w, m, 2 * m - w)
    b = np.where(m < n_mb - w, w + 2 * m + 1, n_mb + m)
    return f, b


def test_des_dependency_sits_at_index_k_or_k_minus_1():
    # k_models.cu computes the 1F1B ops by increasing op index k with two rows of end times:
    # valid iff F(s-1, m) sits at index k or k-1 of stage s-1 when F(s, m) is op k of stage s,
    # and B(s+1, m) at k or k-1 of stage s+1 when B(s, m) is op k (any pp, n_mb).
    for pp in range(1, 41):
        for n_mb in range(1, 80, 3):
            pos = _op_positions(pp, n_mb)
            f, b = _closed_positions(pp, n_mb)
            for s in range(pp):
                assert [pos[s][("F", m)] for m in range(n_mb)] == f[s].tolist()
                assert [pos[s][("B", m)] for m in range(n_mb)] == b[s].tolist()
    for pp in range(2, 129):
        for n_mb in list(range(1, 140)) + [255, 256, 257, 500, 511, 512, 1000, 1024]:
            f, b = _closed_positions(pp, n_mb)
            df = f[1:] - f[:-1]          # k(s) - index of F(s-1) in stage s-1
            db = b[:-1] - b[1:]          # k(s) - index of B(s+1) in stage s+1
            assert df.min() >= 0 and df.max() <= 1, (pp, n_mb)
            assert db.min() >= 0 and db.max() <= 1, (pp, n_mb)
