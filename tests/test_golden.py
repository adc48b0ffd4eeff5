"""The oracle against the golden fixtures under tests/golden/ (each file carries its
citation): the Fig.4 toy with hand-derived latencies and optimum, SPEC's worked values,
the Random123 Philox KATs, the survey's 1F1B DES table, and the enumeration counts."""
import itertools
import json
import os

import numpy as np
import pytest

import oracle as O
import workloads as W
from des import simulate

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def close(a, b, rel=1e-12):
    return abs(a - b) <= rel * max(abs(a), abs(b), 1e-300)


def test_every_fixture_cites_its_source():
    for name in sorted(os.listdir(GOLD)):
        assert "cite" in load(name), name


# ------------------------------------------------------------------ Fig.4 toy
def _fig4_R(g):
    n = len(g["nodes"])
    B = np.full((n, n), g["fast_Bps"])
    for a, b in g["slow_undirected_pairs"]:
        B[a, b] = B[b, a] = g["slow_Bps"]
    B[np.arange(n), np.arange(n)] = g["intra_Bps"]
    return O.inverse_bandwidth(B)


def _fig4_K(g):
    c = g["consts"]
    return O.raw_consts(c["pp"], c["dp"], c["spn"], c["n_nodes"], c["n_mb"], c["S"], c["m2"], c["md"])


def test_fig4_cases():
    g = load("fig4_toy.json")
    R, K = _fig4_R(g), _fig4_K(g)
    for case in g["cases"]:
        bd = O.latency(K, R, case["perm"])
        assert close(bd.T, case["T"]) and close(bd.t_pp, case["t_pp"]) and close(bd.t_dp, case["t_dp"]), case["name"]


def test_fig4_optimum_by_brute_force():
    g = load("fig4_toy.json")
    R, K = _fig4_R(g), _fig4_K(g)
    best = min(O.latency(K, R, list(p)).T for p in itertools.permutations(range(6)))
    assert close(best, g["optimum"]["T"])


# ------------------------------------------------------------------ SPEC worked values
def test_spec_worked_values():
    g = load("spec_worked_values.json")
    for case in g["cases"]:
        kind, n, inter, intra = case["bw"]
        assert kind == "uniform"
        R = O.inverse_bandwidth(W.uniform_bandwidth(n, inter, intra))
        bd = O.latency(O.raw_consts(*case["consts"]), R, case["perm"])
        for field, want in case["expect"].items():
            got = getattr(bd, field)
            assert (got == want) if want == 0.0 else close(got, want, g["tolerance_rel"]), (case["cite"], field, got)


# ------------------------------------------------------------------ Philox KATs (R14)
def test_philox_known_answers():
    for v in load("philox_kat.json")["vectors"]:
        ctr = [int(x, 16) for x in v["ctr"]]
        key = [int(x, 16) for x in v["key"]]
        assert tuple(O.philox(ctr, key)) == tuple(int(x, 16) for x in v["out"])


# ------------------------------------------------------------------ 1F1B DES table (R6)
@pytest.mark.parametrize("row", load("des_1f1b_uniform_hops.json")["rows"], ids=lambda r: f"pp{r['pp']}-nmb{r['n_mb']}")
def test_des_table(row):
    pp, n_mb = row["pp"], row["n_mb"]
    # one stage per node (spn = 1), one-way hop time 1: m2 * R = 2 with R = 1/B = 1
    R = O.inverse_bandwidth(W.uniform_bandwidth(pp, 1.0, 1.0))
    K = O.raw_consts(pp, 1, 1, pp, n_mb, 2.0, 2.0, 0.0)
    assert close(O.latency(K, R, list(range(pp))).T, row["ours"])
    des, _ = simulate(pp, n_mb, 1.0, 1.0, [1.0] * (pp - 1))
    assert close(des, row["des"])


# ------------------------------------------------------------------ enumeration counts
def test_enumeration_counts():
    g = load("enumeration_counts.json")
    for ex in g["spec_examples"]:
        cl = O.make_cluster(ex["G"] // ex["g"], ex["g"])
        mo = O.make_model(10**6, 8, 2, 8, 16)
        triples = {(c.pp, c.tp, c.dp) for c in O.enumerate_configs(cl, mo, ex["G"])}
        assert len(triples) == ex["triples"]
    for name, want in g["workloads"].items():
        w = W.WORKLOADS[name]
        m = w.model
        cl = O.make_cluster(w.n_nodes, w.gpus_per_node, w.cap_bytes, w.margin_permille)
        mo = O.make_model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
        cfgs = O.enumerate_configs(cl, mo, w.bs_global)
        assert len(cfgs) == want["E"], name
        assert sum(1 for c in cfgs if c.feasible) == want["F"], name
