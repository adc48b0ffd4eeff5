"""Pins of the oracle's enumeration (Alg.1 l.3-5) and memory filter
(Alg.1 l.7, soft margin P:370; analytic estimator = DESIGN.md R11)
against facts that do not come from the oracle itself."""
import itertools
import math

import pytest

import oracle as O
import workloads as W
from des import simulate


def _triples(G, g, L=10**6, bs=None):
    cl = O.make_cluster(G // g, g)
    mo = O.make_model(L, 8, 2, 8, 16)
    bs = bs if bs is not None else G
    seen = []
    for c in O.enumerate_configs(cl, mo, bs):
        t = (c.pp, c.tp, c.dp)
        if not seen or seen[-1] != t:
            seen.append(t)
    return seen


def _n_ordered_factorizations3(G):
    # number of ordered triples with product G = prod_p C(e_p + 2, 2)
    n, out, p = G, 1, 2
    while n > 1:
        e = 0
        while n % p == 0:
            n //= p; e += 1
        out *= math.comb(e + 2, 2)
        p += 1
    return out


def test_spec_factorization_examples():
    # S:65 G=12 with g=12: 18 ordered triples (closed form 3*6)
    t = _triples(12, 12)
    assert len(t) == 18 == _n_ordered_factorizations3(12)
    # S:66 Fig.1: 12 GPUs, 3-way PP, 2-way TP, 2-way DP
    assert (3, 2, 2) in _triples(12, 2)
    # S:67 G=1
    assert _triples(1, 1) == [(1, 1, 1)]


@pytest.mark.parametrize("G,g", [(16, 8), (24, 4), (64, 8), (36, 6), (128, 8), (1024, 8), (96, 12)])
def test_enumeration_matches_brute_force_triples(G, g):
    got = _triples(G, g)
    want = [(pp, tp, G // (pp * tp)) for pp in range(1, G + 1) for tp in range(1, g + 1)
            if G % pp == 0 and g % tp == 0 and G % (pp * tp) == 0]
    assert got == want                      # same set AND canonical order (pp, tp ascending)
    if g == G:
        assert len(got) == _n_ordered_factorizations3(G)


def test_microbatch_loop_is_divisors_of_minibatch():
    cl = O.make_cluster(2, 4)
    mo = O.make_model(64, 8, 2, 8, 16)
    cf = O.enumerate_configs(cl, mo, 48)
    by = {}
    for c in cf:
        by.setdefault((c.pp, c.tp, c.dp), []).append(c.mb)
        assert c.n_mb * c.mb * c.dp == 48
    for (pp, tp, dp), mbs in by.items():
        assert mbs == [d for d in range(1, 48 // dp + 1) if (48 // dp) % d == 0]
    # dp must divide bs_global (Alg.1 l.4): bs=6 on 8 GPUs excludes dp in {4, 8}
    assert all(6 % c.dp == 0 for c in O.enumerate_configs(cl, mo, 6))
    assert [c.e for c in cf] == list(range(len(cf)))


def test_pp_bounded_by_layers():
    cl = O.make_cluster(4, 8)
    mo = O.make_model(6, 8, 2, 8, 16)
    assert max(c.pp for c in O.enumerate_configs(cl, mo, 32)) == 4   # divisors of 32 that are <= 6


def test_baseline_config_counts():
    # E and F at C1..C5 (computed at survey time by independent code)
    want = {"C1": (78, 78), "C2": (158, 62), "C3": (157, 57), "C4": (144, 35), "C5": (192, 16)}
    for k, (E, F) in want.items():
        w = W.WORKLOADS[k]
        m = w.model
        cl = O.make_cluster(w.n_nodes, w.gpus_per_node, w.cap_bytes, w.margin_permille)
        mo = O.make_model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
        cf = O.enumerate_configs(cl, mo, w.bs_global)
        assert len(cf) == E
        assert sum(c.feasible for c in cf) == F


# ----------------------------------------------------------------------------- memory
def test_memory_hand_arithmetic():
    # L=2 h=4 a=2 s=8 V=10, pp=2 tp=2 mb=1 n_mb=3 (worked by hand in DESIGN.md 5):
    # layer params 12*16+13*4 = 244; stage1 P = 244+40+32 = 316, W1 = 16*158 = 2528
    # act = ceil((8*1*4*44 + 5*2*64*1)/2) = 1024, in-flight min(2,3)=2 -> A1 = 2048
    mo = O.make_model(2, 4, 2, 8, 10)
    assert O.stage_memory(mo, 2, 2, 1, 3, 1) == 4576
    # stage 2: P = 244+40 (tied head), W2 = 16*142 = 2272, in-flight 1 -> 3296
    assert O.stage_memory(mo, 2, 2, 1, 3, 2) == 3296
    assert O.memory(mo, 2, 2, 1, 3) == 4576
    # L=5, pp=2 -> 3 layers/stage; tp=1 mb=2 n_mb=1, overhead 7:
    # P1 = 3*244+40+32 = 804 -> 12864; act = 8*2*4*34 + 5*2*64*2 = 3456; A1 = 1*3*3456
    mo2 = O.make_model(5, 4, 2, 8, 10, overhead=7)
    assert O.stage_memory(mo2, 2, 1, 2, 1, 1) == 12864 + 10368 + 7


def test_memory_matches_published_closed_forms():
    # parameter count: Narayanan et al. SC21, P = 12 L h^2 + 13 L h + V h + s h (pp=tp=1)
    for (L, h, a, s, V) in [(24, 1024, 16, 1024, 50257), (32, 2560, 32, 2048, 50257), (3, 8, 2, 4, 7)]:
        with_w = O.make_model(L, h, a, s, V, bpps=1)
        no_w = O.make_model(L, h, a, s, V, bpps=0)
        P = O.stage_memory(with_w, 1, 1, 1, 1, 1) - O.stage_memory(no_w, 1, 1, 1, 1, 1)
        assert P == 12 * L * h * h + 13 * L * h + V * h + s * h
        # activations per layer, Korthikanti et al. 2022 Table 2, no parallelism: s b h (34 + 5 a s / h)
        for b in (1, 2, 4):
            A = O.stage_memory(no_w, 1, 1, b, 1, 1)
            assert A * h == L * s * b * h * (34 * h + 5 * a * s)
        # tensor parallel t without SP: s b h (10 + 24/t + 5 a s/(h t)), whenever it is an integer
        for t in (2, 4, 8):
            A = O.stage_memory(no_w, 1, t, 2, 1, 1)
            exact = s * 2 * h * (10 * h * t + 24 * h + 5 * a * s)
            assert A == L * -(-exact // (h * t))


def test_memory_is_stage_one_and_inflight_is_1f1b_bound():
    mo = O.make_model(16, 8, 2, 8, 16, bpps=0)        # activations only
    for pp in (1, 2, 3, 4, 8):
        for n_mb in (1, 2, 3, 5, 8, 17):
            per = [O.stage_memory(mo, pp, 1, 1, n_mb, s) for s in range(1, pp + 1)]
            _, peaks = simulate(pp, n_mb, 1.0, 2.0)            # independent DES of Fig.2b
            unit = per[-1] // peaks[-1]
            assert [v // unit for v in per] == peaks         # in-flight = DES peak
            assert all(v % unit == 0 for v in per)
            _, gp = simulate(pp, n_mb, 1.0, 2.0, schedule="gpipe")
            assert gp[0] == n_mb                             # Fig.2a keeps every microbatch
    full = O.make_model(32, 2560, 32, 2048, 50257)
    for pp in (1, 2, 4, 8, 16, 32):
        for tp in (1, 2, 4, 8):
            for mb, n_mb in ((1, 64), (4, 2), (8, 1)):
                per = [O.stage_memory(full, pp, tp, mb, n_mb, s) for s in range(1, pp + 1)]
                assert O.memory(full, pp, tp, mb, n_mb) == max(per) == per[0]


def test_memory_monotone_in_microbatch():
    mo = O.make_model(32, 2560, 32, 2048, 50257)
    for pp, tp in itertools.product((1, 2, 4, 8), (1, 2, 8)):
        vals = [O.memory(mo, pp, tp, mb, 512 // mb) for mb in (1, 2, 4, 8, 16)]
        assert vals == sorted(vals)


def test_soft_margin_rule():
    MiB = 1 << 20
    # predicted 30000 MiB vs 32768 MiB with a 10% margin -> threshold 29491.2 MiB
    assert not O.feasible(30000 * MiB, 32768 * MiB, 100)
    assert O.feasible(29491 * MiB, 32768 * MiB, 100)
    assert not O.feasible(29492 * MiB, 32768 * MiB, 100)
    assert O.feasible(0, 32768 * MiB, 100)
    assert O.feasible(32768 * MiB, 32768 * MiB, 0)          # boundary inclusive
    assert not O.feasible(32768 * MiB + 1, 32768 * MiB, 0)
    cap = 80_000_000_000
    assert O.feasible(72_000_000_000, cap, 100) and not O.feasible(72_000_000_001, cap, 100)
