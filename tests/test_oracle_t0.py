"""Pins of the oracle's self-calibrated initial temperature (NEXT-1, reading R24
of DESIGN.md): 1/T0 = ln(1.25) / median|Delta| over 100 seeded moves of the identity, so
that the median move is accepted with probability exp(-median / T0) = 0.8."""
import math

import numpy as np
import pytest

import oracle as O
import workloads as W


def _list_move(a, kind, p, q):
    # the textbook string operations (Python list semantics, as tests/test_oracle_moves.py)
    a = list(a)
    if kind == O.SWAP:
        a[p], a[q] = a[q], a[p]
    elif kind == O.MIGRATE:
        a.insert(q, a.pop(p))
    else:
        lo, hi = min(p, q), max(p, q)
        a[lo:hi + 1] = a[lo:hi + 1][::-1]
    return a


def _c2_consts():
    w = W.WORKLOADS["C2"]
    B, prof = W.workload_inputs(w)
    m = w.model
    cl = O.make_cluster(w.n_nodes, w.gpus_per_node, w.cap_bytes, w.margin_permille)
    mo = O.make_model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
    P = O.make_profile(prof)
    feas = [c for c in O.enumerate_configs(cl, mo, w.bs_global, P) if c.feasible]
    return w, O.inverse_bandwidth(B), [(c, O.constants(cl, mo, c, P)) for c in feas]


def _independent_beta(K, R, seed, e, wm, wr, tau=0.05):
    """The calibration rebuilt from pinned pieces: the Philox draws (KAT-pinned), the
    textbook string moves, the definition of the latency, numpy's median and libm's log."""
    ident = list(range(K.N))
    L0 = O.latency(K, R, ident).T
    d = []
    for i in range(100):
        p, q, t = O.draw_ctr(i, 0, e, 1, seed, K.N)
        d.append(abs(O.latency(K, R, _list_move(ident, O.move_kind(t, wm, wr), p, q)).T - L0))
    med = float(np.median(np.asarray(d)))
    return (math.log(1.25) / med if med > 0 else 1.0 / (tau * L0)), med, L0


@pytest.mark.parametrize("wm,wr", [(0, 0), (683, 682)])
def test_calibration_matches_its_definition_and_accepts_the_median_move_with_p08(wm, wr):
    w, R, Ks = _c2_consts()
    checked = 0
    for c, K in Ks[::5]:
        beta = O.calibrate_beta(K, R, w.seed, c.e, wm, wr)
        ref, med, L0 = _independent_beta(K, R, w.seed, c.e, wm, wr)
        assert beta == ref, (c.e, beta, ref)
        if med > 0:
            checked += 1
            assert abs(math.exp(-med * beta) - 0.8) < 4e-16       # p(accept median) = 0.8
    assert checked >= 5


def test_draw_ctr_fourth_word_zero_is_the_sa_stream():
    # counter (i, c, e, 0) is the SA proposal's block (R14); word 1 is a disjoint stream
    for i, c, e, N in [(0, 0, 0, 7), (5, 3, 11, 64), (999, 17, 40, 256)]:
        p, q, t = O.draw_ctr(i, c, e, 0, 0x2405, N)
        p2, q2, _, t2 = O.draw_move(i, c, e, 0x2405, N)
        assert (p, q, t) == (p2, q2, t2)
    assert [O.draw_ctr(i, 0, 3, 1, 9, 1 << 20) for i in range(8)] != \
           [O.draw_ctr(i, 0, 3, 0, 9, 1 << 20)[:3] for i in range(8)]


def test_zero_median_falls_back_to_tau_l0():
    # pp = 1: every move keeps the latency (no hops, stage-1 multiset fixed), median 0
    B = W.bandwidth_matrix(4, 0.2, 0.3, 3)
    R = O.inverse_bandwidth(B)
    K = O.raw_consts(1, 8, 2, 4, 16, 0.02, 8e8, 2e9)
    L0 = O.latency(K, R, list(range(K.N))).T
    assert O.calibrate_beta(K, R, 77, 2, 0, 0, tau=0.05) == 1.0 / (0.05 * L0)


def test_calibrated_chain_decisions_follow_beta0():
    # trace replay: the chain with t0 < 0 starts from beta0 = calibrate_beta and every
    # uphill decision is u < exp_det(-(Delta * beta_i)), beta_i = beta_{i-1} / alpha
    B = W.bandwidth_matrix(6, 0.3, 0.3, 5)
    R = O.inverse_bandwidth(B)
    K = O.raw_consts(4, 3, 2, 6, 12, 0.4, 3e8, 6e9)
    seed, chain, e, iters, alpha = 0x77, 3, 9, 600, 0.999
    beta = O.calibrate_beta(K, R, seed, e)
    out = O.sa_chain(K, R, iters, seed, chain, e, alpha=alpha, t0=-1.0, trace=True)
    default = O.sa_chain(K, R, iters, seed, chain, e, alpha=alpha, trace=True)
    assert out.trace != default.trace                   # the temperature is not the tau default
    perm = list(range(K.N))
    cur = O.latency(K, R, perm).T
    ia = 1.0 / alpha
    uphill = 0
    for (i, p, q, acc, L) in out.trace:
        _, _, u = O.draw(i, chain, e, seed, K.N)
        cand = _list_move(perm, O.SWAP, p, q)
        assert L == O.latency(K, R, cand).T
        d = L - cur
        if d > 0:
            uphill += 1
            assert acc == (1 if u < O.exp_det(-(d * beta)) else 0), i
        else:
            assert acc == 1
        if acc:
            perm, cur = cand, L
        beta = beta * ia
    assert uphill > 50
