"""Pins of the oracle's latency model (Eq.3-6, readings R5-R10 of DESIGN.md)
against hand arithmetic, the Fig.4 toy, symmetry/monotonicity invariants, and an
independent discrete-event simulation of the 1F1B schedule (tests/des.py)."""
import itertools

import numpy as np
import pytest

import oracle as O
import workloads as W
from des import simulate

REL = 1e-12


def close(a, b, rel=REL):
    return abs(a - b) <= rel * max(abs(a), abs(b), 1e-300)


def _single_gpu_nodes(Bnodes):
    return O.inverse_bandwidth(np.asarray(Bnodes, dtype=np.float64))


# ------------------------------------------------------------ SPEC worked values
def test_t_bubble_and_straggler_examples():
    R = _single_gpu_nodes(W.uniform_bandwidth(3, 1e10, 1e12))
    # S:202 pp=1, C=2, T_TP=0.5 -> 2.5 (the (pp-1) term vanishes)
    K = O.raw_consts(1, 3, 1, 3, 1, 2.5, 0.0, 0.0)
    assert close(O.latency(K, R, [0, 1, 2]).t_bubble, 2.5)
    # S:203 pp=3, C=1, T_TP=0, per-hop t_pp=0.1 -> 3.2 (R6: Eq.5 sums the pp-1 hops)
    K = O.raw_consts(3, 1, 1, 3, 1, 1.0, 1e9, 0.0)           # m2 * R = 1e9/1e10 = 0.1 per hop
    bd = O.latency(K, R, [0, 1, 2])
    assert close(bd.t_bubble, 3.2) and close(bd.t_pp, 0.2)
    # S:204 pp=2, C=0, T_TP=0, t_pp=1 -> 1.0
    R2 = _single_gpu_nodes(W.uniform_bandwidth(2, 1.0, 1.0))
    K = O.raw_consts(2, 1, 1, 2, 1, 0.0, 1.0, 0.0)
    assert close(O.latency(K, R2, [0, 1]).t_bubble, 1.0)
    # S:212 t_straggler pp=4, C=1, T_TP=0.25 -> 3.75 ; pp=1 -> 0
    R4 = _single_gpu_nodes(W.uniform_bandwidth(4, 1e10, 1e12))
    assert close(O.latency(O.raw_consts(4, 1, 1, 4, 4, 1.25, 0.0, 0.0), R4, [0, 1, 2, 3]).t_straggler, 3.75)
    assert O.latency(O.raw_consts(1, 1, 1, 4, 4, 1.25, 0.0, 0.0), R4, [0]).t_straggler == 0.0


def test_t_pp_examples():
    # S:221 pp=2, one inter-node hop at 10 GB/s, msg_pp=1e9 B -> 0.2 s
    R = _single_gpu_nodes(W.uniform_bandwidth(2, 1e10, 3e11))
    K = O.raw_consts(2, 1, 1, 2, 2, 0.0, 2e9, 0.0)
    assert close(O.latency(K, R, [0, 1]).t_pp, 0.2)
    # pp=1 -> 0 (empty sum)
    assert O.latency(O.raw_consts(1, 2, 1, 2, 2, 0.0, 2e9, 0.0), R, [0, 1]).t_pp == 0.0
    # S:222 two dp paths, one containing a slow link -> the slow path's sum
    B = W.uniform_bandwidth(4, 1e10, 3e11)
    B[2, 3] = 5e9
    R = _single_gpu_nodes(B)
    K = O.raw_consts(2, 2, 1, 4, 2, 0.0, 2e9, 0.0)
    assert close(O.latency(K, R, [0, 1, 2, 3]).t_pp, 0.4)
    assert close(O.latency(K, R, [2, 3, 0, 1]).t_pp, 0.4)
    assert close(O.latency(K, R, [3, 2, 1, 0]).t_pp, 0.2)   # reverse direction is fast (directed B)


def test_t_dp_examples():
    # S:229 dp=1 -> 0
    R = _single_gpu_nodes(W.uniform_bandwidth(2, 1e10, 3e11))
    assert O.latency(O.raw_consts(2, 1, 1, 2, 2, 1.0, 2e9, 1e9), R, [0, 1]).t_dp == 0.0
    # S:230 |W_intra|=1, |W_inter|=2, msg_dp=1e9, B=10 GB/s -> 2*1*1e9/(2*1e10) = 0.1 s
    K = O.raw_consts(1, 2, 1, 2, 2, 1.0, 0.0, 1e9)
    bd = O.latency(K, R, [0, 1])
    assert close(bd.t_dp, 0.1) and bd.t_in == 0.0 and bd.k == 2
    # S:231 heterogeneous inter links {10, 5} GB/s in one ring -> the min (5 GB/s)
    B = W.uniform_bandwidth(3, 1e10, 3e11)
    B[2, 0] = 5e9
    R = _single_gpu_nodes(B)
    K = O.raw_consts(1, 3, 1, 3, 2, 1.0, 0.0, 1e9)
    assert close(O.latency(K, R, [0, 1, 2]).t_ex, (2 * 2 * 1e9) / (3 * 5e9))
    # intra term (Eq.6 first line): 4 DP peers on one node, 4(c-1)/c msg / B_intra
    R = _single_gpu_nodes(W.uniform_bandwidth(2, 1e10, 2e11))
    K = O.raw_consts(1, 4, 4, 2, 1, 1.0, 0.0, 1e9)           # 4 slots per node
    bd = O.latency(K, R, [0, 1, 2, 3])
    assert close(bd.t_in, 4 * 3 * 1e9 / (4 * 2e11)) and bd.t_ex == 0.0 and bd.k == 1


def test_t_pipette_examples():
    # S:236 pp=1, n_mb=4, C=1.0, T_TP=0.1, t_dp=0.3 -> 4.7 s
    R = _single_gpu_nodes(W.uniform_bandwidth(2, 1e10, 3e11))
    K = O.raw_consts(1, 2, 1, 2, 4, 1.1, 0.0, 3e9)           # qe(2)*R = 3e9/1e10 = 0.3
    assert close(O.latency(K, R, [0, 1]).T, 4.7)
    # S:237 pp=2, n_mb=2, C=2, rest 0 -> 6.0 (and the DES of the same schedule)
    K = O.raw_consts(2, 1, 1, 2, 2, 2.0, 0.0, 0.0)
    assert close(O.latency(K, R, [0, 1]).T, 6.0)
    assert simulate(2, 2, 1.0, 1.0)[0] == 6.0


# ------------------------------------------------------------------- 1F1B DES (P4)
def _pipeline(pp, n_mb, S, hop):
    B = W.uniform_bandwidth(pp, 1.0 / hop if hop else 1e300, 1e12)
    R = _single_gpu_nodes(B)
    K = O.raw_consts(pp, 1, 1, pp, n_mb, S, 2.0 if hop else 0.0, 0.0)
    return O.latency(K, R, list(range(pp))).T


@pytest.mark.parametrize("pp", [1, 2, 3, 4, 5, 6, 8])
def test_closed_form_equals_des_without_hops(pp):
    for n_mb in range(1, 8 * pp + 1):
        for f, b in ((1.0, 1.0), (1.0, 2.0), (2.0, 3.0)):
            des, _ = simulate(pp, n_mb, f, b)
            assert close(_pipeline(pp, n_mb, f + b, 0.0), des), (pp, n_mb, f, b)


@pytest.mark.parametrize("pp", [2, 3, 4, 6, 8])
def test_closed_form_vs_des_with_uniform_hops(pp):
    # R6 evidence: with a uniform one-way hop h the DES exceeds Eq.3-5 by exactly 2(pp-2)h
    for k in (1, 2, 4, 8):
        n_mb = k * pp
        for h in (1.0, 0.25):
            des, _ = simulate(pp, n_mb, 1.0, 1.0, [h] * (pp - 1))
            assert close(des - _pipeline(pp, n_mb, 2.0, h), 2 * (pp - 2) * h), (pp, n_mb, h)


def test_hidden_critical_path_grows_with_microbatches():
    # Eq.1 (T_prev) misses the 1F1B hidden paths; with hops its error grows with n_mb/pp
    pp, h = 4, 1.0
    for n_mb in (8, 16, 32):
        des, _ = simulate(pp, n_mb, 1.0, 1.0, [h] * (pp - 1))
        ours = _pipeline(pp, n_mb, 2.0, h)
        t_prev = (n_mb - 1) * 2.0 + pp * 2.0 + (pp - 1) * 2 * h      # Eq.1 with T_DP = 0
        assert abs(ours - des) < abs(t_prev - des)


# ------------------------------------------------------------------- Fig.4 toy (P9)
FIG4 = O.raw_consts(3, 2, 1, 6, 6, 1.0, 2e9, 1e10)


def test_fig4_alphabetical_and_dedicated():
    R = O.inverse_bandwidth(W.fig4_toy())
    # Fig.4a alphabetical: pipelines (a,b,c),(d,e,f); slow a->b, b->c, d->e; DP a<->d slow
    bd = O.latency(FIG4, R, [0, 1, 2, 3, 4, 5])
    assert close(bd.T, 9.8) and close(bd.t_pp, 0.4) and close(bd.t_dp, 1.0)
    # Fig.4b: "the pipeline group of node (a, b, c) is changed into node (f, b, d)"
    assert close(O.latency(FIG4, R, [5, 1, 3, 2, 4, 0]).T, 8.9)


def test_fig4_brute_force_optimum():
    R = O.inverse_bandwidth(W.fig4_toy())
    vals = np.array([O.latency(FIG4, R, list(p)).T for p in itertools.permutations(range(6))])
    assert close(vals.min(), 8.9)
    assert int(np.sum(np.abs(vals - 8.9) < 1e-9)) == 124
    assert close(9.8 / vals.min(), 1.101123595505618)


# ------------------------------------------------------------------- invariants (P5-P8, P13)
def _random_case(rng, n_nodes, spn, pp, dp):
    B = W.bandwidth_matrix(n_nodes, 0.3, 0.3, int(rng.integers(1 << 30)))
    K = O.raw_consts(pp, dp, spn, n_nodes, 4 * pp, 0.37, 2.0 * 3e8, 5e9)
    return B, K


def test_homogeneous_bandwidth_invariance():
    rng = np.random.default_rng(7)
    # spn = 1 (tp = g): only inter-node links are ever used, so uniform inter B suffices;
    # dp = 1 with spn > 1: hops may stay inside a node, so intra must equal inter too
    R1 = O.inverse_bandwidth(W.uniform_bandwidth(8, 1e10, 2e11))
    R = O.inverse_bandwidth(W.uniform_bandwidth(8, 1e10, 1e10))
    for (spn, pp, dp) in [(1, 2, 4), (1, 4, 2), (1, 8, 1), (2, 8, 1), (4, 4, 1)]:
        K = O.raw_consts(pp, dp, spn, 8, 2 * pp, 0.5, 1e9, 3e9)
        RR = R1 if spn == 1 else R
        ref = O.latency(K, RR, list(range(pp * dp))).T
        for _ in range(50):
            assert O.latency(K, RR, rng.permutation(pp * dp)).T == ref
    # spn > 1: latency depends on the mapping only through the stage-1 occupancy multiset (R19)
    K = O.raw_consts(2, 4, 2, 8, 4, 0.5, 1e9, 3e9)
    seen = {}
    for _ in range(300):
        p = rng.permutation(8)
        occ = tuple(sorted(np.bincount(p[::2] // 2, minlength=8)))
        T = O.latency(K, R, p).T
        assert seen.setdefault(occ, T) == T
    assert len(set(seen.values())) > 1
    # the counterexample of R19: 2 nodes x 2 GPUs, all B = 1e10, pp = dp = 2 -> 6.4 vs 7.4
    R2 = O.inverse_bandwidth(np.full((2, 2), 1e10))
    K = O.raw_consts(2, 2, 2, 2, 4, 1.0, 2e9, 1e10)
    assert close(O.latency(K, R2, [0, 1, 2, 3]).T, 6.4)
    assert close(O.latency(K, R2, [0, 2, 1, 3]).T, 7.4)


def test_node_relabeling_symmetry():
    rng = np.random.default_rng(11)
    for n_nodes, spn, pp, dp in [(4, 2, 2, 4), (8, 1, 4, 2), (6, 4, 3, 8), (8, 8, 8, 8)]:
        B, K = _random_case(rng, n_nodes, spn, pp, dp)
        R = O.inverse_bandwidth(B)
        sigma = rng.permutation(n_nodes)
        Bs = np.empty_like(B)
        Bs[np.ix_(sigma, sigma)] = B                     # node a is renamed sigma[a]
        Rs = O.inverse_bandwidth(Bs)
        for _ in range(20):
            p = rng.permutation(pp * dp)
            ps = sigma[p // spn] * spn + p % spn
            assert O.latency(K, R, p).T == O.latency(K, Rs, ps).T


def test_monotone_in_bandwidth():
    rng = np.random.default_rng(3)
    for n_nodes, spn, pp, dp in [(4, 2, 2, 4), (8, 1, 4, 2), (6, 4, 3, 8)]:
        B, K = _random_case(rng, n_nodes, spn, pp, dp)
        for _ in range(30):
            p = rng.permutation(pp * dp)
            a, b = rng.integers(n_nodes, size=2)
            B2 = B.copy()
            B2[a, b] *= rng.uniform(0.1, 0.99)
            assert O.latency(K, O.inverse_bandwidth(B2), p).T >= O.latency(K, O.inverse_bandwidth(B), p).T


def test_scaling_bandwidth_and_messages_by_powers_of_two():
    rng = np.random.default_rng(5)
    B, K = _random_case(rng, 8, 2, 4, 4)
    for j in (-3, 1, 7):
        K2 = O.raw_consts(4, 4, 2, 8, K.n_mb, K.S, K.m2 * 2.0 ** j, K.md * 2.0 ** j)
        for _ in range(10):
            p = rng.permutation(16)
            a, b = O.latency(K, O.inverse_bandwidth(B), p), O.latency(K2, O.inverse_bandwidth(B * 2.0 ** j), p)
            assert (a.t_pp, a.t_dp, a.T) == (b.t_pp, b.t_dp, b.T)


def test_degenerate_cases():
    # G = 1: T = n_mb * S
    R = O.inverse_bandwidth(np.array([[2e11]]))
    K = O.raw_consts(1, 1, 1, 1, 7, 0.3, 1e9, 1e9)
    bd = O.latency(K, R, [0])
    assert bd.T == 7.0 * 0.3 and bd.t_pp == 0.0 and bd.t_dp == 0.0
    # pp = 1 -> T_PP = 0 ; dp = 1 -> T_DP = 0
    B = W.bandwidth_matrix(4, 0.2, 0.2, 1)
    assert O.latency(O.raw_consts(1, 8, 2, 4, 8, 1.0, 1e9, 1e9), O.inverse_bandwidth(B), list(range(8))).t_pp == 0.0
    assert O.latency(O.raw_consts(8, 1, 2, 4, 8, 1.0, 1e9, 1e9), O.inverse_bandwidth(B), list(range(8))).t_dp == 0.0


def test_is_permutation():
    assert O.is_permutation([2, 0, 1])
    assert not O.is_permutation([0, 0, 1])
    assert not O.is_permutation([0, 3, 1])
