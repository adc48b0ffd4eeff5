"""Pins of the oracle's full SA move set (NEXT-1: the paper's migration, swap and reverse
movements; move selection reading R21 of DESIGN.md)."""
import itertools
import json
import os

import numpy as np
import pytest

import oracle as O
import workloads as W

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
KIND = {"swap": O.SWAP, "migrate": O.MIGRATE, "reverse": O.REVERSE}


def test_spec_move_examples():
    g = json.load(open(os.path.join(GOLD, "sa_moves.json")))
    idx = {c: i for i, c in enumerate(g["string"])}
    for case in g["cases"]:
        out = O.apply_move(list(range(4)), KIND[case["kind"]], case["p"], case["q"])
        assert [g["string"][v] for v in out] == case["out"], case["cite"]
        assert list(out) == [idx[c] for c in case["out"]]


def _list_move(a, kind, p, q):
    # the textbook string operations (Python list semantics)
    a = list(a)
    if kind == O.SWAP:
        a[p], a[q] = a[q], a[p]
    elif kind == O.MIGRATE:
        x = a.pop(p)
        a.insert(q, x)
    else:
        lo, hi = min(p, q), max(p, q)
        a[lo:hi + 1] = a[lo:hi + 1][::-1]
    return a


@pytest.mark.parametrize("N", [2, 3, 5, 8, 13])
def test_moves_match_string_operations_and_undo(N):
    rng = np.random.default_rng(N)
    base = rng.permutation(N).astype(np.uint16)
    for p, q in itertools.permutations(range(N), 2):
        for kind in (O.SWAP, O.MIGRATE, O.REVERSE):
            out = O.apply_move(base, kind, p, q)
            assert list(out) == _list_move(base, kind, p, q)
            assert sorted(out) == sorted(base)                       # still a bijection (Eq.2)
            assert list(O.apply_move(out, kind, p, q, undo=True)) == list(base)


def test_move_kind_thresholds_and_frequencies():
    # t in [0, 2048): swap below 2048 - wm - wr, migrate below 2048 - wr, else reverse
    assert O.move_kind(0, 683, 682) == O.SWAP and O.move_kind(682, 683, 682) == O.SWAP
    assert O.move_kind(683, 683, 682) == O.MIGRATE and O.move_kind(1365, 683, 682) == O.MIGRATE
    assert O.move_kind(1366, 683, 682) == O.REVERSE and O.move_kind(2047, 683, 682) == O.REVERSE
    assert all(O.move_kind(t, 0, 0) == O.SWAP for t in range(2048))
    n, counts, ts = 30000, np.zeros(3), []
    for i in range(n):
        p, q, u, t = O.draw_move(i, 3, 5, 0xABCDEF, 17)
        assert (p, q, u) == O.draw(i, 3, 5, 0xABCDEF, 17)            # the swap draw is unchanged
        assert 0 <= t < 2048
        ts.append(t)
        counts[O.move_kind(t, 683, 682)] += 1
    expect = n * np.array([683, 683, 682]) / 2048
    assert np.sum((counts - expect) ** 2 / expect) < 13.8            # chi^2, 2 dof, p = 0.001
    # t is uniform on its 2048 values and independent of u's bits: 16 bins of t
    h = np.bincount(np.asarray(ts) >> 7, minlength=16)
    assert np.sum((h - n / 16) ** 2 / (n / 16)) < 37.7               # chi^2, 15 dof, p = 0.001


def test_swap_only_weights_reproduce_the_swap_chain():
    B = W.bandwidth_matrix(4, 0.3, 0.3, 11)
    R = O.inverse_bandwidth(B)
    K = O.raw_consts(4, 2, 2, 4, 16, 0.5, 2e8, 4e9)
    a = O.sa_chain(K, R, 500, 99, 1, 2, trace=True)
    b = O.sa_chain(K, R, 500, 99, 1, 2, trace=True, w_migrate=0, w_reverse=0)
    assert a.trace == b.trace and a.best == b.best and np.array_equal(a.best_perm, b.best_perm)


@pytest.mark.parametrize("wm,wr", [(683, 682), (1024, 0), (0, 1024), (2048, 0), (0, 2048)])
def test_trace_replay_with_all_moves(wm, wr):
    B = W.bandwidth_matrix(6, 0.3, 0.3, 5)
    R = O.inverse_bandwidth(B)
    K = O.raw_consts(4, 3, 2, 6, 12, 0.4, 3e8, 6e9)
    seed, chain, e, iters = 0x1234, 7, 3, 400
    out = O.sa_chain(K, R, iters, seed, chain, e, trace=True, w_migrate=wm, w_reverse=wr)
    perm = list(range(K.N))
    cur = O.latency(K, R, perm).T
    best, kinds = cur, set()
    for (i, p, q, acc, L) in out.trace:
        p2, q2, u, t = O.draw_move(i, chain, e, seed, K.N)
        assert (p, q) == (p2, q2)
        kind = O.move_kind(t, wm, wr)
        kinds.add(kind)
        cand = _list_move(perm, kind, p, q)
        assert L == O.latency(K, R, cand).T                          # each proposal = the definition
        if L <= cur:
            assert acc == 1                                          # downhill always accepted
        if acc:
            perm, cur = cand, L
            best = min(best, L)
    assert best == out.best
    assert O.latency(K, R, out.best_perm).T == out.best
    want = {O.SWAP} if wm == wr == 0 else ({O.MIGRATE} if wm == 2048 else ({O.REVERSE} if wr == 2048 else None))
    if want is not None:
        assert kinds == want


def test_full_move_set_reaches_fig4_optimum():
    R = O.inverse_bandwidth(W.fig4_toy())
    K = O.raw_consts(3, 2, 1, 6, 6, 1.0, 2e9, 1e10)
    bests = [O.sa_chain(K, R, 3000, 7 + s, 0, 0, w_migrate=683, w_reverse=682).best for s in range(10)]
    assert sum(abs(b - 8.9) < 1e-9 for b in bests) >= 9


def test_search_with_moves_is_sharding_invariant():
    w = W.WORKLOADS["C1"]
    B, prof = W.workload_inputs(w)
    m = w.model
    cl = O.make_cluster(w.n_nodes, w.gpus_per_node, w.cap_bytes, w.margin_permille)
    mo = O.make_model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
    P = O.make_profile(prof)
    r1 = O.search(cl, B, P, mo, w.bs_global, 2, 200, 5, w_migrate=683, w_reverse=682, world=1)
    r3 = O.search(cl, B, P, mo, w.bs_global, 2, 200, 5, w_migrate=683, w_reverse=682, world=3)
    assert (r1.latency, r1.cfg_index, r1.chain) == (r3.latency, r3.cfg_index, r3.chain)
    assert np.array_equal(r1.perm, r3.perm)
