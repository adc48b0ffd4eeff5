"""Pins of NEXT-4: the memory estimator MLP of Eq.7, reading R23,
with the packaged parameters (paper_2405_18093_b200/data/mem_mlp.json)."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MLP = json.load(open(os.path.join(ROOT, "paper_2405_18093_b200", "data", "mem_mlp.json")))
PARAMS = np.asarray(MLP["params"], dtype=np.float64)


def test_log_det_is_within_an_ulp_of_libm():
    rng = np.random.default_rng(0)
    xs = np.concatenate([np.arange(1, 5000), rng.integers(1, 1 << 40, 5000)]).astype(np.float64)
    for x in xs:
        got, want = O.log_det(float(x)), math.log(float(x))
        assert abs(got - want) <= 2 * math.ulp(max(want, 1e-300)) or got == want, x
    for k in range(0, 60):
        assert O.log_det(float(2 ** k)) == k * 0.6931471805599453 or abs(O.log_det(float(2 ** k)) - k * math.log(2)) <= 4 * math.ulp(k * math.log(2) + 1e-300)


def _numpy_forward(feat):
    # the same network with numpy's matmul (a library primitive) and libm's log / exp
    p = PARAMS
    mean, sd = p[:10], p[10:20]
    x = (np.log(np.asarray(feat, dtype=np.float64)) - mean) / sd
    o, dims = 20, MLP["layers"]
    for l in range(5):
        n_in, n_out = dims[l], dims[l + 1]
        Wm = p[o:o + n_out * n_in].reshape(n_out, n_in); o += n_out * n_in
        b = p[o:o + n_out]; o += n_out
        x = Wm @ x + b
        if l < 4:
            x = np.maximum(x, 0.0)
    y_std, y_mean = p[o], p[o + 1]
    return math.exp(min(float(x[0]) * y_std + y_mean, 16.0)) * 1e9


def test_mlp_inference_matches_a_numpy_forward_pass():
    assert PARAMS.size == O.lib().or_mlp_param_count() == 123023
    rng = np.random.default_rng(1)
    for _ in range(200):
        n = int(rng.choice([8, 16, 32, 64, 128]))
        tp, pp = int(rng.choice([1, 2, 4, 8])), int(rng.choice([1, 2, 4, 8, 16]))
        dp = max(1, n // (tp * pp))
        bs = int(rng.choice([64, 256, 512]))
        mb = int(rng.choice([1, 2, 4]))
        feat = [n, 32, 2560, 32, tp, pp, dp, mb, max(1, bs // dp), bs]
        got, want = O.mlp_memory(PARAMS, feat), _numpy_forward(feat)
        assert abs(got - want) <= 1e-9 * want + 1, (feat, got, want)


def test_enumeration_with_the_mlp_filter():
    w = W.WORKLOADS["C2"]
    m = w.model
    cl = O.make_cluster(w.n_nodes, w.gpus_per_node, w.cap_bytes, w.margin_permille)
    mo = O.make_model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
    analytic = O.enumerate_configs(cl, mo, w.bs_global)
    O.set_memory_model(PARAMS)
    try:
        cfgs = O.enumerate_configs(cl, mo, w.bs_global)
    finally:
        O.set_memory_model(None)
    assert [(c.pp, c.tp, c.dp, c.mb) for c in cfgs] == [(c.pp, c.tp, c.dp, c.mb) for c in analytic]
    G = w.n_nodes * w.gpus_per_node
    errs = []
    for c, a in zip(cfgs, analytic):
        feat = [G, m.n_layers, m.hidden, m.heads, c.tp, c.pp, c.dp, c.mb, w.bs_global // c.dp, w.bs_global]
        assert c.mem_bytes == O.mlp_memory(PARAMS, feat)
        assert bool(c.feasible) == O.feasible(c.mem_bytes, w.cap_bytes, w.margin_permille)
        errs.append(abs(c.mem_bytes - a.mem_bytes) / a.mem_bytes)
    # an estimate of the analytic memory (64 GPUs: twice the training range)
    assert np.median(errs) < 0.25
    assert O.enumerate_configs(cl, mo, w.bs_global)[0].mem_bytes == analytic[0].mem_bytes   # reset works
