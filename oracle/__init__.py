"""CPU oracle for Pipette (arXiv 2405.18093) -- ctypes wrapper around oracle/oracle.c.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this module.
The product package ``paper_2405_18093_b200`` never imports it, and the two share
no code (see oracle/oracle.h and DESIGN.md section 5).

Every function documents the PAPER.md passage ("P:n") it follows; the C source
holds the arithmetic, this file only marshals arguments.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_HDR = os.path.join(_HERE, "oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-Wall"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (no FMA contraction, no fast-math)."""
    stale = (not os.path.exists(_LIB)
             or os.path.getmtime(_LIB) < max(os.path.getmtime(_SRC), os.path.getmtime(_HDR)))
    if force or stale:
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class Cluster(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("gpus_per_node", C.c_int32),
                ("mem_capacity_bytes", C.c_uint64), ("mem_margin_permille", C.c_int32)]


class Model(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("hidden", C.c_int32), ("heads", C.c_int32),
                ("seq_len", C.c_int32), ("vocab", C.c_int32), ("bytes_per_elem", C.c_int32),
                ("bytes_per_param_state", C.c_int32), ("overhead_bytes", C.c_uint64)]


class Profile(C.Structure):
    _fields_ = [("tp", C.c_int32), ("mb", C.c_int32), ("c_layer_s", C.c_double), ("tp_layer_s", C.c_double)]


class Config(C.Structure):
    _fields_ = [("pp", C.c_int32), ("tp", C.c_int32), ("dp", C.c_int32), ("mb", C.c_int32),
                ("n_mb", C.c_int32), ("e", C.c_int32), ("mem_bytes", C.c_uint64),
                ("feasible", C.c_int32), ("has_profile", C.c_int32)]


class Consts(C.Structure):
    _fields_ = [("pp", C.c_int32), ("dp", C.c_int32), ("spn", C.c_int32), ("N", C.c_int32),
                ("n_nodes", C.c_int32), ("n_mb", C.c_int32),
                ("S", C.c_double), ("m2", C.c_double), ("md", C.c_double), ("r", C.c_double),
                ("Sb", C.c_double), ("Ss", C.c_double)]


class Breakdown(C.Structure):
    _fields_ = [("T", C.c_double), ("t_pp", C.c_double), ("t_in", C.c_double), ("t_ex", C.c_double),
                ("t_dp", C.c_double), ("t_bubble", C.c_double), ("t_straggler", C.c_double),
                ("k", C.c_int32)]


class ChainResult(C.Structure):
    _fields_ = [("best", C.c_double), ("best_t_pp", C.c_double), ("best_t_dp", C.c_double),
                ("L0", C.c_double), ("best_step", C.c_int32), ("accepted", C.c_uint32)]


class TraceRecord(C.Structure):
    _fields_ = [("i", C.c_uint32), ("p", C.c_uint16), ("q", C.c_uint16), ("accept", C.c_uint32),
                ("L", C.c_double)]


class Plan(C.Structure):
    _fields_ = [("status", C.c_int32), ("E", C.c_int32), ("F", C.c_int32), ("cfg", Config),
                ("bd", Breakdown), ("cfg_index", C.c_int32), ("chain", C.c_int32),
                ("best_step", C.c_int32), ("n_slots", C.c_int32),
                ("sa_steps", C.c_uint64), ("sa_accepted", C.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P = C.POINTER
        L.or_enumerate.argtypes = [P(Cluster), P(Model), C.c_int64, P(Profile), C.c_int32, P(Config), C.c_int32]
        L.or_enumerate.restype = C.c_int32
        L.or_stage_memory.argtypes = [P(Model), C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32]
        L.or_stage_memory.restype = C.c_uint64
        L.or_memory.argtypes = [P(Model), C.c_int32, C.c_int32, C.c_int32, C.c_int32]
        L.or_memory.restype = C.c_uint64
        L.or_feasible.argtypes = [C.c_uint64, C.c_uint64, C.c_int32]
        L.or_feasible.restype = C.c_int32
        L.or_constants.argtypes = [P(Cluster), P(Model), P(Config), P(Profile), C.c_int32, P(Consts)]
        L.or_constants.restype = C.c_int32
        L.or_qi.argtypes = [P(Consts), C.c_int32]
        L.or_qi.restype = C.c_double
        L.or_qe.argtypes = [P(Consts), C.c_int32]
        L.or_qe.restype = C.c_double
        L.or_inverse_bandwidth.argtypes = [P(C.c_double), C.c_int32, P(C.c_double)]
        L.or_latency.argtypes = [P(Consts), P(C.c_double), P(C.c_uint16), P(Breakdown)]
        L.or_latency.restype = C.c_double
        L.or_is_permutation.argtypes = [P(C.c_uint16), C.c_int32]
        L.or_is_permutation.restype = C.c_int32
        L.or_philox4x32_10.argtypes = [P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)]
        L.or_exp_det.argtypes = [C.c_double]
        L.or_exp_det.restype = C.c_double
        L.or_draw.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_int32,
                              P(C.c_uint32), P(C.c_uint32), P(C.c_double)]
        L.or_sa_chain.argtypes = [P(Consts), P(C.c_double), C.c_int32, C.c_uint64, C.c_uint32, C.c_uint32,
                                  C.c_double, C.c_double, C.c_double, P(ChainResult), P(C.c_uint16),
                                  P(TraceRecord), C.c_int32]
        L.or_search.argtypes = [P(Cluster), P(C.c_double), P(Profile), C.c_int32, P(Model), C.c_int64,
                                C.c_int32, C.c_int32, C.c_uint64, C.c_double, C.c_double, C.c_double,
                                C.c_int32, P(Plan), P(C.c_uint16), C.c_int32, P(C.c_double), P(C.c_int32)]
        L.or_search.restype = C.c_int32
        L.or_draw_move.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_int32,
                                   P(C.c_uint32), P(C.c_uint32), P(C.c_double), P(C.c_uint32)]
        L.or_move_kind.argtypes = [C.c_uint32, C.c_int32, C.c_int32]
        L.or_draw_ctr.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_int32,
                                  P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)]
        L.or_calibrate_beta.argtypes = [P(Consts), P(C.c_double), C.c_uint64, C.c_uint32, C.c_int32, C.c_int32,
                                        C.c_double]
        L.or_calibrate_beta.restype = C.c_double
        L.or_move_kind.restype = C.c_int32
        L.or_apply_move.argtypes = [P(C.c_uint16), C.c_int32, C.c_uint32, C.c_uint32]
        L.or_undo_move.argtypes = [P(C.c_uint16), C.c_int32, C.c_uint32, C.c_uint32]
        L.or_sa_chain_moves.argtypes = [P(Consts), P(C.c_double), C.c_int32, C.c_uint64, C.c_uint32, C.c_uint32,
                                        C.c_double, C.c_double, C.c_double, C.c_int32, C.c_int32, P(ChainResult),
                                        P(C.c_uint16), P(TraceRecord), C.c_int32]
        L.or_search_moves.argtypes = [P(Cluster), P(C.c_double), P(Profile), C.c_int32, P(Model), C.c_int64,
                                      C.c_int32, C.c_int32, C.c_uint64, C.c_double, C.c_double, C.c_double,
                                      C.c_int32, C.c_int32, C.c_int32, P(Plan), P(C.c_uint16), C.c_int32,
                                      P(C.c_double), P(C.c_int32)]
        L.or_search_moves.restype = C.c_int32
        L.or_log_det.argtypes = [C.c_double]
        L.or_log_det.restype = C.c_double
        L.or_mlp_param_count.restype = C.c_int64
        L.or_mlp_memory.argtypes = [P(C.c_double), P(C.c_double)]
        L.or_mlp_memory.restype = C.c_uint64
        L.or_set_memory_model.argtypes = [P(C.c_double)]
        L.or_des_1f1b.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_double, P(C.c_double), P(C.c_double)]
        L.or_des_1f1b.restype = C.c_double
        L.or_models.argtypes = [P(Consts), P(C.c_double), P(C.c_uint16), P(C.c_double), P(C.c_double),
                                P(C.c_double)]
        _lib = L
    return _lib


# --------------------------------------------------------------------------- helpers
def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u16ptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint16))


def make_cluster(n_nodes, gpus_per_node, cap=80_000_000_000, margin_permille=100) -> Cluster:
    return Cluster(n_nodes, gpus_per_node, int(cap), int(margin_permille))


def make_model(L, h, a, seq, V, bpe=2, bpps=16, overhead=0) -> Model:
    return Model(L, h, a, seq, V, bpe, bpps, int(overhead))


def make_profile(entries) -> tuple:
    """entries: iterable of (tp, mb, c_layer_s, tp_layer_s)."""
    entries = list(entries)
    arr = (Profile * max(1, len(entries)))()
    for i, (tp, mb, c, t) in enumerate(entries):
        arr[i] = Profile(int(tp), int(mb), float(c), float(t))
    return arr, len(entries)


def enumerate_configs(cluster: Cluster, model: Model, bs_global: int, profile=None) -> list:
    """Alg.1 l.3-5 with the memory filter of l.7."""
    prof, nprof = profile if profile is not None else make_profile([])
    E = lib().or_enumerate(C.byref(cluster), C.byref(model), bs_global, prof, nprof, None, 0)
    out = (Config * max(1, E))()
    lib().or_enumerate(C.byref(cluster), C.byref(model), bs_global, prof, nprof, out, E)
    return [out[i] for i in range(E)]


def stage_memory(model, pp, tp, mb, n_mb, s) -> int:
    return int(lib().or_stage_memory(C.byref(model), pp, tp, mb, n_mb, s))


def memory(model, pp, tp, mb, n_mb) -> int:
    return int(lib().or_memory(C.byref(model), pp, tp, mb, n_mb))


def feasible(mem, cap, margin_permille) -> bool:
    return bool(lib().or_feasible(int(mem), int(cap), int(margin_permille)))


def constants(cluster, model, cfg: Config, profile) -> Consts:
    prof, nprof = profile
    K = Consts()
    st = lib().or_constants(C.byref(cluster), C.byref(model), C.byref(cfg), prof, nprof, C.byref(K))
    if st != 0:
        raise KeyError(f"profile entry missing for tp={cfg.tp} mb={cfg.mb}")
    return K


def raw_consts(pp, dp, spn, n_nodes, n_mb, S, m2, md) -> Consts:
    """Constants from explicit values (same normative operation order as or_constants)."""
    K = Consts()
    K.pp, K.dp, K.spn, K.N, K.n_nodes, K.n_mb = pp, dp, spn, pp * dp, n_nodes, n_mb
    K.S, K.m2, K.md = float(S), float(m2), float(md)
    K.r = float(n_mb) / float(pp)
    K.Sb = float(pp) * K.S
    K.Ss = float(pp - 1) * K.S
    return K


def inverse_bandwidth(B: np.ndarray) -> np.ndarray:
    B = np.ascontiguousarray(B, dtype=np.float64)
    n = B.shape[0]
    R = np.empty_like(B)
    lib().or_inverse_bandwidth(_dptr(B), n, _dptr(R))
    return R


def latency(K: Consts, R: np.ndarray, perm) -> Breakdown:
    """Eq.3-6 of one mapping, from the definition."""
    R = np.ascontiguousarray(R, dtype=np.float64)
    perm = np.ascontiguousarray(perm, dtype=np.uint16)
    assert perm.shape[0] == K.N
    bd = Breakdown()
    lib().or_latency(C.byref(K), _dptr(R), _u16ptr(perm), C.byref(bd))
    return bd


def qi(K, c):
    return lib().or_qi(C.byref(K), c)


def qe(K, k):
    return lib().or_qe(C.byref(K), k)


def is_permutation(perm) -> bool:
    perm = np.ascontiguousarray(perm, dtype=np.uint16)
    return bool(lib().or_is_permutation(_u16ptr(perm), perm.shape[0]))


def philox(ctr, key):
    c = (C.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    k = (C.c_uint32 * 2)(*[int(x) & 0xFFFFFFFF for x in key])
    o = (C.c_uint32 * 4)()
    lib().or_philox4x32_10(c, k, o)
    return tuple(o)


def exp_det(x: float) -> float:
    return lib().or_exp_det(float(x))


def draw(i, c, e, seed, N):
    p, q, u = C.c_uint32(), C.c_uint32(), C.c_double()
    lib().or_draw(i, c, e, seed, N, C.byref(p), C.byref(q), C.byref(u))
    return p.value, q.value, u.value


def log_det(x: float) -> float:
    return lib().or_log_det(float(x))


_mlp_keep = None


def set_memory_model(params):
    """Eq.7's MLP as the memory estimator of enumerate_configs (None: analytic, R11)."""
    global _mlp_keep
    if params is None:
        _mlp_keep = None
        lib().or_set_memory_model(None)
        return
    a = np.ascontiguousarray(np.asarray(params, dtype=np.float64))
    assert a.size == lib().or_mlp_param_count()
    _mlp_keep = a
    lib().or_set_memory_model(_dptr(a))


def mlp_memory(params, feat) -> int:
    a = np.ascontiguousarray(np.asarray(params, dtype=np.float64))
    f = np.ascontiguousarray(np.asarray(feat, dtype=np.float64))
    return int(lib().or_mlp_memory(_dptr(a), _dptr(f)))


def des_1f1b(pp, n_mb, f, b, hop_f, hop_b=None) -> float:
    """Makespan of one pipeline under the 1F1B schedule (NEXT-2, R22)."""
    hf = np.ascontiguousarray(np.asarray(hop_f if pp > 1 else [0.0], dtype=np.float64))
    hb = hf if hop_b is None else np.ascontiguousarray(np.asarray(hop_b if pp > 1 else [0.0], dtype=np.float64))
    return lib().or_des_1f1b(pp, n_mb, f, b, _dptr(hf), _dptr(hb))


def models(K: Consts, R: np.ndarray, perm):
    """(T_Pipette Eq.3, T_prev Eq.1, T_DES) of one plan (NEXT-2, R22)."""
    R = np.ascontiguousarray(R, dtype=np.float64)
    p = np.ascontiguousarray(np.asarray(perm, dtype=np.uint16))
    a, b, c = C.c_double(), C.c_double(), C.c_double()
    lib().or_models(C.byref(K), _dptr(R), _u16ptr(p), C.byref(a), C.byref(b), C.byref(c))
    return a.value, b.value, c.value


def draw_move(i, c, e, seed, N):
    """(p, q, u, t): the draw of R14 plus the 11-bit move selector t of R21."""
    p, q, u, t = C.c_uint32(), C.c_uint32(), C.c_double(), C.c_uint32()
    lib().or_draw_move(i, c, e, seed, N, C.byref(p), C.byref(q), C.byref(u), C.byref(t))
    return p.value, q.value, u.value, t.value


SWAP, MIGRATE, REVERSE = 0, 1, 2


def move_kind(t, w_migrate, w_reverse) -> int:
    return lib().or_move_kind(t, w_migrate, w_reverse)


def apply_move(perm, kind, p, q, undo=False) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(perm, dtype=np.uint16)).copy()
    (lib().or_undo_move if undo else lib().or_apply_move)(_u16ptr(a), kind, p, q)
    return a


@dataclass
class ChainOut:
    best: float
    best_t_pp: float
    best_t_dp: float
    L0: float
    best_step: int
    accepted: int
    best_perm: np.ndarray
    trace: list | None


def draw_ctr(i: int, c: int, e: int, d: int, seed: int, N: int):
    """One Philox draw of counter (i, c, e, d) as (p, q, t) (R14, R21; d = 1: R24's stream)."""
    p, q, t = C.c_uint32(), C.c_uint32(), C.c_uint32()
    lib().or_draw_ctr(i, c, e, d, seed, N, C.byref(p), C.byref(q), C.byref(t))
    return p.value, q.value, t.value


def calibrate_beta(K: Consts, R: np.ndarray, seed: int, e: int, w_migrate=0, w_reverse=0, tau=0.05) -> float:
    """SPEC S:448 (R24): 1/T0 with exp(-median|Delta| / T0) = 0.8 over 100 seeded moves of
    the identity mapping (counter (i, 0, e, 1)); 1/(tau L0) when the median is 0.  The SA
    chains use it when t0 < 0."""
    R = np.ascontiguousarray(R, dtype=np.float64)
    return float(lib().or_calibrate_beta(C.byref(K), _dptr(R), seed, e, w_migrate, w_reverse, tau))


def sa_chain(K: Consts, R: np.ndarray, iterations: int, seed: int, chain: int, e: int,
             alpha=0.999, tau=0.05, t0=0.0, trace: bool = False, w_migrate=0, w_reverse=0) -> ChainOut:
    """One SA chain of worker dedication; swap only unless move weights
    (1/2048 units, R21) are given."""
    R = np.ascontiguousarray(R, dtype=np.float64)
    res = ChainResult()
    bp = np.zeros(max(1, K.N), dtype=np.uint16)
    tr = (TraceRecord * iterations)() if trace and iterations > 0 else None
    if w_migrate == 0 and w_reverse == 0:
        lib().or_sa_chain(C.byref(K), _dptr(R), iterations, seed, chain, e, alpha, tau, t0,
                          C.byref(res), _u16ptr(bp), tr, iterations if tr is not None else 0)
    else:
        lib().or_sa_chain_moves(C.byref(K), _dptr(R), iterations, seed, chain, e, alpha, tau, t0, w_migrate,
                                w_reverse, C.byref(res), _u16ptr(bp), tr, iterations if tr is not None else 0)
    tlist = None
    if tr is not None:
        tlist = [(r.i, r.p, r.q, r.accept, r.L) for r in tr] if K.N >= 2 else []
    return ChainOut(res.best, res.best_t_pp, res.best_t_dp, res.L0, res.best_step, res.accepted,
                    bp[:K.N].copy(), tlist)


@dataclass
class SearchOut:
    status: int
    E: int
    F: int
    cfg: tuple
    n_mb: int
    mem_bytes: int
    latency: float
    t_pp: float
    t_dp: float
    t_bubble: float
    t_straggler: float
    cfg_index: int
    chain: int
    best_step: int
    perm: np.ndarray
    sa_steps: int
    sa_accepted: int
    per_config_best: np.ndarray
    per_config_chain: np.ndarray


def search(cluster, B, profile, model, bs_global, chains, iterations, seed,
           alpha=0.999, tau=0.05, t0=0.0, world=1, w_migrate=0, w_reverse=0) -> SearchOut:
    """Alg.1 with `world` simulated ranks (sharding + two-step min)."""
    B = np.ascontiguousarray(B, dtype=np.float64)
    prof, nprof = profile
    plan = Plan()
    cap = 65536
    perm = np.zeros(cap, dtype=np.uint16)
    E = len(enumerate_configs(cluster, model, bs_global, profile))
    pcb = np.full(max(1, E), np.inf)
    pcc = np.full(max(1, E), -1, dtype=np.int32)
    st = lib().or_search_moves(C.byref(cluster), _dptr(B), prof, nprof, C.byref(model), bs_global,
                               chains, iterations, seed, alpha, tau, t0, w_migrate, w_reverse, world,
                               C.byref(plan), _u16ptr(perm), cap, _dptr(pcb),
                               pcc.ctypes.data_as(C.POINTER(C.c_int32)))
    c = plan.cfg
    return SearchOut(st, plan.E, plan.F, (c.pp, c.tp, c.dp, c.mb), c.n_mb, int(c.mem_bytes),
                     plan.bd.T, plan.bd.t_pp, plan.bd.t_dp, plan.bd.t_bubble, plan.bd.t_straggler,
                     plan.cfg_index, plan.chain, plan.best_step, perm[:plan.n_slots].copy(),
                     int(plan.sa_steps), int(plan.sa_accepted), pcb[:plan.F].copy(), pcc[:plan.F].copy())
