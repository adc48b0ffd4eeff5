"""ctypes mirror of include/pipette.h (argument marshalling only, no arithmetic).

The library is loaded from the package's lib/ directory; if it is missing the import
of the product API fails loudly -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PIPETTE_LIB") or os.path.join(_PKG, "lib", "libpipette.so")   # override: A/B tools only

OK, NO_FEASIBLE, E_INVALID, E_PROFILE, E_CUDA, E_NCCL, E_UNSUPPORTED = range(7)


class Cluster(C.Structure):
    _fields_ = [("n_nodes", C.c_int32), ("gpus_per_node", C.c_int32),
                ("mem_capacity_bytes", C.c_uint64), ("mem_margin_permille", C.c_int32)]


class ProfileEntry(C.Structure):
    _fields_ = [("tp", C.c_int32), ("mb", C.c_int32), ("c_layer_s", C.c_double), ("tp_layer_s", C.c_double)]


HOST_ALLREDUCE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_int64, C.c_int32)


class Dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("device", C.c_int32), ("nccl_unique_id", C.c_void_p),
                ("host_allreduce", HOST_ALLREDUCE), ("host_user", C.c_void_p)]


class Model(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("hidden", C.c_int32), ("heads", C.c_int32), ("seq_len", C.c_int32),
                ("vocab", C.c_int32), ("bytes_per_elem", C.c_int32), ("bytes_per_param_state", C.c_int32),
                ("overhead_bytes", C.c_uint64)]


class Config(C.Structure):
    _fields_ = [("pp", C.c_uint16), ("tp", C.c_uint16), ("dp", C.c_uint16), ("mb", C.c_uint16)]


class TraceRecord(C.Structure):
    _fields_ = [("i", C.c_uint32), ("p", C.c_uint16), ("q", C.c_uint16), ("accept", C.c_uint32),
                ("latency", C.c_double)]


class ChainResult(C.Structure):
    _fields_ = [("best", C.c_double), ("best_t_pp", C.c_double), ("best_t_dp", C.c_double), ("L0", C.c_double),
                ("best_step", C.c_int32), ("accepted", C.c_uint32), ("cfg_index", C.c_int32),
                ("chain", C.c_int32), ("rank", C.c_int32), ("n_slots", C.c_int32)]


class SaOpts(C.Structure):
    _fields_ = [("alpha", C.c_double), ("tau", C.c_double), ("t0", C.c_double),
                ("chains", C.POINTER(ChainResult)), ("chain_perms", C.POINTER(C.c_uint16)),
                ("chain_perm_stride", C.c_int32), ("chains_cap", C.c_int64),
                ("trace_items", C.POINTER(C.c_int64)), ("n_trace", C.c_int32), ("trace_cap", C.c_int32),
                ("trace", C.POINTER(TraceRecord)), ("w_migrate", C.c_int32), ("w_reverse", C.c_int32)]


class Plan(C.Structure):
    _fields_ = [("cfg", Config), ("n_mb", C.c_int32), ("latency_s", C.c_double), ("t_bubble", C.c_double),
                ("t_straggler", C.c_double), ("t_pp", C.c_double), ("t_dp", C.c_double),
                ("mem_bytes", C.c_uint64), ("cfg_index", C.c_int32), ("chain", C.c_int32),
                ("best_step", C.c_int32), ("n_slots", C.c_int32), ("perm", C.POINTER(C.c_uint16)),
                ("perm_cap", C.c_int32), ("configs_enumerated", C.c_uint64), ("configs_rejected_oom", C.c_uint64),
                ("sa_steps", C.c_uint64), ("sa_accepted", C.c_uint64), ("enumerate_ms", C.c_double),
                ("sa_ms", C.c_double), ("argmin_ms", C.c_double), ("combine_ms", C.c_double)]


EXPORTS = ("pipette_init", "pipette_enumerate", "pipette_set_bandwidth", "pipette_set_stream", "pipette_eval", "pipette_eval_models", "pipette_profile_bandwidth", "pipette_set_memory_model", "pipette_measure_peaks", "pipette_measure_smem_bw", "pipette_search",
           "pipette_shard_items", "pipette_nccl_unique_id", "pipette_last_launch_count", "pipette_last_search_stats", "pipette_last_task_profile", "pipette_destroy",
           "pipette_last_error", "pipette_strerror")

_lib = None


def lib() -> C.CDLL:
    """Load libpipette.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2405_18093_b200.build` "
                           "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    vp = C.c_void_p
    L.pipette_init.argtypes = [P(vp), P(Cluster), P(C.c_double), P(ProfileEntry), C.c_int32, P(Dist)]
    L.pipette_init.restype = C.c_int
    L.pipette_set_bandwidth.argtypes = [vp, P(C.c_double)]
    L.pipette_set_bandwidth.restype = C.c_int
    L.pipette_set_stream.argtypes = [vp, vp]
    L.pipette_set_stream.restype = C.c_int
    L.pipette_enumerate.argtypes = [vp, P(Model), C.c_int64, P(C.c_int32), P(C.c_int32), P(Config),
                                    P(C.c_int32), P(C.c_uint64), P(C.c_uint8), C.c_int32]
    L.pipette_enumerate.restype = C.c_int
    L.pipette_eval.argtypes = [vp, P(Model), C.c_int64, C.c_int64, vp, vp, C.c_int32, vp, vp, vp, vp]
    L.pipette_eval.restype = C.c_int
    L.pipette_eval_models.argtypes = [vp, P(Model), C.c_int64, C.c_int64, vp, vp, C.c_int32, vp, vp, vp, vp, vp]
    L.pipette_eval_models.restype = C.c_int
    L.pipette_profile_bandwidth.argtypes = [C.c_int32, P(C.c_int32), C.c_uint64, C.c_int32, P(C.c_double),
                                            P(C.c_double), C.c_char_p, C.c_int32]
    L.pipette_profile_bandwidth.restype = C.c_int
    L.pipette_set_memory_model.argtypes = [vp, P(C.c_double), C.c_int64]
    L.pipette_set_memory_model.restype = C.c_int
    L.pipette_measure_peaks.argtypes = [C.c_int32, P(C.c_double), P(C.c_double)]
    L.pipette_measure_smem_bw.argtypes = [C.c_int32, P(C.c_double)]
    L.pipette_measure_smem_bw.restype = C.c_int
    L.pipette_measure_peaks.restype = C.c_int
    L.pipette_search.argtypes = [vp, P(Model), C.c_int64, C.c_int32, C.c_int32, C.c_uint64, P(SaOpts),
                                 P(Plan), P(Plan), C.c_int32]
    L.pipette_search.restype = C.c_int
    L.pipette_shard_items.argtypes = [C.c_int64, C.c_int32, C.c_int32, P(C.c_int64), C.c_int64]
    L.pipette_shard_items.restype = C.c_int64
    L.pipette_nccl_unique_id.argtypes = [vp]
    L.pipette_nccl_unique_id.restype = C.c_int
    L.pipette_last_launch_count.argtypes = [vp]
    L.pipette_last_launch_count.restype = C.c_int64
    L.pipette_last_search_stats.argtypes = [vp, C.POINTER(C.c_int64), C.c_int32]
    L.pipette_last_search_stats.restype = C.c_int32
    L.pipette_last_task_profile.argtypes = [vp, P(C.c_uint64), C.c_int64]
    L.pipette_last_task_profile.restype = C.c_int64
    L.pipette_destroy.argtypes = [vp]
    L.pipette_destroy.restype = None
    L.pipette_last_error.argtypes = [vp]
    L.pipette_last_error.restype = C.c_char_p
    L.pipette_strerror.argtypes = [C.c_int]
    L.pipette_strerror.restype = C.c_char_p
    _lib = L
    return L
