"""B200-native Pipette plan evaluator (arXiv 2405.18093) -- Python binding.

Thin ctypes layer over libpipette.so (include/pipette.h): it converts arguments and
results, nothing else.  Every step of the path (enumeration, memory filter, Eq.3-6
latency, SA chains, argmin, NCCL combine) runs in the library's CUDA kernels.  torch is
used only for device memory, streams and torch.distributed process groups.

    from paper_2405_18093_b200 import Pipette, Model
    pip = Pipette(n_nodes=8, gpus_per_node=8, bandwidth=B, profile=entries)
    plan = pip.search(Model(32, 2560, 32, 2048, 50257), bs_global=512, chains=1024,
                      iterations=10000, seed=1)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _abi

__all__ = ["Pipette", "Model", "PipetteError", "shard_items", "nccl_unique_id", "torch_host_allreduce", "STATUS"]

STATUS = {0: "ok", 1: "oom", 2: "invalid_config", 3: "invalid_mapping", 4: "no_profile"}


class PipetteError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"pipette status {status}: {msg}")
        self.status = status


@dataclass(frozen=True)
class Model:
    """GPT-style model shape (pipette_model)."""
    n_layers: int
    hidden: int
    heads: int
    seq_len: int
    vocab: int = 50257
    bytes_per_elem: int = 2
    bytes_per_param_state: int = 16
    overhead_bytes: int = 0

    def c(self) -> _abi.Model:
        return _abi.Model(self.n_layers, self.hidden, self.heads, self.seq_len, self.vocab,
                          self.bytes_per_elem, self.bytes_per_param_state, int(self.overhead_bytes))


@dataclass
class Plan:
    cfg: tuple
    n_mb: int
    latency_s: float
    t_bubble: float
    t_straggler: float
    t_pp: float
    t_dp: float
    mem_bytes: int
    cfg_index: int
    chain: int
    best_step: int
    perm: np.ndarray
    configs_enumerated: int
    configs_rejected_oom: int
    sa_steps: int
    sa_accepted: int
    timings_ms: dict = field(default_factory=dict)


def _plan(p: _abi.Plan, perm: np.ndarray) -> Plan:
    return Plan((p.cfg.pp, p.cfg.tp, p.cfg.dp, p.cfg.mb), p.n_mb, p.latency_s, p.t_bubble, p.t_straggler,
                p.t_pp, p.t_dp, int(p.mem_bytes), p.cfg_index, p.chain, p.best_step, perm[:p.n_slots].copy(),
                int(p.configs_enumerated), int(p.configs_rejected_oom), int(p.sa_steps), int(p.sa_accepted),
                {"enumerate": p.enumerate_ms, "sa": p.sa_ms, "argmin": p.argmin_ms, "combine": p.combine_ms})


def shard_items(n_items: int, rank: int, world: int) -> np.ndarray:
    """Items j that `rank` runs (R18: j mod world == rank), from the library's host logic."""
    L = _abi.lib()
    cnt = L.pipette_shard_items(n_items, rank, world, None, 0)
    out = np.zeros(max(1, cnt), dtype=np.int64)
    L.pipette_shard_items(n_items, rank, world, out.ctypes.data_as(C.POINTER(C.c_int64)), cnt)
    return out[:cnt]


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = _abi.lib().pipette_nccl_unique_id(buf)
    if st != 0:
        raise PipetteError(st, "ncclGetUniqueId failed")
    return buf.raw


def profile_bandwidth(devices=None, bytes_per_copy: int = 256 << 20, reps: int = 5):
    """NEXT-3: Alg.1 l.1 on this box (pipette_profile_bandwidth).  Returns (B, ms): the
    directed n x n bytes/s matrix over `devices` (default: every visible GPU) with the
    intra-GPU copy bandwidth on the diagonal, and the median copy times."""
    L = _abi.lib()
    if devices is None:
        import torch
        devices = list(range(torch.cuda.device_count()))
    devs = np.ascontiguousarray(devices, dtype=np.int32)
    n = len(devs)
    bw = np.zeros((n, n), dtype=np.float64)
    ms = np.zeros((n, n), dtype=np.float64)
    err = C.create_string_buffer(512)
    st = L.pipette_profile_bandwidth(n, devs.ctypes.data_as(C.POINTER(C.c_int32)), int(bytes_per_copy), int(reps),
                                     bw.ctypes.data_as(C.POINTER(C.c_double)), ms.ctypes.data_as(C.POINTER(C.c_double)),
                                     err, 512)
    if st != 0:
        raise PipetteError(st, err.value.decode())
    return bw, ms


def measure_peaks(device: int = 0) -> dict:
    """Measured FP64 (DADD + DMUL) and 32-bit ALU op rates of this GPU (roofline denominators)."""
    f, a = C.c_double(), C.c_double()
    st = _abi.lib().pipette_measure_peaks(device, C.byref(f), C.byref(a))
    if st != 0:
        raise PipetteError(st, "pipette_measure_peaks failed")
    sm = C.c_double()
    st = _abi.lib().pipette_measure_smem_bw(device, C.byref(sm))
    if st != 0:
        raise PipetteError(st, "pipette_measure_smem_bw failed")
    return {"fp64_ops_per_s": f.value, "alu_ops_per_s": a.value, "smem_bytes_per_s": sm.value}


def load_memory_mlp(path=None) -> dict:
    """The packaged Eq.7 MLP (data/mem_mlp.json, trained by tools/train_mem_mlp.py)."""
    import json
    import os
    path = path or os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "mem_mlp.json")
    with open(path) as f:
        return json.load(f)


_SIGN = np.uint64(1 << 63)


def torch_host_allreduce(group=None):
    """A pipette_dist.host_allreduce over a torch.distributed process group (e.g. gloo):
    the library hands over a host uint64 buffer and the op (0 min, 1 sum); this only moves
    it through dist.all_reduce (plumbing; uint64 order kept by flipping the sign bit)."""
    import torch
    import torch.distributed as dist

    def fn(user, buf, count, op):
        try:
            a = np.ctypeslib.as_array(buf, shape=(int(count),))
            if op == 0:
                a ^= _SIGN
            t = torch.from_numpy(a.view(np.int64))
            dist.all_reduce(t, op=dist.ReduceOp.MIN if op == 0 else dist.ReduceOp.SUM, group=group)
            if op == 0:
                a ^= _SIGN
            return 0
        except Exception:   # noqa: BLE001 -- reported to the library as a failed transport
            return 1
    return fn


class Pipette:
    """A pipette_ctx on one GPU.  For world > 1 pass rank/world/device and either the
    128-byte NCCL id from rank 0 (see `from_torch_distributed`) or `host_allreduce`, a
    callable (user, buf, count, op) -> int run on host buffers (`torch_host_allreduce`)."""

    def __init__(self, n_nodes: int, gpus_per_node: int, bandwidth, profile, mem_capacity_bytes: int = 80_000_000_000,
                 mem_margin_permille: int = 100, rank: int = 0, world: int = 1, device: int | None = None,
                 nccl_id: bytes | None = None, host_allreduce=None):
        import torch
        self._L = _abi.lib()
        self.n_nodes, self.gpus_per_node = int(n_nodes), int(gpus_per_node)
        self.rank, self.world = int(rank), int(world)
        self.device = torch.cuda.current_device() if device is None else int(device)
        B = np.ascontiguousarray(bandwidth, dtype=np.float64)
        if B.shape != (n_nodes, n_nodes):
            raise ValueError(f"bandwidth must be {n_nodes}x{n_nodes}")
        prof = list(profile)
        arr = (_abi.ProfileEntry * max(1, len(prof)))()
        for i, (tp, mb, c, t) in enumerate(prof):
            arr[i] = _abi.ProfileEntry(int(tp), int(mb), float(c), float(t))
        cl = _abi.Cluster(self.n_nodes, self.gpus_per_node, int(mem_capacity_bytes), int(mem_margin_permille))
        self._idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        self._host_ar = _abi.HOST_ALLREDUCE(host_allreduce) if host_allreduce is not None else _abi.HOST_ALLREDUCE()
        dist = _abi.Dist(self.rank, self.world, self.device,
                         C.cast(self._idbuf, C.c_void_p) if self._idbuf is not None else None, self._host_ar, None)
        h = C.c_void_p()
        st = self._L.pipette_init(C.byref(h), C.byref(cl), B.ctypes.data_as(C.POINTER(C.c_double)), arr,
                                  len(prof), C.byref(dist))
        if st != 0:
            raise PipetteError(st, self._L.pipette_last_error(None).decode())
        self._h = h

    @classmethod
    def from_torch_distributed(cls, n_nodes, gpus_per_node, bandwidth, profile, transport: str = "nccl", **kw):
        """Build a context on every rank of the default torch.distributed process group:
        transport "nccl": rank 0 creates the NCCL id, torch.distributed broadcasts it (plumbing
        only); "host": the combine's reductions go through the process group itself
        (`torch_host_allreduce`; e.g. gloo, or ranks sharing one GPU)."""
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(), dist.get_world_size()
        if transport == "host":
            dev = kw.pop("device", torch.cuda.current_device())
            return cls(n_nodes, gpus_per_node, bandwidth, profile, rank=rank, world=world, device=dev,
                       host_allreduce=torch_host_allreduce() if world > 1 else None, **kw)
        if transport != "nccl":
            raise ValueError(f"transport must be 'nccl' or 'host', not {transport!r}")
        obj = [nccl_unique_id() if rank == 0 else None]
        if world > 1:
            dist.broadcast_object_list(obj, src=0)
        dev = kw.pop("device", torch.cuda.current_device())
        return cls(n_nodes, gpus_per_node, bandwidth, profile, rank=rank, world=world, device=dev,
                   nccl_id=obj[0] if world > 1 else None, **kw)

    def _check(self, st):
        if st != 0:
            raise PipetteError(st, self._L.pipette_last_error(self._h).decode())

    def close(self):
        if getattr(self, "_h", None):
            self._L.pipette_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def last_launch_count(self) -> int:
        return int(self._L.pipette_last_launch_count(self._h))

    def last_search_stats(self) -> dict:
        """Work plan of the last search on this rank (pipette_last_search_stats)."""
        out = (C.c_int64 * 7)()
        k = int(self._L.pipette_last_search_stats(self._h, out, 7))
        keys = ("mode", "tasks", "chunks", "grid", "warps_per_block", "smem_bytes", "table_bytes")
        return {keys[i]: int(out[i]) for i in range(k)}

    def last_task_profile(self) -> np.ndarray:
        """(tasks, 4) uint64: [start ns, end ns, SM id, config e] of the last search's SA warp tasks."""
        n = int(self._L.pipette_last_task_profile(self._h, None, 0))
        out = np.zeros((max(1, n), 4), dtype=np.uint64)
        if n > 0:
            self._L.pipette_last_task_profile(self._h, out.ctypes.data_as(C.POINTER(C.c_uint64)), n)
        return out[:max(0, n)]

    def set_bandwidth(self, bandwidth):
        B = np.ascontiguousarray(bandwidth, dtype=np.float64)
        if B.shape != (self.n_nodes, self.n_nodes):
            raise ValueError("bandwidth shape")
        self._check(self._L.pipette_set_bandwidth(self._h, B.ctypes.data_as(C.POINTER(C.c_double))))

    def enumerate(self, model: Model, bs_global: int):
        """K1: (configs (E,4) int array, n_mb, mem_bytes uint64, feasible bool), canonical order."""
        m = model.c()
        E, F = C.c_int32(), C.c_int32()
        self._check(self._L.pipette_enumerate(self._h, C.byref(m), int(bs_global), C.byref(E), C.byref(F),
                                              None, None, None, None, 0))
        n = E.value
        cf = (_abi.Config * max(1, n))()
        nmb = np.zeros(max(1, n), dtype=np.int32)
        mem = np.zeros(max(1, n), dtype=np.uint64)
        fe = np.zeros(max(1, n), dtype=np.uint8)
        self._check(self._L.pipette_enumerate(self._h, C.byref(m), int(bs_global), C.byref(E), C.byref(F), cf,
                                              nmb.ctypes.data_as(C.POINTER(C.c_int32)),
                                              mem.ctypes.data_as(C.POINTER(C.c_uint64)),
                                              fe.ctypes.data_as(C.POINTER(C.c_uint8)), n))
        cfgs = np.array([(cf[i].pp, cf[i].tp, cf[i].dp, cf[i].mb) for i in range(n)], dtype=np.int64).reshape(n, 4)
        return cfgs, nmb[:n], mem[:n], fe[:n].astype(bool)

    # ------------------------------------------------------------------ eval stream
    def eval(self, model: Model, bs_global: int, cfg, perm, out=None, stream=None):
        """cfg: (n, 4) int16/uint16 CUDA tensor of (pp, tp, dp, mb); perm: (n, stride) int16
        CUDA tensor of slot ids.  Returns (latency f64, mem int64 [u64 bits], status uint8)
        CUDA tensors; asynchronous on `stream` (default: torch's current stream)."""
        import torch
        n = int(cfg.shape[0])
        if cfg.dtype not in (torch.int16, torch.uint16) or perm.dtype not in (torch.int16, torch.uint16):
            raise TypeError("cfg and perm must be 16-bit integer tensors")
        if not (cfg.is_cuda and perm.is_cuda and cfg.is_contiguous() and perm.is_contiguous()):
            raise ValueError("cfg and perm must be contiguous CUDA tensors")
        if out is None:
            out = (torch.empty(n, dtype=torch.float64, device=cfg.device),
                   torch.empty(n, dtype=torch.int64, device=cfg.device),
                   torch.empty(n, dtype=torch.uint8, device=cfg.device))
        lat, mem, status = out
        s = torch.cuda.current_stream(cfg.device) if stream is None else stream
        m = model.c()
        self._check(self._L.pipette_eval(self._h, C.byref(m), int(bs_global), n, cfg.data_ptr(), perm.data_ptr(),
                                         int(perm.shape[1]) if perm.dim() == 2 else 1, lat.data_ptr(),
                                         mem.data_ptr(), status.data_ptr(), C.c_void_p(s.cuda_stream)))
        return lat, mem, status

    def set_memory_model(self, params=None):
        """NEXT-4: Eq.7's MLP memory estimator (flat float64 parameters, e.g.
        load_memory_mlp()["params"]) for every later enumeration; None = analytic (R11)."""
        if params is None:
            self._check(self._L.pipette_set_memory_model(self._h, None, 0))
            return
        a = np.ascontiguousarray(np.asarray(params, dtype=np.float64))
        self._check(self._L.pipette_set_memory_model(self._h, a.ctypes.data_as(C.POINTER(C.c_double)), a.size))

    def eval_models(self, model: Model, bs_global: int, cfg, perm, stream=None):
        """NEXT-2: (T_Pipette Eq.3, T_prev Eq.1, T_DES 1F1B simulation, status) CUDA tensors
        of the candidates (same inputs as eval)."""
        import torch
        n = int(cfg.shape[0])
        if cfg.dtype not in (torch.int16, torch.uint16) or perm.dtype not in (torch.int16, torch.uint16):
            raise TypeError("cfg and perm must be 16-bit integer tensors")
        if not (cfg.is_cuda and perm.is_cuda and cfg.is_contiguous() and perm.is_contiguous()):
            raise ValueError("cfg and perm must be contiguous CUDA tensors")
        tp, tprev, tdes = (torch.empty(n, dtype=torch.float64, device=cfg.device) for _ in range(3))
        status = torch.empty(n, dtype=torch.uint8, device=cfg.device)
        s = torch.cuda.current_stream(cfg.device) if stream is None else stream
        m = model.c()
        self._check(self._L.pipette_eval_models(self._h, C.byref(m), int(bs_global), n, cfg.data_ptr(),
                                                perm.data_ptr(), int(perm.shape[1]) if perm.dim() == 2 else 1,
                                                tp.data_ptr(), tprev.data_ptr(), tdes.data_ptr(), status.data_ptr(),
                                                C.c_void_p(s.cuda_stream)))
        return tp, tprev, tdes, status

    # ------------------------------------------------------------------ search
    def search(self, model: Model, bs_global: int, chains: int, iterations: int, seed: int,
               alpha: float = 0.999, tau: float = 0.05, t0: float = 0.0, per_config: bool = False,
               chain_results: bool = False, trace_items=None, trace_cap: int = 0, stream=None,
               w_migrate: int = 0, w_reverse: int = 0):
        """Alg.1 on the device (collective when world > 1).  Returns the best Plan, plus
        (per-config plans, per-chain results, traces) when requested.  w_migrate and
        w_reverse (1/2048 units) enable the paper's full move set (R21); 0, 0 = swap only."""
        import torch
        s = torch.cuda.current_stream(self.device) if stream is None else stream
        self._check(self._L.pipette_set_stream(self._h, C.c_void_p(s.cuda_stream)))
        m = model.c()
        cap = self.n_nodes * self.gpus_per_node
        opts = _abi.SaOpts()
        opts.alpha, opts.tau, opts.t0 = float(alpha), float(tau), float(t0)
        opts.w_migrate, opts.w_reverse = int(w_migrate), int(w_reverse)
        keep = []
        n_items = 0
        if chain_results:
            n_items = int(self.enumerate(model, bs_global)[3].sum()) * int(chains)
        if chain_results:
            cres = (_abi.ChainResult * n_items)()
            for i in range(n_items):
                cres[i].rank = -1
            cperm = np.zeros((n_items, cap), dtype=np.uint16)
            opts.chains = cres
            opts.chain_perms = cperm.ctypes.data_as(C.POINTER(C.c_uint16))
            opts.chain_perm_stride = cap
            opts.chains_cap = n_items
            keep += [cres, cperm]
        if trace_items is not None:
            ti = np.ascontiguousarray(trace_items, dtype=np.int64)
            tr = (_abi.TraceRecord * max(1, len(ti) * trace_cap))()
            opts.trace_items = ti.ctypes.data_as(C.POINTER(C.c_int64))
            opts.n_trace = len(ti)
            opts.trace_cap = int(trace_cap)
            opts.trace = tr
            keep += [ti, tr]
        plan = _abi.Plan()
        pbuf = np.zeros(cap, dtype=np.uint16)
        plan.perm = pbuf.ctypes.data_as(C.POINTER(C.c_uint16))
        plan.perm_cap = cap
        pcs, pbufs, n_pc = None, [], 0
        if per_config:
            n_pc = max(1, int(self.enumerate(model, bs_global)[3].sum()))   # one plan per feasible config
            pcs = (_abi.Plan * n_pc)()
            for i in range(n_pc):
                b = np.zeros(cap, dtype=np.uint16)
                pbufs.append(b)
                pcs[i].perm = b.ctypes.data_as(C.POINTER(C.c_uint16))
                pcs[i].perm_cap = cap
        st = self._L.pipette_search(self._h, C.byref(m), int(bs_global), int(chains), int(iterations),
                                    int(seed) & 0xFFFFFFFFFFFFFFFF, C.byref(opts), C.byref(plan), pcs, n_pc)
        if st == _abi.NO_FEASIBLE:
            raise PipetteError(st, self._L.pipette_last_error(self._h).decode())
        self._check(st)
        best = _plan(plan, pbuf)
        result = {"plan": best}
        if per_config:
            F = int(plan.configs_enumerated - plan.configs_rejected_oom)
            result["per_config"] = [_plan(pcs[i], pbufs[i]) for i in range(min(F, n_pc))]
        if chain_results:
            rows = []
            for j in range(n_items):
                r = cres[j]
                if r.rank >= 0:
                    rows.append({"item": j, "best": r.best, "best_t_pp": r.best_t_pp, "best_t_dp": r.best_t_dp,
                                 "L0": r.L0, "best_step": r.best_step, "accepted": r.accepted,
                                 "cfg_index": r.cfg_index, "chain": r.chain, "rank": r.rank,
                                 "perm": cperm[j, :r.n_slots].copy()})
            result["chains"] = rows
        if trace_items is not None:
            tl = []
            for t in range(len(ti)):
                tl.append([(tr[t * trace_cap + i].i, tr[t * trace_cap + i].p, tr[t * trace_cap + i].q,
                            tr[t * trace_cap + i].accept, tr[t * trace_cap + i].latency) for i in range(trace_cap)])
            result["trace"] = tl
        return result
