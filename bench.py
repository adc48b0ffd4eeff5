#!/usr/bin/env python
"""Benchmark of the Pipette hot path on B200 (contract: DESIGN.md section 8).

A step = one pipette_search (Alg.1: K1 enumerate + memory filter, K3 SA chains, K4 argmin,
NCCL combine) on BASELINE config C5 -- 1024 GPUs (128 nodes x 8),
GPT 39B, bs 1536, 65,536 SA chains x 10k swaps per feasible config -- the configuration
BASELINE.json ties to "sharded across 1/2/4/8 B200 with NCCL argmin".  Row a10 (the eval
stream) is measured beside it ("eval_stream"), and C2 (64 GPUs) is reported as an extra.

Multi-GPU (torchrun): STRONG scaling by default -- the 65,536 chains per config are one
fixed problem, work items j = f * chains + c are striped j mod W (R18), and the per-rank
winners are combined with NCCL; `--weak` runs chains * N instead.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload C1..C5] [--weak]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FP64_LANES_PER_SM = 64          # B200 (sm_100) FP64 units per SM per clock
N_SMS = 148
DEFAULT_WORKLOAD = "C5"


def ncu_traffic(kernel, workload):
    """Per-launch DRAM bytes of `kernel` on `workload` from the committed ncu capture (or None)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        d = d.get(f"{kernel}@{workload}") or (d.get(kernel) if workload == "C2" else None)
        return int(d["read_bytes"]) + int(d["write_bytes"]) if d else None
    except Exception:
        return None


def ncu_pipes(summary):
    """Pipe utilisation of a kernel from its committed ncu summary (profiles/), or None."""
    try:
        vals = {}
        for line in open(os.path.join(ROOT, "profiles", summary)):
            parts = line.split()
            if len(parts) >= 2 and not line.startswith("#"):
                try:
                    vals[parts[0]] = float(parts[1])
                except ValueError:
                    pass
        pick = {"issue_active": "smsp__issue_active.avg.pct_of_peak_sustained_active",
                "alu_pipe": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                "fma_pipe": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                "fp64_pipe": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                "lsu_pipe": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"}
        out = {k: vals[m] / 100 for k, m in pick.items() if m in vals}
        out["source"] = f"profiles/{summary}"
        return out if len(out) > 1 else None
    except Exception:
        return None


def peaks():
    try:
        return json.load(open(PEAKS))
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "fallback": True}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi-equivalent sampling (NVML) of SM clock and throttle reasons during the
    timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device: int):
        self.samples, self.reasons, self._stop = [], 0, threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                fn = getattr(self.nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    self.nv.nvmlDeviceGetCurrentClocksThrottleReasons
                self.reasons |= fn(self.h)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv and os.environ.get("PIPETTE_BENCH_NO_CLOCKS") != "1":
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv and hasattr(self, "t"):
            self.t.join()

    def summary(self):
        if not self.nv or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        rs = [name for bit, name in self.REASONS.items() if self.reasons & bit and name != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": rs,
                "samples": len(self.samples)}


# --------------------------------------------------------------------------- roofline counts
def fp64_ops_per_step(pp: int, dp: int) -> int:
    """Algorithmic FP64 operations of one SA proposal: re-sum of the two
    touched pipelines (pp-1 hops x (mul + add) each), Eq.3-4 composition (5), the
    Metropolis difference (1) and the temperature update (1)."""
    return (4 * (pp - 1) if pp >= 2 and dp >= 2 else 2 * (pp - 1)) + 7


# Philox4x32-10: 10 rounds x 2 IMAD.WIDE (FMA pipe) + 2 LOP3 (ALU); draw of p, q, u 8 (ALU);
# stage/pipeline of p and q and the touched hop positions 12 (ALU)
INT_ALU_OPS_PER_STEP = 20 + 8 + 12
INT_FMA_OPS_PER_STEP = 20


def smem_bytes_per_step(pp: int, dp: int) -> int:
    """Algorithmic shared-memory bytes of one SA proposal: the slot bytes of p
    and q read and written (12), the R term of every hop of the re-summed pipelines (8 B
    each), and the two cached pipeline sums read and written (32, pp >= 2)."""
    if pp < 2:
        return 4
    a = 2 if dp >= 2 else 1
    return 12 + 8 * a * (pp - 1) + 32


def setup(name: str):
    w = W.WORKLOADS[name]
    B, prof = W.workload_inputs(w)
    return w, B, prof


# --------------------------------------------------------------------------- CPU oracle legs
def _oracle_prep(w, B, prof):
    import oracle as O
    m = w.model
    cl = O.make_cluster(w.n_nodes, w.gpus_per_node, w.cap_bytes, w.margin_permille)
    mo = O.make_model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
    P = O.make_profile(prof)
    R = O.inverse_bandwidth(B)
    feas = [c for c in O.enumerate_configs(cl, mo, w.bs_global, P) if c.feasible]
    return O, R, [(c, O.constants(cl, mo, c, P)) for c in feas]


def oracle_sample(w, B, prof, seconds: float, threads: int = 1):
    """The CPU oracle (oracle/, as it stands) on a bounded sample of workload w: `threads`
    host threads (each one ctypes call per chain; ctypes releases the GIL, so the C oracle
    runs on that many cores), each taking full-length chains round-robin over the feasible
    configs, disjoint chain ids per thread, until `seconds`.  Returns (evals/s aggregate,
    seconds, chains)."""
    O, R, Ks = _oracle_prep(w, B, prof)
    counts = [0] * threads
    stop = time.perf_counter() + seconds

    def worker(t):
        i = t
        while time.perf_counter() < stop:
            c, K = Ks[i % len(Ks)]
            O.sa_chain(K, R, w.iterations, w.seed, i // len(Ks), c.e)
            counts[t] += w.iterations if K.N >= 2 else 0
            i += threads

    t0 = time.perf_counter()
    ths = [threading.Thread(target=worker, args=(t,)) for t in range(threads)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    dt = time.perf_counter() - t0
    steps = sum(counts)
    return steps / dt, dt, steps // max(1, w.iterations)


def cpu_baseline(w, B, prof, seconds: float):
    """cpu_baseline of the bench line: the oracle on one core and on every host core."""
    cores = host_cores()
    v1, dt1, n1 = oracle_sample(w, B, prof, seconds / 2, threads=1)
    vn, dtn, nn = oracle_sample(w, B, prof, seconds / 2, threads=cores)
    return {"value": vn, "unit": "evals/s", "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"{nn} full-length ({w.iterations}-swap) chains of {w.name} round-robin over its feasible "
                      f"configs on {cores} host threads (disjoint chains, {dtn:.1f} s)",
            "single_core": {"value": v1, "cores": 1, "sample": f"{n1} chains, {dt1:.1f} s"}}


def run_reference(args):
    """--impl reference: the CPU oracle on the host cores (rank 0 only), same workload,
    metric and unit as our arm; each step a bounded sample of args.ref_seconds."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w, B, prof = setup(args.workload)
    cores = host_cores()
    import oracle as O
    m = w.model
    cl = O.make_cluster(w.n_nodes, w.gpus_per_node, w.cap_bytes, w.margin_permille)
    mo = O.make_model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)
    cfgs = O.enumerate_configs(cl, mo, w.bs_global, O.make_profile(prof))
    ref_config = run_config(w, args.weak, args.gpus, [c.pp * c.dp for c in cfgs if c.feasible], len(cfgs))
    for _ in range(args.warmup):
        oracle_sample(w, B, prof, min(0.5, args.ref_seconds), threads=cores)
    vals, secs, nch = [], 0.0, 0
    for _ in range(args.steps):
        v, dt, c = oracle_sample(w, B, prof, args.ref_seconds, threads=cores)
        vals.append(v); secs += dt; nch += c
    value = float(np.mean(vals))
    line = {"metric": "plan evaluations/sec", "value": value, "unit": "evals/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * secs / args.steps, "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (workloads/)",
            "config": ref_config,
            "timing": {"l2": "n/a (host)", "parallelism": f"host threads ({cores}), rank 0 only"},
            "cpu_baseline": {"value": value, "unit": "evals/s", "cores": cores, "kind": "oracle",
                             "cpu_model": cpu_model(),
                             "sample": f"{nch} full-length SA chains in total on {cores} host threads, round-robin "
                                       f"over the feasible configs, {args.ref_seconds:.0f} s per step x {args.steps} steps"},
            "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def run_config(w, weak: bool, world: int, n_per_feasible, n_enumerated: int) -> dict:
    """`config` of both arms (identical for the same workload): the workload and its size.
    n_per_feasible: N = pp*dp of every feasible configuration (a chain with N < 2 proposes nothing)."""
    chains = w.chains * world if weak else w.chains
    return {"workload": workload_text(w, weak), "chains_per_config": chains,
            "feasible_configs": len(n_per_feasible), "enumerated_configs": int(n_enumerated),
            "sa_proposals_per_step": int(sum(chains * w.iterations for N in n_per_feasible if N >= 2))}


def workload_text(w, weak: bool) -> str:
    return (f"{w.name}: {w.n_nodes * w.gpus_per_node} GPUs ({w.n_nodes} nodes x {w.gpus_per_node}), {w.model.name}, "
            f"bs_global {w.bs_global}, {w.chains} SA chains/config{'/GPU' if weak else ''} x {w.iterations} swaps")


# --------------------------------------------------------------------------- our arm
def sa_roofline(cfgs, feas, chains, iterations, world, sa_avg_s, measured, pk, workload):
    """Roofline of k_sa_chains: algorithmic FP64, ALU, FMA and SMEM work per
    proposal against measured peaks; frac = roofline time / measured kernel time."""
    ops = alu = fma = sbytes = props = props1 = 0
    for (pp, tp, dp, mb), f in zip(cfgs.tolist(), feas.tolist()):
        if f and pp * dp >= 2:
            n = chains * iterations
            ops += fp64_ops_per_step(pp, dp) * n
            alu += INT_ALU_OPS_PER_STEP * n
            fma += INT_FMA_OPS_PER_STEP * n
            sbytes += smem_bytes_per_step(pp, dp) * n
            props += n
            if pp == 1:
                props1 += n
    mhz = pk.get("sm_max_mhz", 1965.0)
    fp64_nominal = N_SMS * FP64_LANES_PER_SM * mhz * 1e6
    fp64_peak = measured["fp64_ops_per_s"] if measured else fp64_nominal
    alu_peak = measured["alu_ops_per_s"] if measured else N_SMS * 64 * mhz * 1e6
    fma_peak = N_SMS * 128 * mhz * 1e6           # 4 SMSPs x 32 FMA lanes (IMAD.WIDE issues there)
    smem_peak = (measured or {}).get("smem_bytes_per_s") or N_SMS * 128 * mhz * 1e6
    loc = 1.0 / world
    ceil = {}
    for key, work, peak, unit in (("fp64", ops, fp64_peak, "DADD/DMUL per s"),
                                  ("alu", alu, alu_peak, "int32 ALU-pipe ops per s"),
                                  ("fma", fma, fma_peak, "FMA-pipe ops per s (IMAD.WIDE)"),
                                  ("smem", sbytes, smem_peak, "shared-memory B/s")):
        t = work * loc / peak
        ceil[key] = {"work_per_proposal": work / max(props, 1), "peak": peak, "unit": unit,
                     "bound_proposals_per_s": props * loc / t if t else None, "frac": t / sa_avg_s}
    binding = max(ceil, key=lambda k: ceil[k]["frac"])
    t_roof = max(c["frac"] for c in ceil.values()) * sa_avg_s
    return {"kernel": "k_sa_chains", "bound": "alu", "achieved": props * loc / sa_avg_s / 1e9,
            "peak": props * loc / t_roof / 1e9, "unit": "G proposals/s (min of FP64, ALU, FMA, SMEM ceilings)",
            "frac": t_roof / sa_avg_s, "binding_ceiling": binding, "ceilings": ceil,
            "fp64_achieved_tflops": ops * loc / sa_avg_s / 1e12, "fp64_peak_tflops": fp64_peak / 1e12,
            "peak_source": ("measured on this GPU (pipette_measure_peaks / _smem_bw); FMA pipe nominal 148 x 128 "
                            "x sm_max_mhz" if measured else "nominal (148 SMs x lanes x sm_max_mhz)"),
            "sa_kernel_ms": sa_avg_s * 1000.0,
            "pp1_share_of_proposals": props1 / max(props, 1),
            "traffic": ncu_traffic("k_sa_chains", workload),
            "traffic_note": "DRAM bytes per launch (ncu): chain state lives in shared memory, R and lists in L2",
            "pipes": ncu_pipes(f"r02_sa_{workload.lower()}_fullsize_ncu_digest.txt"),
            "note": "counts and ceilings in DESIGN.md 8; pipes = ncu pipe utilisation of the committed capture"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2405_18093_b200 import Model, Pipette

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        # stdout carries one JSON line: NCCL_DEBUG=VERSION makes NCCL printf its version banner
        # to stdout, so that level is lifted to WARN, and NCCL's log lines go to stderr.
        if os.environ.get("NCCL_DEBUG", "").upper() == "VERSION":
            os.environ["NCCL_DEBUG"] = "WARN"
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")    # > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def context(w, B, prof):
        kw = dict(mem_capacity_bytes=w.cap_bytes, mem_margin_permille=w.margin_permille)
        return (Pipette.from_torch_distributed(w.n_nodes, w.gpus_per_node, B, prof, device=local, **kw) if world > 1
                else Pipette(w.n_nodes, w.gpus_per_node, B, prof, device=local, **kw))

    def model_of(w):
        m = w.model
        return Model(m.n_layers, m.hidden, m.heads, m.seq_len, m.vocab)

    def timed_steps(pip, model, w, chains, steps):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        sa_ms, launches, res = [], 0, None
        barrier()
        with ClockSampler(local) as clk:
            for k in range(steps):
                if os.environ.get("PIPETTE_BENCH_NO_FLUSH") != "1":   # (diagnostics only)
                    flush.fill_(k & 0xFF)
                evs[k][0].record(stream)
                res = pip.search(model, w.bs_global, chains, w.iterations, w.seed)
                evs[k][1].record(stream)
                sa_ms.append(res["plan"].timings_ms["sa"])
                launches += pip.last_launch_count
            barrier()
        step_ms = [a.elapsed_time(b) for a, b in evs]
        t = torch.tensor([sum(step_ms), sum(sa_ms)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return res, step_ms, float(t[0]), float(t[1]), launches, clk.summary()

    w, B, prof = setup(args.workload)
    model = model_of(w)
    pip = context(w, B, prof)
    chains = w.chains * world if args.weak else w.chains

    # first call: enumeration read-back, host work plan, device tables, the search itself
    barrier()
    tc = time.perf_counter()
    res = pip.search(model, w.bs_global, chains, w.iterations, w.seed)
    torch.cuda.synchronize()
    cold_ms = (time.perf_counter() - tc) * 1000.0
    for _ in range(max(0, args.warmup - 1)):
        res = pip.search(model, w.bs_global, chains, w.iterations, w.seed)

    res, step_ms, t_max, sa_max, launches, clocks = timed_steps(pip, model, w, chains, args.steps)
    plan = res["plan"]
    evals_per_step = plan.sa_steps                    # global SA proposals (all ranks)
    value = evals_per_step * args.steps / (t_max / 1000.0)

    cfgs, nmb, mem, feas = pip.enumerate(model, w.bs_global)
    pk = peaks()
    measured = None
    try:   # DADD/DMUL, ALU and shared-memory rates measured on this GPU at this clock
        from paper_2405_18093_b200 import measure_peaks
        measured = measure_peaks(local)
    except Exception:
        pass
    sa_avg_s = (sa_max / args.steps) / 1000.0
    roofline = sa_roofline(cfgs, feas, chains, w.iterations, world, sa_avg_s, measured, pk, w.name)
    roofline["sa_share_of_step"] = (sa_max / t_max) if t_max else None

    # ---------------- e2e through the public API: host bandwidth matrix in, plan out
    e2e = None
    if not args.no_e2e:
        Bh = np.ascontiguousarray(B)
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for k in range(args.steps):
            pip.set_bandwidth(Bh)                     # H2D of the profiled matrix (Alg.1 l.1 output)
            pip.search(model, w.bs_global, chains, w.iterations, w.seed)   # D2H of the plan
        ev1.record(stream)
        barrier()
        te = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        F = int(feas.sum())
        row_words = 4 + (max(int(c[0] * c[2]) for c in cfgs[feas]) + 3) // 4
        e2e = {"value": evals_per_step * args.steps / (float(te[0]) / 1000.0), "unit": "evals/s",
               "h2d_bytes_per_step": int(Bh.nbytes), "d2h_bytes_per_step": int(8 * F * (row_words + 2) + 8)}

    # ---------------- extra workload (C2, 64 GPUs), same world and scaling, short
    extra = {}
    if not args.no_extra and args.workload != "C2":
        w2, B2, prof2 = setup("C2")
        pip2, model2 = context(w2, B2, prof2), model_of(w2)
        ch2 = w2.chains * world if args.weak else w2.chains
        for _ in range(2):
            pip2.search(model2, w2.bs_global, ch2, w2.iterations, w2.seed)
        r2, sm2, tm2, sa2, _, _ = timed_steps(pip2, model2, w2, ch2, 5)
        c2, _, _, f2 = pip2.enumerate(model2, w2.bs_global)
        props1 = sum(ch2 * w2.iterations for c, f in zip(c2.tolist(), f2.tolist()) if f and c[0] == 1 and c[2] >= 2)
        extra["C2"] = {"value": r2["plan"].sa_steps * 5 / (tm2 / 1000.0), "unit": "evals/s",
                       "ms_per_step": tm2 / 5, "workload": workload_text(w2, args.weak),
                       "pp1_share_of_proposals": props1 / max(1, r2["plan"].sa_steps),
                       "evals_with_arithmetic_per_s": (r2["plan"].sa_steps - props1) * 5 / (tm2 / 1000.0)}
        pip2.close()

    # ---------------- eval stream (row a10), HBM-bound, measured beside the step
    eval_stream = None
    if not args.no_eval and rank == 0:
        eval_stream = bench_eval(pip, model, w, cfgs, feas, pk, plan_cfg_index=plan.cfg_index)

    # ---------------- CPU baseline: the oracle on this host, rank 0 at N=1 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(w, B, prof, args.cpu_seconds)

    if rank == 0:
        line = {"metric": "plan evaluations/sec", "value": value, "unit": "evals/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max / args.steps,
                "time_to_best_plan_ms": {"warm": t_max / args.steps, "cold_first_call": cold_ms,
                                         "note": "warm: device time of one pipette_search (max over ranks); "
                                                 "cold: host wall time of the first call on rank 0 "
                                                 "(enumeration read-back, work plan, tables, search)"},
                "higher_is_better": True, "scaling": "weak" if args.weak else "strong", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (workloads/: B with per-link variance, Megatron-flop profile)",
                "config": run_config(w, args.weak, world, [int(c[0]) * int(c[2]) for c, f in zip(cfgs, feas) if f],
                                     len(feas)),
                "timing": {"l2": "flushed between timed steps (256 MiB write)",
                           "parallelism": f"chains striped j mod {world} (R18), NCCL combine"},
                "plan": {"cfg": list(plan.cfg), "latency_s": plan.latency_s, "cfg_index": plan.cfg_index,
                         "chain": plan.chain, "best_step": plan.best_step},
                "phase_ms": plan.timings_ms, "step_ms": [round(x, 3) for x in step_ms],
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
                "clocks": clocks, "eval_stream": eval_stream, "extra_workloads": extra or None}
        print(json.dumps(line))
    pip.close()
    if world > 1:
        dist.destroy_process_group()


def _eval_time(pip, model, w, cfg, perm, reps=5):
    import torch
    n = cfg.shape[0]
    out = (torch.empty(n, dtype=torch.float64, device="cuda"), torch.empty(n, dtype=torch.int64, device="cuda"),
           torch.empty(n, dtype=torch.uint8, device="cuda"))
    for _ in range(3):
        pip.eval(model, w.bs_global, cfg, perm, out=out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        pip.eval(model, w.bs_global, cfg, perm, out=out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 1000.0)
    return statistics.median(ts), out


def _perms(n, Ns, stride, seed):
    """n random mappings; row i is a uniform permutation of [0, Ns[i]) (padded to stride)."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    keys = torch.rand((n, stride), device="cuda", generator=g)
    col = torch.arange(stride, device="cuda").unsqueeze(0)
    keys = torch.where(col < Ns.unsqueeze(1), keys, 2.0 + col.to(keys.dtype))   # padding sorts last
    perm = torch.argsort(keys, dim=1).to(torch.int16)
    return perm.contiguous()


def bench_eval(pip, model, w, cfgs, feas, pk, n=1 << 22, plan_cfg_index=None):
    """pipette_eval (row a10) on 2^22 random mappings: (1) homogeneous batch of the search's
    best configuration, (2) mixed batch over every feasible config.  HBM
    roofline with 8 + 2N + 17 algorithmic bytes per candidate."""
    import torch
    fi = [i for i in range(len(feas)) if feas[i]]
    out = {}
    idx = plan_cfg_index if plan_cfg_index is not None else max(fi, key=lambda i: (cfgs[i][0] * cfgs[i][2], -i))
    for tag, rows in (("homogeneous", [idx] * n), ("mixed", [fi[k % len(fi)] for k in range(n)])):
        rows = np.asarray(rows)
        np.random.default_rng(3).shuffle(rows)
        cf = torch.from_numpy(cfgs[rows].astype(np.int16)).cuda().contiguous()
        Ns = torch.from_numpy((cfgs[rows, 0] * cfgs[rows, 2]).astype(np.int64)).cuda()
        stride = int(((Ns.max().item() + 7) // 8) * 8)
        perm = _perms(n, Ns, stride, 5)
        t, res = _eval_time(pip, model, w, cf, perm)
        alg = float((8 + 2 * Ns.double() + 17).sum().item())
        gbs = alg / t / 1e9
        st = res[2].cpu().numpy()
        out[tag] = {"value": n / t, "unit": "candidates/s", "batch": n, "stride": stride,
                    "configs": [list(map(int, cfgs[idx]))] if tag == "homogeneous" else int(len(fi)),
                    "status_ok_or_oom": bool(((st == 0) | (st == 1)).all()),
                    "roofline": {"kernel": "k_eval_stream", "bound": "hbm", "achieved": gbs,
                                 "peak": pk.get("hbm_gbs"), "unit": "GB/s", "frac": gbs / pk.get("hbm_gbs", 6538.3),
                                 "traffic": (ncu_traffic("k_eval_stream", w.name) if tag == "homogeneous" else None),
                                 "alg_bytes_per_candidate": alg / n,
                                 "note": f"batch {(n * stride * 2 + 25 * n) / 1e9:.2f} GB > L2"}}
        del perm, cf
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(W.WORKLOADS))
    ap.add_argument("--weak", action="store_true", help="chains x N per config (default: strong, fixed chains)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-eval", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--ref-seconds", type=float, default=5.0)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
