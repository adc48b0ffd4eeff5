"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NO arithmetic of the method (no memory model, no latency model,
no SA): only the input recipes of DESIGN.md section 6 -- cluster shapes, bandwidth
matrices with per-link variance, profile tables, model shapes, random candidate
mappings.  Both sides receive the same numpy arrays from here.

Recipe (after SURVEY.md 8(d)):
  * g = 8 GPUs per node, the paper's node shape.
  * intra[a] = 240e9 * U(0.95, 1.0) B/s (attained NCCL busbw of an NVSwitch node).
  * inter[a][b] = 25e9 * clip(LogNormal(0, sigma), 0.5, 1.0) B/s (HDR 200 Gb/s),
    then a planted fraction f_slow of directed pairs * 0.5 (the 2x of P:227).
  * c_layer = (72 mb s h^2 + 12 mb s^2 h) / (tp * 312e12 * 0.5) s  (Megatron fwd+bwd
    flops per layer, A100 bf16 at 50%), tp_layer = [tp>1] 4 (2(tp-1)/tp) 2 mb s h / 240e9 s.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

V_GPT = 50257


@dataclass(frozen=True)
class ModelSpec:
    name: str
    n_layers: int
    hidden: int
    heads: int
    seq_len: int
    vocab: int = V_GPT
    bytes_per_elem: int = 2
    bytes_per_param_state: int = 16
    overhead_bytes: int = 0


@dataclass(frozen=True)
class Workload:
    name: str
    n_nodes: int
    gpus_per_node: int
    model: ModelSpec
    bs_global: int
    cap_bytes: int
    margin_permille: int
    chains: int
    iterations: int
    sigma: float
    f_slow: float
    topo_seed: int

    @property
    def seed(self) -> int:
        return 0x2405180930000000 + int(self.name[1:])


GPT_345M = ModelSpec("GPT-345M", 24, 1024, 16, 1024)
GPT3_2_7B = ModelSpec("GPT-3 2.7B", 32, 2560, 32, 2048)
GPT3_6_7B = ModelSpec("GPT-3 6.7B", 32, 4096, 32, 2048)
GPT3_13B = ModelSpec("GPT-3 13B", 40, 5120, 40, 2048)
GPT_39B = ModelSpec("GPT 39B", 48, 8192, 64, 2048)

# BASELINE.json "configs" C1..C5.
WORKLOADS = {
    "C1": Workload("C1", 2, 8, GPT_345M, 64, 80_000_000_000, 100, 1, 1000, 0.10, 0.10, 1),
    "C2": Workload("C2", 8, 8, GPT3_2_7B, 512, 80_000_000_000, 100, 1024, 10000, 0.10, 0.10, 2),
    "C3": Workload("C3", 16, 8, GPT3_6_7B, 512, 80_000_000_000, 100, 8192, 10000, 0.25, 0.20, 3),
    "C4": Workload("C4", 32, 8, GPT3_13B, 512, 80_000_000_000, 100, 1024, 10000, 0.10, 0.10, 4),
    "C5": Workload("C5", 128, 8, GPT_39B, 1536, 80_000_000_000, 100, 65536, 10000, 0.10, 0.10, 5),
}


def divisors(n: int) -> list[int]:
    return [d for d in range(1, n + 1) if n % d == 0]


def bandwidth_matrix(n_nodes: int, sigma: float = 0.10, f_slow: float = 0.10, seed: int = 0,
                     inter_nominal: float = 25e9, intra_nominal: float = 240e9) -> np.ndarray:
    """n x n directed bandwidth matrix in bytes/s, diagonal = intra-node bandwidth."""
    rng = np.random.Generator(np.random.PCG64(seed))
    B = inter_nominal * np.clip(rng.lognormal(0.0, sigma, size=(n_nodes, n_nodes)), 0.5, 1.0)
    off = ~np.eye(n_nodes, dtype=bool)
    slow = (rng.random((n_nodes, n_nodes)) < f_slow) & off
    B = np.where(slow, B * 0.5, B)
    intra = intra_nominal * rng.uniform(0.95, 1.0, size=n_nodes)
    B[np.arange(n_nodes), np.arange(n_nodes)] = intra
    return np.ascontiguousarray(B, dtype=np.float64)


def uniform_bandwidth(n_nodes: int, inter: float, intra: float) -> np.ndarray:
    B = np.full((n_nodes, n_nodes), float(inter))
    B[np.arange(n_nodes), np.arange(n_nodes)] = float(intra)
    return B


def profile_entries(model: ModelSpec, gpus_per_node: int, bs_global: int) -> list[tuple]:
    """(tp, mb, c_layer_s, tp_layer_s) for tp | g and mb | bs_global."""
    s, h = model.seq_len, model.hidden
    out = []
    for tp in divisors(gpus_per_node):
        for mb in divisors(bs_global):
            c = (72.0 * mb * s * h * h + 12.0 * mb * s * s * h) / (tp * 312e12 * 0.5)
            t = 0.0 if tp == 1 else 4.0 * (2.0 * (tp - 1) / tp) * (2.0 * mb * s * h) / 240e9
            out.append((tp, mb, c, t))
    return out


def workload_inputs(w: Workload):
    """(B, profile entries) for a BASELINE config."""
    B = bandwidth_matrix(w.n_nodes, w.sigma, w.f_slow, w.topo_seed)
    return B, profile_entries(w.model, w.gpus_per_node, w.bs_global)


def random_perms(N: int, count: int, seed: int) -> np.ndarray:
    """count x N uint16 uniformly random permutations (argsort of seeded uniform keys)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    keys = rng.random((count, N))
    return np.argsort(keys, axis=1, kind="stable").astype(np.uint16)


def fig4_toy():
    """The six-node toy of Fig.4 as a fixture: nodes a..f, one GPU
    each, 2e10 B/s links except 1e10 on the undirected pairs {a,b},{b,c},{d,e},{a,d};
    intra 3e11.  pp=3, dp=2, tp=1, n_mb=6, S=1 s, msg_pp=1e9 B, msg_dp=1e10 B."""
    n = 6
    B = np.full((n, n), 2e10)
    for a, b in [(0, 1), (1, 2), (3, 4), (0, 3)]:
        B[a, b] = B[b, a] = 1e10
    B[np.arange(n), np.arange(n)] = 3e11
    return B
