"""A tiny discrete-event simulator of one pipeline's training iteration.

Independent check of the closed-form 1F1B latency (Eq.3-4) and of the
1F1B in-flight bound used by the memory filter: it knows nothing of
Eq.3-6, it only executes the schedule of Fig.2 event by event.

Schedule (Megatron-LM's 1F1B op order, the "memory-efficient schedule" of P:110):
stage s (0-based) runs warm-up min(pp-s-1, n_mb) forwards, then alternates one
forward / one backward until its forwards are exhausted, then cools down with the
remaining backwards.  GPipe order (Fig.2a): all forwards, then all backwards.
Dependencies: F(s,m) after F(s-1,m) + hop(s-1); B(s,m) after B(s+1,m) + hop(s);
a stage runs one block at a time.  A hop delays only the dependency edge.
"""
from __future__ import annotations


def op_order(pp: int, n_mb: int, s: int, schedule: str = "1f1b") -> list[tuple[str, int]]:
    if schedule == "gpipe":
        return [("F", m) for m in range(n_mb)] + [("B", m) for m in range(n_mb)]
    warm = min(pp - s - 1, n_mb)
    ops, f, b = [], 0, 0
    for _ in range(warm):
        ops.append(("F", f)); f += 1
    for _ in range(n_mb - warm):
        ops.append(("F", f)); f += 1
        ops.append(("B", b)); b += 1
    for _ in range(warm):
        ops.append(("B", b)); b += 1
    return ops


def simulate(pp: int, n_mb: int, f: float, b: float, hops=None, schedule: str = "1f1b"):
    """Returns (makespan, peak_inflight per stage).  hops[s] = one-way delay s -> s+1."""
    hops = [0.0] * max(0, pp - 1) if hops is None else list(hops)
    orders = [op_order(pp, n_mb, s, schedule) for s in range(pp)]
    end = {}
    ptr = [0] * pp
    free = [0.0] * pp
    remaining = sum(len(o) for o in orders)
    while remaining:
        progressed = False
        for s in range(pp):
            while ptr[s] < len(orders[s]):
                kind, m = orders[s][ptr[s]]
                if kind == "F":
                    dep = 0.0
                    if s > 0:
                        if ("F", s - 1, m) not in end:
                            break
                        dep = end[("F", s - 1, m)] + hops[s - 1]
                    dur = f
                else:
                    if s < pp - 1:
                        if ("B", s + 1, m) not in end:
                            break
                        dep = end[("B", s + 1, m)] + hops[s]
                    else:
                        dep = end[("F", s, m)]
                    dur = b
                start = max(free[s], dep)
                end[(kind, s, m)] = start + dur
                free[s] = start + dur
                ptr[s] += 1
                remaining -= 1
                progressed = True
        if not progressed:
            raise RuntimeError("deadlock in schedule")
    peaks = []
    for s in range(pp):
        cur = peak = 0
        for kind, _ in orders[s]:
            cur += 1 if kind == "F" else -1
            peak = max(peak, cur)
        peaks.append(peak)
    return max(end.values()), peaks
