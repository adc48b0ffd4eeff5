"""Compact digest of an ncu report (run where ncu is, e.g. on the GPU box, so that only the
digest travels back): headline metrics, stall reasons per issue, and the top source lines
by executed warp instructions and by stall samples.

    python tools/ncu_digest.py REPORT.ncu-rep [units [lines.tsv]] > digest.txt

`units` (optional) divides the instruction counts (e.g. SA warp-steps = chains*iters/32).
"""
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
]


def run(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    units = float(sys.argv[2]) if len(sys.argv) > 2 else None
    rows = list(csv.reader(io.StringIO(run(rep, "--page", "raw", "--csv"))))
    d = dict(zip(rows[0], rows[2])) if len(rows) > 2 else {}
    u = dict(zip(rows[0], rows[1])) if len(rows) > 2 else {}
    print(f"# ncu digest of {rep}")
    for k in METRICS:
        if k in d:
            print(f"{k} {d[k].replace(',', '')} {u.get(k, '')}".rstrip())
    for k, v in d.items():
        if "issue_stalled" in k and k.endswith("per_issue_active.ratio"):
            try:
                if float(v) >= 0.02:
                    print(f"{k} {v}")
            except ValueError:
                pass
    if units and "smsp__inst_executed.sum" in d:
        print(f"warp_inst_per_unit {float(d['smsp__inst_executed.sum'].replace(',', '')) / units:.1f}")
    src = list(csv.reader(io.StringIO(run(rep, "--page", "source", "--csv", "--print-source", "cuda,sass"))))
    out, fname, hdr = [], None, None
    for r in src:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) > 3 and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 10 or r[0] in ("", "Function Name"):
            continue
        try:
            ins, samp, thr = int(r[7]), int(r[4]), int(r[8])
        except ValueError:
            continue
        out.append((ins, samp, thr, f"{fname}:{r[0]}", r[1][:80]))
    if len(sys.argv) > 3:   # the whole per-line table (file:line, warp inst, samples, thread inst)
        with open(sys.argv[3], "w") as f:
            for ins, samp, thr, loc, s in out:
                f.write(f"{loc}\t{ins}\t{samp}\t{thr}\n")
    ti = sum(o[0] for o in out) or 1
    ts = sum(o[1] for o in out) or 1
    for key, name in ((0, "instructions"), (1, "stall samples")):
        print(f"# top source lines by {name} (total warp inst {ti:.3e}, samples {ts})")
        for ins, samp, thr, loc, s in sorted(out, key=lambda o: -o[key])[:30]:
            per = f" {ins / units:7.1f}/unit" if units else ""
            print(f"{100 * ins / ti:5.1f}% inst{per} {100 * samp / ts:5.1f}% samp lanes {thr / max(ins, 1):4.1f}  {loc:20s} {s}")


if __name__ == "__main__":
    main()
