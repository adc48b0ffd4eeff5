"""Per-source-line totals (instructions executed, stall samples) from
`ncu -i X.ncu-rep --page source --csv --print-source cuda,sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out, fname, hdr = [], None, None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 3 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 10 or r[0] in ("", "Function Name"):
        continue
    try:
        ins = int(r[7]); samp = int(r[4]); thr = int(r[8])
    except ValueError:
        continue
    out.append((ins, samp, thr, f"{fname}:{r[0]}", r[1][:90]))
tot_i = sum(o[0] for o in out) or 1
tot_s = sum(o[1] for o in out) or 1
key = 1 if "--samples" in sys.argv else 0
out.sort(key=lambda o: -o[key])
print(f"total warp inst {tot_i:.3e}, samples {tot_s}")
for ins, samp, thr, loc, src in out[:top]:
    print(f"{100*ins/tot_i:5.1f}% inst {100*samp/tot_s:5.1f}% samp  lanes {thr/max(ins,1):4.1f}  {loc:18s} {src}")
