"""Static check of the no-contraction rule in the built library's SASS:
every DFMA of the hot kernels must belong to a correctly rounded division (__ddiv_rn:
a MUFU.RCP64H followed by DFMA Newton steps), never to model arithmetic.

    python tools/sass_fma_check.py [libpipette.so]   -> JSON per kernel"""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HOT = ("k_sa_chains", "k_eval_stream", "k_models")
WINDOW = 96   # instructions after a MUFU.RCP64H that belong to its division sequence (incl. the slow path)


def analyse(lib):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur and re.search(r"/\*[0-9a-f]{4,}\*/", line):
            funcs[cur].append(line)
    res = {}
    for name, ins in funcs.items():
        if not any(h in name for h in HOT):
            continue
        last_rcp, stray, dfma = -10**9, 0, 0
        for i, l in enumerate(ins):
            if "MUFU.RCP64H" in l:
                last_rcp = i
            if re.search(r"\bDFMA\b", l):
                dfma += 1
                if i - last_rcp > WINDOW:
                    stray += 1
        res[name] = {"instructions": len(ins), "dfma": dfma, "dfma_outside_division": stray,
                     "dadd": sum(bool(re.search(r"\bDADD\b", l)) for l in ins),
                     "dmul": sum(bool(re.search(r"\bDMUL\b", l)) for l in ins)}
    return res


if __name__ == "__main__":
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2405_18093_b200", "lib", "libpipette.so")
    print(json.dumps(analyse(lib), indent=1))
