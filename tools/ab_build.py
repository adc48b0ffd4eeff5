"""Build libpipette.so of another git revision into lib/ab/libpipette_<rev>.so (A/B timing
on one box: PIPETTE_LIB=<path> python tools/search_probe.py C2)."""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rev = sys.argv[1]
wt = f"/tmp/pipette_ab_{rev}"
if os.path.exists(wt):
    subprocess.call(["git", "-C", ROOT, "worktree", "remove", "--force", wt])
subprocess.check_call(["git", "-C", ROOT, "worktree", "add", "--detach", wt, rev])
subprocess.check_call([sys.executable, "-m", "paper_2405_18093_b200.build", "--force"], cwd=wt)
dst = os.path.join(ROOT, "paper_2405_18093_b200", "lib", "ab")
os.makedirs(dst, exist_ok=True)
out = os.path.join(dst, f"libpipette_{rev}.so")
shutil.copy(os.path.join(wt, "paper_2405_18093_b200", "lib", "libpipette.so"), out)
subprocess.call(["git", "-C", ROOT, "worktree", "remove", "--force", wt])
print(out)
