"""Diagnostic (with the GSR_COUNT_EVAL variant builds): forward work units on one view."""
import os
import subprocess
import sys

for k, what in ((1, "(key, block) evaluations"), (2, "keys visited"), (3, "(key, block) with >= 1 composited pixel")):
    out = subprocess.run([sys.executable, "tools/mask_stats.py", sys.argv[1] if len(sys.argv) > 1 else "scannetpp"],
                         env={**os.environ, "GSR_LIB": f"libgsr_ce{k}.so"}, capture_output=True, text=True).stdout
    line = [l for l in out.splitlines() if "blended=" in l][0]
    print(what, line.split("blended=")[1].split()[0])
