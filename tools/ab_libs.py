"""Interleaved A/B of library builds on the box: python tools/ab_libs.py C3,C5 base=,nofrel=vlibs/libnasch_nofrel.so [reps]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from waves_sweep import CHILD  # noqa: E402

cfgs = sys.argv[1].split(",")
libs = [kv.split("=") for kv in sys.argv[2].split(",")]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
for rep in range(reps):
    for cfg in cfgs:
        for name, path in libs:
            env = dict(os.environ, R=ROOT)
            if path:
                env["NASCH_B200_LIB"] = os.path.join(ROOT, path)
            p = subprocess.run([sys.executable, "-c", CHILD, cfg], env=env, capture_output=True, text=True)
            out = p.stdout.strip().splitlines()
            print(name, out[-1] if out else p.stderr[-300:], flush=True)
