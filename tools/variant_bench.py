"""Interleaved A/B timing of experimental library builds
(tools/build_variant.sh), one child process per run.

  python tools/variant_bench.py --libs base,wide --configs C3 --reps 2
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from waves_sweep import CHILD  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--libs", default="base")
    ap.add_argument("--configs", default="C3")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    res = {}
    for rep in range(a.reps):
        for cfg in a.configs.split(","):
            for lib in a.libs.split(","):
                path = os.path.join(ROOT, "variants", f"libnasch_{lib}.so")
                env = dict(os.environ, R=ROOT, NASCH_B200_LIB=path)
                p = subprocess.run([sys.executable, "-c", CHILD, cfg], env=env, capture_output=True, text=True)
                out = p.stdout.strip().splitlines()
                if not out or not out[-1].startswith("{"):
                    print(lib, cfg, "ERROR", p.stderr[-300:], flush=True)
                    continue
                r = json.loads(out[-1])
                res.setdefault((cfg, lib), []).append(r["car_updates_per_s"])
                print(json.dumps({"rep": rep, "config": cfg, "lib": lib, "cu_s": r["car_updates_per_s"]}), flush=True)
    for (cfg, lib), v in res.items():
        print(f"{cfg} {lib}: best {max(v):.4e} mean {sum(v)/len(v):.4e}")


if __name__ == "__main__":
    main()
