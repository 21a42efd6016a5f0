"""Throughput against the temporal-blocked grid size (NASCH_B200_WAVES:
blocks = waves x resident blocks), one child process per setting.

  python tools/waves_sweep.py [--configs C3,C5,C4] [--waves 1,2,4,10] [--out ...]

C3: the bench workload (512 steps); C5: L=1e8, N=6e7, p=0.5 (2000 steps, no
snapshots); C4: the 4096-ring ensemble (1000 steps).  CUDA-event times on
the engine stream (tools/bench_configs.py)."""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import json, os, sys
sys.path.insert(0, os.path.join(os.environ["R"], "tools"))
import bench_configs as bc
name = sys.argv[1]
if name == "C1":
    r = bc.ring("C1", 1000, 200, 0.13, 1000, 42, 0)
elif name == "C2":
    r = bc.ring("C2", 10**6, 2 * 10**5, 0.25, 10**4, 2, 5)
elif name == "C3":
    r = bc.ring("C3", 10**9, 2 * 10**8, 0.13, 512, 3, 0)
elif name == "C5":
    r = bc.ring("C5", 10**8, 6 * 10**7, 0.5, 2000, 5, 0)
else:
    r = bc.c4(T=1000)
print(json.dumps({"config": name, "car_updates_per_s": r["gpu_car_updates_per_s"],
                  "seconds": r["gpu_seconds"]}))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C3,C5,C4")
    ap.add_argument("--waves", default="1,2,4,6,10,16")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    rows = []
    for cfg in a.configs.split(","):
        for w in a.waves.split(","):
            env = dict(os.environ, R=ROOT, NASCH_B200_WAVES=w)
            p = subprocess.run([sys.executable, "-c", CHILD, cfg], env=env, capture_output=True, text=True)
            line = p.stdout.strip().splitlines()[-1] if p.stdout.strip() else ""
            row = json.loads(line) if line.startswith("{") else {"config": cfg, "error": p.stderr[-400:]}
            row["waves"] = int(w)
            rows.append(row)
            print(json.dumps(row), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"gpu": "1 B200", "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
