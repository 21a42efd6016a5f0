import os, sys, json, subprocess
ROOT = os.environ.get("GRAFT_REPO_ROOT", "/root/repo")
code = r'''
import os, sys, json
sys.path.insert(0, os.environ["R"])
sys.path.insert(0, os.path.join(os.environ["R"], "tools"))
from bench_configs import ring
r = ring("C3", 10**9, 2*10**8, 0.13, 512, 3, 0)
print(json.dumps({"grid": os.environ.get("NASCH_B200_GRID", "default"), "cu_s": r["gpu_car_updates_per_s"], "sec": r["gpu_seconds"]}))
'''
for g in sys.argv[1:]:
    env = dict(os.environ, R=ROOT)
    if g != "default":
        env["NASCH_B200_GRID"] = g
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(out.stdout.strip() or out.stderr[-500:], flush=True)
