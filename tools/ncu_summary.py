"""Summarise an ncu report (read here, on the CPU box) into profiles/.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/<name> [--L .. --N .. --steps-per-launch K]

Writes <name>.json (per-kernel metrics) and <name>.md (table), and, with
--step-kernel, profiles/ncu_step_kernel.json, which bench.py reads for the
roofline `traffic` field (DRAM bytes per launch of the step kernel).
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum",
    "sm__inst_executed.avg.per_cycle_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "sm__cycles_elapsed.avg.per_second",
    "lts__t_bytes.sum",
]
STALLS = "smsp__average_warps_issue_stalled_"


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v) * scale.get(unit, 1)


def to_seconds(v, unit):
    scale = {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
             "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}
    return float(v) * scale.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--L", type=int, default=10**9)
    ap.add_argument("--N", type=int, default=2 * 10**8)
    ap.add_argument("--steps-per-launch", type=int, default=1)
    ap.add_argument("--step-kernel", action="store_true")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = {"value": r[i], "unit": units[i]}
        stalls = {h[len(STALLS):]: float(r[i] or 0) for i, h in enumerate(hdr)
                  if h.startswith(STALLS) and h.endswith("_per_issue_active.ratio")}
        d["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
        rd = d["dram__bytes_read.sum"]
        wr = d["dram__bytes_write.sum"]
        dur = d["gpu__time_duration.sum"]
        d["dram_bytes"] = to_bytes(rd["value"], rd["unit"]) + to_bytes(wr["value"], wr["unit"])
        d["seconds"] = to_seconds(dur["value"], dur["unit"])
        d["dram_gbs"] = d["dram_bytes"] / d["seconds"] / 1e9
        inst = float(d["smsp__inst_executed.sum"]["value"])
        d["thread_inst_per_car_update"] = inst * 32 / (a.N * a.steps_per_launch)
        d["car_updates_per_s"] = a.N * a.steps_per_launch / d["seconds"]
        out.append(d)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out + ".json", "w") as f:
        json.dump({"report": os.path.basename(a.report), "L": a.L, "N": a.N,
                   "steps_per_launch": a.steps_per_launch, "kernels": out}, f, indent=1)
    with open(a.out + ".md", "w") as f:
        f.write(f"# ncu summary: {os.path.basename(a.report)} (L={a.L}, N={a.N}, "
                f"{a.steps_per_launch} steps/launch; ncu --set full --clock-control none, "
                "cold cache, serialised)\n\n")
        f.write("| kernel | time | DRAM bytes | DRAM GB/s | DRAM % peak | issue active % | "
                "thread inst / car-update | car-updates/s | regs |\n|---|---|---|---|---|---|---|---|---|\n")
        for d in out:
            f.write(f"| `{d['kernel'][:60]}` | {d['seconds'] * 1e6:.1f} us | {d['dram_bytes'] / 1e9:.3f} GB | "
                    f"{d['dram_gbs']:.0f} | {d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']['value']} | "
                    f"{d.get('smsp__issue_active.avg.pct_of_peak_sustained_active', {}).get('value', '?')} | "
                    f"{d['thread_inst_per_car_update']:.1f} | {d['car_updates_per_s']:.3e} | "
                    f"{d['launch__registers_per_thread']['value']} |\n")
        f.write("\nTop stall reasons (warps stalled per issued instruction):\n\n")
        for d in out:
            f.write(f"- `{d['kernel'][:60]}`: " + ", ".join(
                f"{k} {v:.2f}" for k, v in d["top_stalls_per_issue"].items()) + "\n")
    if a.step_kernel and out:
        # one capture per launch depth; bench.py picks the one its timed
        # region runs at
        d = out[0]
        path = os.path.join(os.path.dirname(a.out), "ncu_step_kernel.json")
        try:
            with open(path) as f:
                prev = json.load(f)
        except (OSError, ValueError):
            prev = {}
        caps = [c for c in prev.get("captures", []) if prev.get("L") == a.L and prev.get("N") == a.N
                and c.get("steps_per_launch") != a.steps_per_launch]
        caps.append({"steps_per_launch": a.steps_per_launch, "kernel": d["kernel"],
                     "dram_bytes_per_launch": d["dram_bytes"],
                     "warp_inst_per_launch": float(d["smsp__inst_executed.sum"]["value"]),
                     "seconds_per_launch_under_ncu": d["seconds"],
                     "source": os.path.basename(a.out) + ".json"})
        caps.sort(key=lambda c: c["steps_per_launch"])
        with open(path, "w") as f:
            json.dump({"L": a.L, "N": a.N, "captures": caps}, f, indent=1)
    print(open(a.out + ".md").read())


if __name__ == "__main__":
    sys.exit(main())
