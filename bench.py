#!/usr/bin/env python
"""bench.py -- car-updates/s of the B200 NaSch engine (BASELINE.json metric).

Workload (config.workload): BASELINE.json config 3, the large single ring
L=1e9 cells, N=2e8 cars (density 0.2), p=0.13, vmax=5, int32 positions,
seeded uniform distinct sorted positions, velocities 0.  A "step" is one
synchronous time step of the whole ring (N car-updates).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

value     device throughput, state resident in HBM, CUDA events on the
          engine's own stream around K steps (barrier + synchronize on both
          sides, max over ranks)
e2e       the same metric through the C ABI with host buffers: set_state
          from host u64 arrays, advance(K), per-step velocity-sum series and
          final state read back to host u64 arrays, wall clock
roofline  HBM-bound: 10 algorithmic bytes per car-update (u32 x and u8 v,
          each read and written once) / average step-kernel duration vs the
          measured copy bandwidth in MEASURED_PEAKS.json
cpu_baseline  the reference's own OpenMP Engine (oracle/_ref, compiled
          unmodified) on this host's cores, bounded step prefix
--impl reference  only that CPU measurement, as its own JSON line
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = dict(L=10**9, N=2 * 10**8, p=0.13, vmax=5, seed=3, T=1000)
WORKLOAD = "C3: single ring L=1e9, N=2e8 (density 0.2), p=0.13, vmax=5, 1000 steps"
BYTES_PER_UPDATE = 10  # u32 x + u8 v, read once and written once per launch
SURVEY_BYTES_PER_UPDATE = 16  # int32 x and v read+written per step
CPU_SAMPLE_SECONDS = 25.0
MIN_WARMUP_STEPS = 512


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_step_kernel():
    """The step kernel's committed ncu capture summary (profiles/) for this
    workload, or {}."""
    path = os.path.join(ROOT, "profiles", "ncu_step_kernel.json")
    try:
        with open(path) as f:
            d = json.load(f)
        if d.get("L") == CONFIG["L"] and d.get("N") == CONFIG["N"]:
            return d
    except Exception:
        pass
    return {}


def ncu_traffic():
    """Per-launch DRAM bytes of the step kernel (ncu), or None."""
    d = ncu_step_kernel()
    return float(d["dram_bytes_per_launch"]) if "dram_bytes_per_launch" in d else None


def issue_bound(launch_ms, spl, n, clocks):
    """The roof that binds once temporal blocking removes HBM: integer
    instruction issue.  Warp instructions per launch come from the ncu
    capture (profiles/); the peak is 1 warp instruction per cycle per SMSP
    (4 per SM) at the SM clock sampled during the timed region."""
    import torch
    d = ncu_step_kernel()
    if "warp_inst_per_launch" not in d or not torch.cuda.is_available():
        return None
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    mhz = clocks.get("sm_mhz") or 1965.0
    peak = sms * 4 * mhz * 1e6
    inst = d["warp_inst_per_launch"]
    achieved = inst / (launch_ms / 1e3)
    return {"unit": "warp-inst/s", "achieved": achieved, "peak": peak, "frac": achieved / peak,
            "warp_inst_per_launch": inst, "thread_inst_per_update": inst * 32 / (n * spl),
            "source": "ncu smsp__inst_executed.sum (" + d.get("source", "") + ") / live launch time"}


class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region, from a
    thread calling NVML every 100 ms (first sample at once).  An
    `nvidia-smi -lms 50` child process cost 3-10 % of this ~125 ms region
    and added outliers (measured), so the sampling is in-process and sparse;
    `nvidia-smi` remains the fallback when NVML is unavailable."""

    PERIOD_S = 0.1

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = None
        self._thread = None
        self.proc = None

    def _nvml_loop(self, nvml, handle):
        names = [("hw_slowdown", nvml.nvmlClocksEventReasonHwSlowdown),
                 ("hw_thermal_slowdown", nvml.nvmlClocksEventReasonHwThermalSlowdown),
                 ("sw_thermal_slowdown", nvml.nvmlClocksEventReasonSwThermalSlowdown),
                 ("sw_power_cap", nvml.nvmlClocksEventReasonSwPowerCap)]
        while True:
            try:
                sm = nvml.nvmlDeviceGetClockInfo(handle, nvml.NVML_CLOCK_SM)
                mx = nvml.nvmlDeviceGetMaxClockInfo(handle, nvml.NVML_CLOCK_SM)
                rs = nvml.nvmlDeviceGetCurrentClocksEventReasons(handle)
                self.rows.append([str(sm), str(mx)] + ["Active" if rs & bit else "Not Active" for _, bit in names])
            except Exception:
                pass
            if self._stop.wait(self.PERIOD_S):
                return

    def __enter__(self):
        if os.environ.get("NASCH_BENCH_NO_SMI"):  # diagnostics only
            return self
        try:
            import threading
            import pynvml as nvml
            nvml.nvmlInit()
            handle = nvml.nvmlDeviceGetHandleByIndex(self.index)
            self._stop = threading.Event()
            self._thread = threading.Thread(target=self._nvml_loop, args=(nvml, handle), daemon=True)
            self._thread.start()
            return self
        except Exception:
            self._thread = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(1.0)  # let nvidia-smi finish its own start-up first
        except Exception:
            self.proc = None
        return self

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __exit__(self, *exc):
        self.out = ""
        if self._thread:
            self._stop.set()
            self._thread.join(timeout=5)
            self.out = "\n".join(", ".join(r) for r in self.rows)
        if self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [s.strip() for s in line.split(",")]
            if len(parts) == 6:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


def make_input():
    from paper_2309_14311_b200 import nasch
    t0 = time.time()
    x, v = nasch.fill_uniform_state(CONFIG["L"], CONFIG["N"], 0, CONFIG["seed"])
    log(f"[bench] generated C3 input in {time.time() - t0:.1f}s")
    return x, v


def cpu_reference_sample(x32, v32, steps_cap=None):
    """Times the reference Engine (oracle/_ref) on a bounded prefix of the
    workload with all physical cores.  Returns a cpu_baseline dict."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    ref = oracle.Ref()
    cores = ref.physical_cores() or os.cpu_count() or 1
    L, N = CONFIG["L"], CONFIG["N"]
    x = x32.astype(np.uint64)
    v = v32.astype(np.uint64)
    # one step to size the sample, then a ~CPU_SAMPLE_SECONDS prefix
    probe = ref.run(L, N, CONFIG["vmax"], CONFIG["p"], CONFIG["seed"], 1, workers=cores,
                    x0=x, v0=v, per_step=False, want_state=False)
    per_step = max(probe["seconds"], 1e-6)
    k = max(1, min(int(CPU_SAMPLE_SECONDS / per_step), 50))
    if steps_cap:
        k = max(1, min(k, steps_cap))
    r = ref.run(L, N, CONFIG["vmax"], CONFIG["p"], CONFIG["seed"], k, workers=cores,
                x0=x, v0=v, per_step=False, want_state=False)
    value = N * k / r["seconds"]
    return {"value": value, "unit": "car-updates/s", "cores": cores, "kind": "reference",
            "sample": f"first {k} steps of the C3 workload from the same initial state, "
                      f"reference Engine (oracle/_ref, unmodified sources, g++ -O3 -fopenmp), "
                      f"{cores} OpenMP workers, advance() timed as `nasch bench` does; "
                      f"includes the reference's mandatory serial per-step FNV checksum",
            "seconds": r["seconds"], "steps": k}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    x, v = make_input()
    cb = cpu_reference_sample(x, v)
    line = {"metric": "car-updates/s", "value": cb["value"], "unit": "car-updates/s",
            "n_gpus": 0 if world == 1 else world, "steps": cb["steps"], "warmup": 1,
            "ms_per_step": 1000.0 * cb["seconds"] / cb["steps"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": WORKLOAD, **CONFIG}, "impl": "reference",
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "car-updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import torch
    from paper_2309_14311_b200 import nasch

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    L, N, p, vmax, seed = CONFIG["L"], CONFIG["N"], CONFIG["p"], CONFIG["vmax"], CONFIG["seed"]
    K, W = args.steps, args.warmup
    # Untimed warm-up of at least MIN_WARMUP_STEPS: the engine captures its
    # launch graph on the first full chunk (256 steps) and the SM clock
    # ramps from idle; with a handful of warm-up steps both landed inside
    # the timed region and gave 10-35 % outliers (measured).
    W_run = max(W, MIN_WARMUP_STEPS)
    x, v = make_input()

    # ---- device-resident throughput -----------------------------------
    prm = nasch.SimParams(length=L, ncars=N, vmax=vmax, p=p, steps=W_run + K, seed=seed)
    if world > 1:
        # one ring, G contiguous segments; the halo + cone-window records
        # are stored into the peer GPUs' HBM by the step kernel once per
        # K-step launch (NCCL all-gather as fallback; DESIGN.md sections 4.6, 6)
        box = [nasch.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        nccl_id = box[0]
        eng = nasch.Engine.distributed(prm, rank, world, nccl_id)
    else:
        eng = nasch.Engine(prm)
    eng.set_checksum(False)
    eng.set_state(x, v)
    eng.advance(W_run)
    stream = torch.cuda.ExternalStream(eng.cuda_stream)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = eng.kernel_launches
    xmode = {0: "none (one segment)", 1: "collective (NCCL all-gather)",
             2: "peer memory (records stored by the step kernel into the peers' HBM)"}[eng.exchange_mode]
    with ClockSampler(local_rank) as clk:
        ev0.record(stream)
        eng.enqueue(K)
        ev1.record(stream)
        eng.synchronize()
        torch.cuda.synchronize()
    launches = eng.kernel_launches - launches0
    spl = eng.steps_per_launch
    kernel_name = (f"nasch_tb_kernel<uint8_t,128,16,16> ({spl} steps per launch)" if spl > 1
                   else "nasch_step_kernel<uint8_t,256,8> (1 step per launch)")
    ms = ev0.elapsed_time(ev1)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    sumv = eng.sumv_series()
    if world == 1:
        xs, vs = eng.snapshot()
        ok = bool((np.diff(xs.astype(np.int64)) > 0).all() and int(xs[-1]) < L
                  and int(vs.sum()) == int(sumv[-1]))
        del xs, vs
    else:
        # whole-ring velocity sums = sum of the ranks' partial series; the
        # wrap series (from the shared plan) must agree on every rank
        tot = torch.tensor(sumv.astype(np.int64), device="cuda")
        dist.all_reduce(tot)
        wraps = eng.wrap_series()
        allw = [None] * world
        dist.all_gather_object(allw, wraps.tolist())
        ok = bool(len(sumv) == W_run + K and all(w == allw[0] for w in allw)
                  and int(tot.max().item()) <= vmax * N)
    eng.close()
    value = N * K / (ms / 1000.0)  # whole ring, max over ranks
    step_ms = ms / K

    # ---- end to end through the C ABI with host buffers ----------------
    x64 = x.astype(np.uint64)
    v64 = v.astype(np.uint64)
    prm2 = nasch.SimParams(length=L, ncars=N, vmax=vmax, p=p, steps=K, seed=seed)
    if world > 1:
        eng2 = nasch.Engine.distributed(prm2, rank, world, nccl_id)
        dist.barrier()
    else:
        # caller-owned output buffers, already faulted in (a serving loop
        # reuses them; first-touch page faults are not the engine's cost)
        outx = np.empty(N, np.uint64)
        outv = np.empty(N, np.uint64)
        outx.fill(0)
        outv.fill(0)
        eng2 = nasch.Engine(prm2)
    eng2.set_checksum(False)
    eng2.advance(0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng2.set_state(x64, v64)
    t_set = time.perf_counter()
    eng2.advance(K)
    t_adv = time.perf_counter()
    series = eng2.sumv_series()
    if world > 1:  # per-step result: whole-ring mean velocity on every rank
        st = torch.tensor(series.astype(np.int64), device="cuda")
        dist.all_reduce(st)
        mean_v = st.cpu().numpy().astype(np.float64) / N
    else:
        mean_v = eng2.mean_velocity_series()
        eng2.snapshot(out_x=outx, out_v=outv)
    t1 = time.perf_counter()
    e2e_s = t1 - t0
    e2e_parts = {"set_state": (t_set - t0) * 1e3, "advance": (t_adv - t_set) * 1e3,
                 "series+state": (t1 - t_adv) * 1e3}
    if dist:
        tt = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    e2e_value = N * K / e2e_s
    e2e_h2d = (4 + 1) * N / K
    e2e_d2h = ((5 * N if world == 1 else 0) + 8 * K * world) / K  # final state + Σv series
    assert len(mean_v) == K
    eng2.close()

    # ---- roofline --------------------------------------------------------
    # 16 algorithmic bytes per car-update (int32 x
    # and v, each read and written once per step); one launch processes
    # N * spl car-updates.  The engine actually moves 10 B per car per launch
    # (u8 velocities) and, temporally blocked, once per spl steps.
    peak, peak_src = peaks()
    peak *= world  # aggregate over the ranks' HBM
    launch_ms = step_ms * spl
    achieved = SURVEY_BYTES_PER_UPDATE * N * spl / (launch_ms / 1000.0) / 1e9
    traffic = ncu_traffic()
    moved_gbs = BYTES_PER_UPDATE * N / (launch_ms / 1000.0) / 1e9

    line = {"metric": "car-updates/s", "value": value, "unit": "car-updates/s",
            "n_gpus": world, "steps": K, "warmup": W, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic (seeded uniform distinct sorted positions, v=0)",
            "config": {"workload": WORKLOAD, **CONFIG,
                       "warmup_steps_run": W_run,
                       "timed_steps": f"steps {W_run}..{W_run + K - 1} of the run",
                       "l2": "no flush: 2.0 GB ping-pong state >> 126 MB L2",
                       "checksum": "off (nasch_sim_set_checksum(0); the reference cannot disable it)",
                       "parallelism": "1 GPU" if world == 1 else f"{world} ranks",
                       **({"segment_exchange": xmode} if world > 1 else {})},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_update": SURVEY_BYTES_PER_UPDATE,
                         "units_per_launch": N * spl, "steps_per_launch": spl,
                         "kernel_ms_avg": launch_ms, "peak_source": peak_src,
                         "kernel": kernel_name,
                         "state_bytes_moved_per_launch": BYTES_PER_UPDATE * N,
                         "state_gbs_moved": moved_gbs,
                         "note": "temporal blocking: the state crosses HBM once per "
                                 f"{spl} steps, so frac > 1 vs the per-step roofline; "
                                 "the kernel is integer-issue bound (DESIGN.md 4.1)"},
            "issue_bound": issue_bound(launch_ms, spl, N, clk.summary()),
            "e2e": {"value": e2e_value, "unit": "car-updates/s", "h2d_bytes_per_step": e2e_h2d,
                    "d2h_bytes_per_step": e2e_d2h,
                    "breakdown_ms_rank0": {k: round(v, 2) for k, v in e2e_parts.items()},
                    "path": "nasch_sim_set_state(u64 host) + nasch_sim_advance(K) + "
                            "mean-velocity series + nasch_sim_state(u64 host), wall clock"},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "invariants_ok": ok}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_reference_sample(x, v)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
