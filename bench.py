#!/usr/bin/env python
"""bench.py -- car-updates/s of the B200 NaSch engine (BASELINE.json metric).

Headline workload (config.workload): BASELINE.json config 3, the large
single ring L=1e9 cells, N=2e8 cars (density 0.2), p=0.13, vmax=5, seeded
uniform distinct sorted positions, velocities 0.  A "step" is one
synchronous time step of the whole ring (N car-updates).  With N GPUs the
ring is split into N contiguous car segments, one process per GPU (strong
scaling; the segments exchange one 2 KB halo/cone record per 16-step launch
through peer memory).  A second leg times BASELINE config 4 (4096
independent rings, sharded by ring ranges across the GPUs with no
communication) and reports it under "c4".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--repeats R]
                  [--impl ours|reference]

--gpus N > 1 without torchrun re-launches itself under
torch.distributed.run with N ranks (one per GPU).

value       device throughput, state resident in HBM: N*K / CUDA-event time
            of K steps on the engine's own stream (barrier + synchronize on
            both sides, max over ranks); the median of R passes (the spread
            is in "passes_ms")
e2e         the same metric through the C ABI with host buffers: set_state32
            from pinned host int32 arrays (BASELINE's state format),
            advance(K), the whole-ring mean-velocity series and the final
            state (each rank: its segment) read back to pinned host int32
            arrays (nasch_sim_state_segment32; nasch_sim_state is the same
            call widened to u64), wall clock, max over ranks
roofline    SURVEY.md 8(d): 16 algorithmic bytes per car-update (int32 x and
            v read and written once per step) x N*k updates per launch / the
            average duration of the timed region's k-step launches (k =
            min(K, 32)), from per-launch CUDA events inside the timed region;
            peak = MEASURED_PEAKS.json.  Temporal blocking moves the state
            once per k steps, so frac > 1; the roof that binds is integer
            issue ("issue_bound")
cpu_baseline  the reference's own OpenMP Engine (oracle/_ref, compiled
            unmodified) on this host's cores, bounded step prefix
--impl reference  only that CPU measurement, as its own JSON line (its
            input comes from the oracle's restatement of the generator: the
            product library is never loaded on that arm)
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = dict(L=10**9, N=2 * 10**8, p=0.13, vmax=5, seed=3, T=1000)
WORKLOAD = "C3: single ring L=1e9, N=2e8 (density 0.2), p=0.13, vmax=5, 1000 steps"
C4_WORKLOAD = ("C4: 4096 independent rings L=1e5, N_j = 5000 + floor(45000 j / 63) (j < 64), "
               "p in {0.0..0.7}, 8 seed replicas, vmax=5, 5000 steps")
BYTES_MOVED_PER_UPDATE = 10  # u32 x + u8 v, read once and written once per launch
SURVEY_BYTES_PER_UPDATE = 16  # int32 x and v read+written per step
CPU_SAMPLE_SECONDS = 25.0
MIN_WARMUP_STEPS = 512
CK_STEPS = 10  # the checksum-on leg (C3 with the reference's per-step FNV-1a)
C4_MIN_WARMUP_STEPS = 64
PARITY_RING = dict(L=10**7, N=2 * 10**6, p=0.13, vmax=5, seed=17, steps=48, init_seed=11)


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


def ncu_step_kernel(k_launch):
    """The step kernel's committed ncu capture summary (profiles/) for this
    workload at this launch depth, or {}."""
    path = os.path.join(ROOT, "profiles", "ncu_step_kernel.json")
    try:
        with open(path) as f:
            d = json.load(f)
        if d.get("L") == CONFIG["L"] and d.get("N") == CONFIG["N"]:
            for c in d.get("captures", []):
                if c.get("steps_per_launch") == k_launch:
                    return c
    except Exception:
        pass
    return {}


def issue_bound(launch_ms, spl, n, clocks, world):
    """The roof that binds once temporal blocking removes HBM: integer
    instruction issue.  Warp instructions per launch come from the ncu
    capture (profiles/, one GPU); the peak is 1 warp instruction per cycle
    per SMSP (4 per SM) at the SM clock sampled during the timed region."""
    import torch
    d = ncu_step_kernel(spl)
    if "warp_inst_per_launch" not in d or not torch.cuda.is_available() or world != 1:
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
    `nvidia-smi -lms 50` child process cost 3-10 % of a ~125 ms region and
    added outliers (measured), so the sampling is in-process and sparse;
    `nvidia-smi` remains the fallback when NVML is unavailable."""

    PERIOD_S = 0.1
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = None
        self._thread = None
        self.proc = None
        self.out = ""

    def _nvml_loop(self, nvml, handle):
        bits = [nvml.nvmlClocksEventReasonHwSlowdown, nvml.nvmlClocksEventReasonHwThermalSlowdown,
                nvml.nvmlClocksEventReasonSwThermalSlowdown, nvml.nvmlClocksEventReasonSwPowerCap]
        while True:
            try:
                sm = nvml.nvmlDeviceGetClockInfo(handle, nvml.NVML_CLOCK_SM)
                mx = nvml.nvmlDeviceGetMaxClockInfo(handle, nvml.NVML_CLOCK_SM)
                rs = nvml.nvmlDeviceGetCurrentClocksEventReasons(handle)
                self.rows.append([str(sm), str(mx)] + ["Active" if rs & b else "Not Active" for b in bits])
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

    def __exit__(self, *exc):
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
        reasons = sorted({self.NAMES[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
# the reference arm (CPU): oracle/_ref only, never the product library

def reference_input():
    """C3 input from the oracle's restatement of the seeded generator."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    t0 = time.time()
    x, v = oracle.Port().fill_uniform_state(CONFIG["L"], CONFIG["N"], 0, CONFIG["seed"])
    log(f"[bench] generated C3 input (oracle generator) in {time.time() - t0:.1f}s")
    return x, v


def cpu_reference_sample(x32, v32, steps_cap=None):
    """Times the reference Engine (oracle/_ref) on a bounded prefix of the
    workload with all physical cores.  Returns a cpu_baseline dict."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    ref = oracle.Ref()
    cores = ref.physical_cores() or os.cpu_count() or 1
    L, N = CONFIG["L"], CONFIG["N"]
    x = np.ascontiguousarray(x32, np.uint64)
    v = np.ascontiguousarray(v32, np.uint64)
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
    x, v = reference_input()
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


# ---------------------------------------------------------------------------
# our arm

class Dist:
    """torch.distributed plumbing for N ranks (NCCL); identity at N=1."""

    def __init__(self, rank, world, local_rank):
        import torch
        self.torch = torch
        self.rank, self.world, self.local_rank = rank, world, local_rank
        self.dist = None
        if world > 1:
            import torch.distributed as dist
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
            self.dist = dist

    def barrier(self):
        if self.dist:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if not self.dist:
            return x
        t = self.torch.tensor([x], device="cuda", dtype=self.torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def all_true(self, ok: bool) -> bool:
        if not self.dist:
            return bool(ok)
        t = self.torch.tensor([0 if ok else 1], device="cuda")
        self.dist.all_reduce(t)
        return int(t.item()) == 0

    def bcast(self, obj):
        if not self.dist:
            return obj
        box = [obj]
        self.dist.broadcast_object_list(box, src=0)
        return box[0]

    def gather(self, obj):
        if not self.dist:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def close(self):
        if self.dist:
            self.dist.barrier()
            self.dist.destroy_process_group()


def nccl_init_summary(path):
    """NCCL INIT lines of this rank (NCCL_DEBUG=INFO, SUBSYS=INIT), echoed
    to stderr so the launcher's log shows nRanks; summary for the line."""
    try:
        with open(path) as f:
            lines = [ln.rstrip() for ln in f if ln.strip()]
    except OSError:
        return None
    keep = [ln for ln in lines if "nRanks" in ln or "NCCL version" in ln or "Init COMPLETE" in ln]
    for ln in keep[:40]:
        log("[nccl] " + ln)
    nranks = set()
    for ln in keep:
        parts = ln.split()
        for i, tok in enumerate(parts[:-1]):
            if tok == "nRanks" and parts[i + 1].isdigit():
                nranks.add(int(parts[i + 1]))
    nranks = sorted(nranks)
    return {"init_lines": len(keep), "nranks_seen": nranks, "log": path}


def multi_gpu_parity(d: Dist, nccl_id):
    """Before timing: the distributed engine (one process per GPU, NCCL +
    peer memory) on a 2e6-car ring for 48 steps with the trajectory
    checksum on, against rank 0's single-GPU engine: the checksum (every
    step's full rank-ordered state), the whole-ring velocity-sum and wrap
    series, the collective state gather and every rank's segment snapshot
    must be identical."""
    from paper_2309_14311_b200 import nasch
    P = PARITY_RING
    x, v = nasch.fill_uniform_state(P["L"], P["N"], P["vmax"], P["init_seed"])
    prm = nasch.SimParams(length=P["L"], ncars=P["N"], vmax=P["vmax"], p=P["p"], steps=P["steps"],
                          seed=P["seed"])
    eng = nasch.Engine.distributed(prm, d.rank, d.world, nccl_id)
    eng.set_checksum(True)
    eng.set_state(x, v)
    eng.advance(P["steps"])
    got = dict(checksum=eng.checksum, sumv=eng.sumv_series().tolist(), wraps=eng.wrap_series().tolist(),
               mode=eng.exchange_mode)
    gx, gv = eng.snapshot()
    sx, sv, first = eng.segment_snapshot()
    eng.close()
    ok = True
    ref = None
    if d.rank == 0:
        r = nasch.Engine(prm)
        r.set_checksum(True)
        r.set_state(x, v)
        r.advance(P["steps"])
        rx, rv = r.snapshot()
        ref = dict(checksum=r.checksum, sumv=r.sumv_series().tolist(), wraps=r.wrap_series().tolist(),
                   x=rx, v=rv)
        r.close()
    ref = d.bcast(ref)
    ok = (got["checksum"] == ref["checksum"] and got["sumv"] == ref["sumv"]
          and got["wraps"] == ref["wraps"] and (gx == ref["x"]).all() and (gv == ref["v"]).all())
    ranks = (first + np.arange(len(sx), dtype=np.uint64)) % np.uint64(P["N"])
    ok = ok and bool((sx == ref["x"][ranks]).all() and (sv == ref["v"][ranks]).all())
    return d.all_true(ok), got["mode"]


def c3_leg(args, d: Dist):
    import torch
    from paper_2309_14311_b200 import nasch

    L, N, p, vmax, seed = CONFIG["L"], CONFIG["N"], CONFIG["p"], CONFIG["vmax"], CONFIG["seed"]
    K, W, R = args.steps, args.warmup, args.repeats
    # Untimed warm-up of at least MIN_WARMUP_STEPS: the engine's first
    # launches and the SM clock ramp from idle landed inside the timed
    # region with a handful of warm-up steps (10-35 % outliers, measured).
    W_run = max(W, MIN_WARMUP_STEPS)
    t0 = time.time()
    x, v = nasch.fill_uniform_state(L, N, 0, seed)
    log(f"[bench] generated C3 input in {time.time() - t0:.1f}s")

    def fresh_id():
        # one NCCL unique id per communicator (an id's bootstrap root serves
        # one initialisation; it is not reused for a second communicator)
        return d.bcast(nasch.nccl_unique_id() if d.rank == 0 else None) if d.world > 1 else None

    parity = None
    if d.world > 1 and not args.no_parity:
        t0 = time.time()
        ok, mode = multi_gpu_parity(d, fresh_id())
        parity = {"ok": ok, "ring": PARITY_RING, "exchange_mode": mode,
                  "checks": "trajectory checksum, whole-ring sumv/wrap series, collective state, "
                            "segment snapshots vs rank 0's single-GPU engine",
                  "seconds": round(time.time() - t0, 2)}
        log(f"[bench] multi-GPU parity self-check: {ok} ({parity['seconds']} s)")

    # ---- device-resident throughput -----------------------------------
    prm = nasch.SimParams(length=L, ncars=N, vmax=vmax, p=p, steps=W_run + R * K + 2 + CK_STEPS, seed=seed)
    eng = (nasch.Engine.distributed(prm, d.rank, d.world, fresh_id()) if d.world > 1
           else nasch.Engine(prm))
    eng.set_checksum(False)
    eng.set_state(x, v)
    eng.advance(W_run)
    stream = torch.cuda.ExternalStream(eng.cuda_stream)
    spl = eng.steps_per_launch
    passes, full_launch_ms, launches = [], [], None
    with ClockSampler(d.local_rank) as clk:
        for _ in range(R):
            d.barrier()
            torch.cuda.synchronize()
            l0 = eng.kernel_launches
            ev0 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            marks, done = [], 0
            while done < K:  # one launch per enqueue: per-launch events
                k = min(spl, K - done)
                eng.enqueue(k)
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                marks.append((k, e))
                done += k
            eng.synchronize()
            torch.cuda.synchronize()
            launches = eng.kernel_launches - l0
            prev = ev0
            k_top = max(k for k, _ in marks)  # the launch depth the region runs at
            for k, e in marks:
                if k == k_top:
                    full_launch_ms.append(prev.elapsed_time(e))
                prev = e
            passes.append(d.max(ev0.elapsed_time(marks[-1][1])))
    ms = statistics.median(passes)
    k_launch = min(spl, K)  # steps per launch of the timed region's launches
    launch_ms = d.max(statistics.median(full_launch_ms))
    xmode = {0: "none (one segment)", 1: "collective (NCCL all-gather)",
             2: "peer memory (records stored by the step kernel into the peers' HBM)"}[eng.exchange_mode]
    sumv = eng.sumv_series()  # whole ring on every rank (collective)
    if d.world == 1:
        xs, vs = eng.snapshot()
        ok = bool((np.diff(xs.astype(np.int64)) > 0).all() and int(xs[-1]) < L
                  and int(vs.sum()) == int(sumv[-1]))
        del xs, vs
    else:
        wraps = eng.wrap_series()
        allw = d.gather(hashlib.sha256(wraps.tobytes() + sumv.tobytes()).hexdigest())
        ok = bool(len(sumv) == W_run + R * K and all(w == allw[0] for w in allw)
                  and int(sumv.max()) <= vmax * N)
    ok = d.all_true(ok)
    # The reference's stock semantics on the same engine: the checksum on,
    # every step's rank-ordered row folded into the FNV-1a digest on the
    # device; one GPU (the segmented ring keeps the slower
    # round-1 digest)
    checksum_leg = None
    if d.world == 1:
        eng.set_checksum(True)
        eng.advance(2)  # the digest's buffers and graph, outside the timing
        torch.cuda.synchronize()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        eng.enqueue(CK_STEPS)
        c1.record(stream)
        eng.synchronize()
        torch.cuda.synchronize()
        ck_ms = c0.elapsed_time(c1)
        checksum_leg = {"value": N * CK_STEPS / (ck_ms / 1e3), "unit": "car-updates/s",
                        "ms_per_step": ck_ms / CK_STEPS, "steps": CK_STEPS,
                        "note": "checksum on (nasch_sim_new's default, the reference cannot turn it off): "
                                "one-step kernel + the nibble-decomposed FNV-1a of every step's row on the device"}
    eng.close()
    value = N * K / (ms / 1000.0)  # whole ring, max over ranks
    step_ms = ms / K

    # ---- end to end through the C ABI with host buffers ----------------
    # Input: BASELINE's int32 state in page-locked host memory (a pinned
    # torch tensor viewed as numpy), uploaded by nasch_sim_set_state32 (the
    # positions DMA'd straight from it, validated on the host, velocities
    # narrowed to bytes).  Output: the reference ABI's nasch_sim_state (u64).
    xin = torch.empty(N, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    vin = torch.empty(N, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    xin[:] = x
    vin[:] = v
    del x, v
    prm2 = nasch.SimParams(length=L, ncars=N, vmax=vmax, p=p, steps=K, seed=seed)
    eng2 = (nasch.Engine.distributed(prm2, d.rank, d.world, fresh_id()) if d.world > 1
            else nasch.Engine(prm2))
    first, count = eng2.shard_range()
    # caller-owned output buffers in BASELINE's int32 format, page-locked
    # like the input and already faulted in (a serving loop reuses them)
    outx = torch.zeros(count, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    outv = torch.zeros(count, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    eng2.set_checksum(False)
    eng2.advance(0)
    d.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if d.world == 1:
        # one call: nasch_sim_job32 streams the upload, the steps and the
        # download by ranges of the ring when K fits one K-step launch (the
        # three calls below otherwise, inside the library)
        eng2.job32(xin, vin, K, out_x=outx, out_v=outv)
        t_set = t_adv = time.perf_counter()
        mean_v = eng2.mean_velocity_series()
    else:
        eng2.set_state(xin, vin)  # each rank validates and uploads its own segment
        t_set = time.perf_counter()
        eng2.advance(K)
        t_adv = time.perf_counter()
        mean_v = eng2.mean_velocity_series()  # whole ring (collective)
        eng2.segment_snapshot32(out_x=outx, out_v=outv)
    t1 = time.perf_counter()
    e2e_s = d.max(t1 - t0)
    parts = ({"job32 (set_state + advance + state, streamed)": (t_set - t0) * 1e3, "series": (t1 - t_set) * 1e3}
             if d.world == 1 else
             {"set_state": (t_set - t0) * 1e3, "advance": (t_adv - t_set) * 1e3,
              "series+state": (t1 - t_adv) * 1e3})
    assert len(mean_v) == K
    eng2.close()
    e2e = {"value": N * K / e2e_s, "unit": "car-updates/s",
           "h2d_bytes_per_step": (4 + 1) * N / K,        # u32 x + u8 v per car, all segments
           "d2h_bytes_per_step": ((4 + 1) * N + 8 * K * d.world) / K,  # final state + series
           "breakdown_ms_rank0": {k: round(t, 2) for k, t in parts.items()},
           "path": "N=1: nasch_sim_job32 (set_state32 from BASELINE's int32 state in pinned host arrays + "
                   "advance(K) + final state to pinned host int32 arrays in rank order, upload / steps / "
                   "download streamed by ranges of the ring when K <= 32) + the mean-velocity series; N>1: "
                   "each rank nasch_sim_set_state32 of its segment + nasch_sim_advance(K) + the whole-ring "
                   "series + nasch_sim_state_segment32; wall clock, max over ranks"}

    # ---- roofline --------------------------------------------------------
    peak, peak_src = peaks()
    peak *= d.world  # aggregate over the ranks' HBM
    achieved = SURVEY_BYTES_PER_UPDATE * N * k_launch / (launch_ms / 1000.0) / 1e9
    traffic = ncu_step_kernel(k_launch).get("dram_bytes_per_launch") if d.world == 1 else None
    clocks = clk.summary()
    kernel = (f"nasch_tb_kernel<uint8_t,128,32,32,1> + cone_init_kernel<uint8_t,256> "
              f"({spl} steps per launch)" if d.world == 1
              else f"nasch_tb_push_kernel<uint8_t,128,32,32,1> + shard_plan_kernel ({spl} steps per launch)")
    line = {"metric": "car-updates/s", "value": value, "unit": "car-updates/s",
            "n_gpus": d.world, "steps": K, "warmup": W, "ms_per_step": step_ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u32", "data": "synthetic (seeded uniform distinct sorted positions, v=0)",
            "config": {"workload": WORKLOAD, **CONFIG,
                       "warmup_steps_run": W_run,
                       "timed_steps": f"{R} passes of {K} steps after step {W_run}; value = median pass",
                       "l2": "no flush: 2.0 GB ping-pong state >> 126 MB L2",
                       "checksum": "off (nasch_sim_set_checksum(0); the reference cannot disable it)",
                       "parallelism": "1 GPU" if d.world == 1 else
                                      f"{d.world} ranks, one contiguous car segment each",
                       **({"segment_exchange": xmode} if d.world > 1 else {})},
            "passes_ms": [round(t, 4) for t in passes],
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_update": SURVEY_BYTES_PER_UPDATE,
                         "units_per_launch": N * k_launch, "steps_per_launch": k_launch,
                         "max_steps_per_launch": spl,
                         "kernel_ms_avg": launch_ms,
                         "kernel_ms_source": f"median of {len(full_launch_ms)} {k_launch}-step launches "
                                             "(CUDA events between launches on the engine stream; "
                                             "step kernel + next-launch plan kernel), max over ranks",
                         "peak_source": peak_src, "kernel": kernel,
                         "state_bytes_moved_per_launch": BYTES_MOVED_PER_UPDATE * N,
                         "state_gbs_moved": BYTES_MOVED_PER_UPDATE * N / (launch_ms / 1000.0) / 1e9,
                         "note": "temporal blocking: the state crosses HBM once per "
                                 f"{k_launch} steps, so frac > 1 vs the per-step roofline; "
                                 "the binding roof is integer issue (issue_bound, DESIGN.md 4.1)"},
            "issue_bound": issue_bound(launch_ms, k_launch, N, clocks, d.world),
            "e2e": e2e,
            **({"checksum_on": checksum_leg} if checksum_leg else {}),
            "gpu_launches": int(launches),
            "clocks": clocks,
            "invariants_ok": ok}
    if parity is not None:
        line["multi_gpu_parity_ok"] = parity["ok"]
        line["multi_gpu_parity"] = parity
    if d.rank == 0 and d.world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_reference_sample(xin, vin)
    return line


def c4_specs():
    """BASELINE config 4: (N, p, seed) of the 4096 rings."""
    dens = [5000 + (45000 * j) // 63 for j in range(64)]
    ps = [0.0, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7]
    return [(N, p, 1 + rep * 1000 + pi * 100 + j)
            for rep in range(8) for pi, p in enumerate(ps) for j, N in enumerate(dens)]


def c4_leg(args, d: Dist):
    """The ensemble: contiguous ring ranges per rank balanced by cars,
    no communication while stepping, one gather of the per-ring flux totals."""
    import torch
    from paper_2309_14311_b200 import nasch

    L = 10**5
    specs = c4_specs()
    total_cars = sum(s[0] for s in specs)
    lo, hi = nasch.partition_rings([s[0] for s in specs], d.world)[d.rank]
    mine = specs[lo:hi]
    K, R = args.steps, args.repeats
    W_run = max(args.warmup, C4_MIN_WARMUP_STEPS)
    t0 = time.time()
    xs, vs = [], []
    for N, _, sd in mine:
        x, v = nasch.fill_uniform_state(L, N, 0, sd)
        xs.append(x)
        vs.append(v)
    # BASELINE's int32 state in page-locked host memory (as the C3 leg): the
    # positions go up in one DMA, scattered into the rings' layout on the device
    ncar = sum(len(a) for a in xs)
    xc = torch.empty(ncar, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    vc = torch.empty(ncar, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    xc[:] = np.concatenate(xs)
    vc[:] = np.concatenate(vs)
    del xs, vs
    log(f"[bench] C4 input ({hi - lo} rings on rank {d.rank}) in {time.time() - t0:.1f}s")

    def make(steps):
        return nasch.Ensemble([nasch.SimParams(length=L, ncars=N, vmax=5, p=p, steps=steps, seed=sd)
                               for N, p, sd in mine])

    ens = make(W_run + R * K)
    ens.set_state_all(xc, vc)
    ens.advance(W_run)
    stream = torch.cuda.ExternalStream(ens.cuda_stream)
    passes = []
    for _ in range(R):
        d.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = ens.kernel_launches
        e0.record(stream)
        ens.enqueue(K)
        e1.record(stream)
        ens.synchronize()
        torch.cuda.synchronize()
        launches = ens.kernel_launches - l0
        passes.append(d.max(e0.elapsed_time(e1)))
    ms = statistics.median(passes)
    ens.close()

    # e2e: host u32 state in (all rings in one call), K steps, per-ring flux
    # totals out
    ens2 = make(K)
    d.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ens2.set_state_all(xc, vc)
    ens2.advance(K)
    totals = ens2.sumv_totals()
    e2e_s = d.max(time.perf_counter() - t0)
    ens2.close()
    parts = d.gather((lo, totals.tolist()))
    allt = np.array([t for _, tot in sorted(parts) for t in tot], dtype=np.uint64)
    value = total_cars * K / (ms / 1e3)
    peak, _ = peaks()
    return {"workload": C4_WORKLOAD, "rings": len(specs), "total_cars": total_cars,
            "rings_on_rank0": hi - lo if d.rank == 0 else None,
            "value": value, "unit": "car-updates/s", "ms_per_step": ms / K, "steps": K,
            "warmup_steps_run": W_run, "passes_ms": [round(t, 4) for t in passes],
            "scaling": "strong (4096 rings split across the ranks)",
            "roofline_frac": value * SURVEY_BYTES_PER_UPDATE / (peak * d.world * 1e9),
            "gpu_launches": int(launches),
            "e2e": {"value": total_cars * K / e2e_s, "unit": "car-updates/s",
                    "h2d_bytes_per_step": 5 * total_cars / K, "d2h_bytes_per_step": 8 * len(specs) / K,
                    "path": "nasch_ensemble_set_state_all32 (int32 state in pinned host arrays) + "
                            "nasch_ensemble_advance(K) + nasch_ensemble_sumv_totals, wall clock, max over ranks"},
            "flux_totals_sha256": hashlib.sha256(allt.tobytes()).hexdigest(),
            "note": "flux totals after K steps: identical for every GPU count"}


def run_ours(args, rank, world, local_rank):
    import torch
    torch.cuda.set_device(local_rank)
    nccl_log = None
    if world > 1 and "NCCL_DEBUG" not in os.environ:
        # INIT lines go to a per-rank file (NCCL writes them to stdout by
        # default, which would break the one-JSON-line contract); rank 0
        # echoes its own to stderr
        nccl_log = f"/tmp/nasch_bench_nccl.{os.getpid()}.log"
        os.environ.update(NCCL_DEBUG="INFO", NCCL_DEBUG_SUBSYS="INIT", NCCL_DEBUG_FILE=nccl_log)
    d = Dist(rank, world, local_rank)
    line = c3_leg(args, d)
    if not args.no_c4:
        line["c4"] = c4_leg(args, d)
    if nccl_log and rank == 0:
        line["nccl"] = nccl_init_summary(nccl_log)
    assert line["n_gpus"] == args.gpus, (line["n_gpus"], args.gpus)
    if rank == 0:
        print(json.dumps(line), flush=True)
    d.close()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn(args):
    """--gpus N > 1 outside torchrun: re-launch under torch.distributed.run,
    one rank per GPU, and pass its exit code through."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    log("[bench] " + " ".join(cmd))
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--repeats", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c4", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"[bench] --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
        sys.exit(2)
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
