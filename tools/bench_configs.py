"""Throughput on every BASELINE.json configuration (1 GPU), next to the
reference's own OpenMP Engine on a bounded sample of the same workload.

  python tools/bench_configs.py [--only C1,C4] [--out profiles/r02_configs.json]

C1  L=1e3,  N=200,   p=0.13, 1000 steps, 200 uniform sites from seed 42, v=0
C2  L=1e6,  N=2e5,   p=0.25, 1e4 steps, v uniform in [0,5]
C3  L=1e9,  N=2e8,   p=0.13, 1000 steps (bench.py's headline workload)
C4  4096 rings L=1e5, N_j = 5000 + floor(45000 j/63), p in {0,..,0.7}, 8 seeds,
    5000 steps; time-averaged flux per ring
C5  L=1e8,  N=6e7,   p=0.5, 2e4 steps, full snapshot every 1000 steps

GPU times are CUDA-event times on the engine stream with the state resident
(snapshots included for C5); checksum off, except the C3-checksum /
C5-checksum rows: the reference's stock semantics, every step's row folded
into the FNV-1a trajectory digest on the device.  C5 runs at the k = 8
BASELINE names and at the engine's default depth.  Every run also checks a
size-independent invariant (sorted positions, exact velocity-sum identity).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import torch  # noqa: E402

from paper_2309_14311_b200 import nasch  # noqa: E402


def ev_time(stream, fn):
    s = torch.cuda.ExternalStream(stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3


def ring(name, L, N, p, T, seed, vinit, snapshot_every=0, cpu_steps=0, ref=None, cores=1, k=None,
         checksum=False):
    if k:
        os.environ["NASCH_B200_K"] = str(k)
    else:
        os.environ.pop("NASCH_B200_K", None)
    x, v = nasch.fill_uniform_state(L, N, vinit, seed)
    # untimed warm-up as bench.py: >= 512 steps (launch-graph capture on the
    # first chunk, SM clock ramp from idle), capped at T for the small rings
    warm = max(8, min(512, T)) if not checksum else 2
    prm = nasch.SimParams(length=L, ncars=N, vmax=5, p=p, steps=T + warm, seed=seed)
    e = nasch.Engine(prm)
    e.set_checksum(checksum)
    e.set_state(x, v)
    e.advance(warm)
    snaps = []
    if snapshot_every:
        # double-buffered snapshots: snapshot i is copied on the device and
        # widened on the host while the next advance runs
        bufs = [(np.empty(N, np.uint64), np.empty(N, np.uint64)) for _ in range(2)]
        for bx, bv in bufs:  # fault the pages in outside the timed region
            bx.fill(0)
            bv.fill(0)
        e.snapshot_async(*bufs[1])  # allocates the staging buffers once
        e.snapshot_wait()

        def body():
            done, i = 0, 0
            while done < T:
                k = min(snapshot_every, T - done)
                e.advance(k)
                if i:
                    e.snapshot_wait()
                    snaps.append(int(bufs[(i - 1) % 2][0][-1]))
                e.snapshot_async(*bufs[i % 2])
                i += 1
                done += k
            e.snapshot_wait()
            snaps.append(int(bufs[(i - 1) % 2][0][-1]))
    else:
        def body():
            e.enqueue(T)
            e.synchronize()
    secs = ev_time(e.cuda_stream, body)
    xs, vs = e.snapshot()
    s = e.sumv_series()
    ok = bool((np.diff(xs.astype(np.int64)) > 0).all() and int(vs.sum()) == int(s[-1]))
    out = {"config": name, "L": L, "N": N, "p": p, "steps": T, "gpu_seconds": secs,
           "gpu_car_updates_per_s": N * T / secs, "steps_per_launch": 1 if checksum else e.steps_per_launch,
           "checksum": "on (every step folded on the device)" if checksum else "off",
           "mean_velocity_last": float(s[-1]) / N, "invariants_ok": ok,
           "snapshots": len(snaps)}
    e.close()
    os.environ.pop("NASCH_B200_K", None)
    if ref is not None and cpu_steps:
        r = ref.run(L, N, 5, p, seed, cpu_steps, workers=cores, x0=x.astype(np.uint64),
                    v0=v.astype(np.uint64), per_step=False, want_state=False)
        out["cpu_reference"] = {"steps": cpu_steps, "workers": cores, "seconds": r["seconds"],
                                "car_updates_per_s": N * cpu_steps / r["seconds"]}
        out["speedup_vs_cpu_reference"] = out["gpu_car_updates_per_s"] / out["cpu_reference"]["car_updates_per_s"]
    return out


def _digest(a):
    """Order-sensitive digest of a u64 array (multiply by odd constants that
    depend on the index, sum mod 2^64)."""
    idx = np.arange(len(a), dtype=np.uint64)
    return int(((a + idx) * np.uint64(0x9E3779B97F4A7C15)).sum(dtype=np.uint64))


def c5_segments(G=4, T=20000, every=1000):
    """C5 as G contiguous car segments on this GPU (the segmented engine,
    in-process peer-memory exchange) with a snapshot every `every` steps,
    each snapshot compared (digest of positions and velocities) with the
    single-GPU engine's at the same step."""
    L, N, p, seed = 10**8, 6 * 10**7, 0.5, 5
    x, v = nasch.fill_uniform_state(L, N, 0, seed)
    prm = nasch.SimParams(length=L, ncars=N, vmax=5, p=p, steps=T, seed=seed)
    ref = nasch.Engine(prm)
    ref.set_checksum(False)
    ref.set_state(x, v)
    want = []
    for _ in range(T // every):
        ref.advance(every)
        xs, vs = ref.snapshot()
        want.append((_digest(xs), _digest(vs)))
    ref.close()
    e = nasch.Engine(prm, G, nasch.Engine.CUDA)
    e.set_checksum(False)
    e.set_state(x, v)
    ok = True
    secs = 0.0
    for i in range(T // every):
        secs += ev_time(e.cuda_stream, lambda: e.advance(every))
        xs, vs, first = e.segment_snapshot()
        ok = ok and first == 0 and (_digest(xs), _digest(vs)) == want[i]
    out = {"config": f"C5 ({G} segments, one GPU)", "L": L, "N": N, "p": p, "steps": T,
           "segments": G, "exchange_mode": e.exchange_mode, "snapshots": T // every,
           "snapshots_equal_single_gpu": ok, "gpu_seconds_stepping": secs,
           "gpu_car_updates_per_s": N * T / secs}
    e.close()
    return out


def c4(ref=None, cores=1, T=5000):
    L = 10**5
    dens = [5000 + (45000 * j) // 63 for j in range(64)]
    ps = [0.0, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7]
    specs = []
    for rep in range(8):
        for pi, p in enumerate(ps):
            for j, N in enumerate(dens):
                specs.append((N, p, 1 + rep * 1000 + pi * 100 + j))
    params = [nasch.SimParams(length=L, ncars=N, vmax=5, p=p, steps=T, seed=sd) for N, p, sd in specs]
    t0 = time.time()
    ens = nasch.Ensemble(params)
    inits = []
    for r, (N, p, sd) in enumerate(specs):
        inits.append(nasch.fill_uniform_state(L, N, 0, sd))
    ens.set_state_all(np.concatenate([x for x, _ in inits]), np.concatenate([v for _, v in inits]))
    inits = inits[:64]
    ens.advance(64)  # warm-up, as bench.py's C4 leg
    T -= 64
    setup = time.time() - t0
    secs = ev_time(ens.cuda_stream, lambda: (ens.enqueue(T), ens.synchronize()))
    T += 64
    tot = ens.sumv_totals().astype(np.float64)
    flux = tot / (T * L)
    cars = sum(N for N, _, _ in specs)
    out = {"config": "C4", "rings": len(specs), "L": L, "total_cars": cars, "steps": T,
           "timed_steps": T - 64, "gpu_seconds": secs, "gpu_car_updates_per_s": cars * (T - 64) / secs,
           "setup_seconds": setup,
           "flux_min": float(flux.min()), "flux_max": float(flux.max()),
           "flux_p0_density_sweep": [float(f) for f in flux[:64:8]]}
    if ref is not None:
        # one slice: the 64 densities at p = 0.0, replica 0, 100 steps each,
        # rings run one after another with all workers each
        ts = 100
        secs_ref = 0.0
        for j in range(64):
            N, p, sd = specs[j]
            x, v = inits[j]
            r = ref.run(L, N, 5, p, sd, ts, workers=cores, x0=x.astype(np.uint64),
                        v0=v.astype(np.uint64), per_step=False, want_state=False)
            secs_ref += r["seconds"]
        slice_cars = sum(specs[j][0] for j in range(64))
        out["cpu_reference"] = {"sample": "64 densities at p=0.0, replica 0, 100 steps each",
                                "workers": cores, "seconds": secs_ref,
                                "car_updates_per_s": slice_cars * ts / secs_ref}
        out["speedup_vs_cpu_reference"] = out["gpu_car_updates_per_s"] / out["cpu_reference"]["car_updates_per_s"]
    # parity spot check: ring 0 against the oracle port on a 200-step prefix
    import oracle
    port = oracle.Port()
    N0, p0, sd0 = specs[0]
    e1 = nasch.Ensemble([nasch.SimParams(length=L, ncars=N0, vmax=5, p=p0, steps=200, seed=sd0)])
    e1.set_state(0, *inits[0])
    e1.advance(200)
    o = port.run(L, 5, p0, sd0, 200, inits[0][0].astype(np.uint64), inits[0][1].astype(np.uint64),
                 want_checksum=False)
    xs, vs = e1.snapshot(0)
    out["parity_ring0_200_steps"] = bool((xs == o["x"]).all() and (vs == o["v"]).all()
                                         and int(e1.sumv_totals()[0]) == int(o["sumv"].sum()))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C1,C2,C3,C4,C5,C5-segments,C3-checksum,C5-checksum")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r02_configs.json"))
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    ref = None
    cores = 1
    if not a.no_cpu:
        import oracle
        ref = oracle.Ref()
        cores = ref.physical_cores() or 1
    want = a.only.split(",")
    res = []
    if "C1" in want:
        res.append(ring("C1", 1000, 200, 0.13, 1000, 42, 0, cpu_steps=1000, ref=ref, cores=1))
    if "C2" in want:
        res.append(ring("C2", 10**6, 2 * 10**5, 0.25, 10**4, 2, 5, cpu_steps=500, ref=ref, cores=cores))
    if "C3" in want:
        res.append(ring("C3", 10**9, 2 * 10**8, 0.13, 1000, 3, 0, cpu_steps=4, ref=ref, cores=cores))
    if "C4" in want:
        res.append(c4(ref, cores))
    if "C5" in want:
        res.append(ring("C5", 10**8, 6 * 10**7, 0.5, 20000, 5, 0, snapshot_every=1000,
                        cpu_steps=10, ref=ref, cores=cores))
        res.append(ring("C5 (k=8)", 10**8, 6 * 10**7, 0.5, 20000, 5, 0, snapshot_every=1000, k=8))
    if "C5-segments" in want:
        res.append(c5_segments())
    if "C3-checksum" in want:
        res.append(ring("C3-checksum", 10**9, 2 * 10**8, 0.13, 20, 3, 0, checksum=True))
    if "C5-checksum" in want:
        res.append(ring("C5-checksum", 10**8, 6 * 10**7, 0.5, 50, 5, 0, checksum=True))
    doc = {"gpu": torch.cuda.get_device_name(0), "cpu_physical_cores": cores, "results": res}
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main()
