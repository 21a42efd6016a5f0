"""Generates tests/golden/reference_vectors.json from the REFERENCE ITSELF:
oracle/_ref/libnasch_ref.so, the unmodified /root/reference sources compiled
by oracle/Makefile (run in the build container, where /root/reference
exists; the GPU box only reads the committed JSON).

    python tests/golden/make_golden.py

Each record: the parameters, the injected initial state (or null for the
reference's own init_state, src/model.cpp:30-40), and what the reference
Engine returned after `steps` steps -- final positions and velocities in rank
order (in full up to 600 cars, always as SHA-256 of their little-endian u64
bytes), every step's velocity sum and origin-crossing count, and the FNV-1a
trajectory checksum (src/engine.hpp:15-51).  The reference is run with 1 and
with 3 workers; the two must agree (its own reproducibility claim)."""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402

CASES = [
    # name, L, N, vmax, p, seed, steps, state: None (init_state) or (vmax_init, state_seed)
    ("frozen-endpoint test_capi.cpp:105-119", 50, 10, 3, 0.5, 1, 20, None),
    ("BASELINE C1", 1000, 200, 5, 0.13, 42, 1000, (0, 42)),
    ("one car", 7, 1, 5, 0.3, 3, 40, None),
    ("full road", 64, 64, 3, 0.5, 4, 10, None),
    ("vmax above L-1", 10, 3, 50, 0.2, 5, 60, None),
    ("p = 0", 300, 60, 5, 0.0, 6, 100, (5, 6)),
    ("p = 1", 300, 60, 5, 1.0, 7, 100, (5, 7)),
    ("L % 32 == 0, vmax 7 (bit-plane grid)", 320, 77, 7, 0.35, 8, 200, (7, 8)),
    ("vmax 300 (u32 velocities)", 5000, 40, 300, 0.25, 9, 150, (100, 9)),
    ("300 cars (four-warp kernel)", 1500, 300, 5, 0.2, 10, 300, (5, 10)),
    ("513 cars (one-CTA kernel)", 3000, 513, 5, 0.3, 11, 300, (3, 11)),
    ("5000 cars (distributed-resident kernel)", 30000, 5000, 5, 0.25, 12, 100, (5, 12)),
    ("700000 cars (temporal-blocked kernel)", 3500000, 700000, 5, 0.13, 13, 40, (0, 13)),
]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.dtype("<u8")).tobytes()).hexdigest()


def main():
    ref, port = O.Ref(), O.Port()
    out = []
    for name, L, N, vmax, p, seed, steps, st in CASES:
        x0 = v0 = None
        if st is not None:
            x0, v0 = port.fill_uniform_state(L, N, st[0], st[1])
            x0, v0 = np.asarray(x0, np.uint64), np.asarray(v0, np.uint64)
        r1 = ref.run(L, N, vmax, p, seed, steps, workers=1, x0=x0, v0=v0)
        r3 = ref.run(L, N, vmax, p, seed, steps, workers=min(3, N), x0=x0, v0=v0)
        assert r1["checksum"] == r3["checksum"] and (r1["x"] == r3["x"]).all() and (r1["v"] == r3["v"]).all()
        assert (r1["sumv"] == r3["sumv"]).all() and (r1["wraps"] == r3["wraps"]).all()
        rec = dict(name=name, L=L, N=N, vmax=vmax, p=p, seed=seed, steps=steps,
                   state=None if st is None else dict(generator="fill_uniform_state", vmax_init=st[0], seed=st[1],
                                                      x0_sha256=sha(x0), v0_sha256=sha(v0)),
                   checksum=int(r1["checksum"]), x_sha256=sha(r1["x"]), v_sha256=sha(r1["v"]),
                   sumv=[int(s) for s in r1["sumv"]], wraps=[int(w) for w in r1["wraps"]])
        if N <= 600:
            rec["x"] = [int(a) for a in r1["x"]]
            rec["v"] = [int(a) for a in r1["v"]]
            if st is not None:
                rec["state"]["x0"] = [int(a) for a in x0]
                rec["state"]["v0"] = [int(a) for a in v0]
        out.append(rec)
        print(name, hex(rec["checksum"]))
    with open(os.path.join(HERE, "reference_vectors.json"), "w") as f:
        json.dump(dict(source="oracle/_ref/libnasch_ref.so (the reference's src/*.cpp, unmodified, g++ -O3 -fopenmp)",
                       records=out), f, separators=(",", ":"))


if __name__ == "__main__":
    main()
