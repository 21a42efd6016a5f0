"""Where the time of a temporal-blocked launch goes (experiment build with
-DNB_TB_TRACE, tools/build_variant.sh trace -DNB_TB_TRACE): per launch, the
%globaltimer of the first/last block start, first/last block end and the
last block's plan (cone simulation for the next launch).

  NASCH_B200_LIB=variants/libnasch_trace.so python tools/tb_trace.py
"""
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2309_14311_b200 import capi, nasch  # noqa: E402

L, N, P, SEED = 10**9, 2 * 10**8, 0.13, 3
lib = capi.load()
fn = lib.nasch_b200_tb_trace
fn.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
x, v = nasch.fill_uniform_state(L, N, 0, SEED)
for k in (16, 4):
    os.environ["NASCH_B200_K"] = str(k)
    e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=5, p=P, steps=10**6, seed=SEED))
    e.set_checksum(False)
    e.set_state(x, v)
    e.advance(256)
    torch.cuda.synchronize()
    buf = np.zeros(64 * 8, np.uint64)
    fn(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), 1)
    for _ in range(10):
        e.advance(k)
    torch.cuda.synchronize()
    fn(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), 0)
    tr = buf.reshape(64, 8).astype(np.int64)
    print("raw", [list(map(int, r[:6])) for r in tr[:4]], file=sys.stderr)
    rows = [r for r in tr if r[0] > 0 and r[3] > 0 and r[0] < 2**62]
    rows.sort(key=lambda r: r[0])
    out = []
    for i, r in enumerate(rows):
        d = {"start_spread_us": (r[1] - r[0]) / 1e3, "end_spread_us": (r[3] - r[2]) / 1e3,
             "body_us": (r[3] - r[0]) / 1e3, "ticket_to_plan_us": (r[4] - r[3]) / 1e3,
             "plan_us": (r[5] - r[4]) / 1e3}
        if i + 1 < len(rows):
            d["gap_to_next_us"] = (rows[i + 1][0] - r[5]) / 1e3
        out.append(d)
    print(json.dumps({"k": k, "launches": out[1:-1]}, indent=None), flush=True)
    e.close()
