"""CPU checks of bench.py's host logic (no GPU): the C4 ring specs, the ring
partition across ranks, the NCCL INIT-line summary, the torchrun re-launch
command and the --gpus / WORLD_SIZE consistency rule."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2309_14311_b200 import nasch  # noqa: E402


def test_c4_specs_match_baseline_config():
    specs = bench.c4_specs()
    assert len(specs) == 4096
    ns = sorted({n for n, _, _ in specs})
    assert ns[0] == 5000 and ns[-1] == 50000 and len(ns) == 64
    assert sorted({p for _, p, _ in specs}) == [0.0, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7]
    assert len({s for _, _, s in specs}) == 4096  # one stream per ring
    assert sum(n for n, _, _ in specs) == 112638272


def test_c4_partition_is_balanced_and_complete():
    ncars = [n for n, _, _ in bench.c4_specs()]
    for world in (1, 2, 4, 8):
        parts = nasch.partition_rings(ncars, world)
        assert parts[0][0] == 0 and parts[-1][1] == len(ncars)
        assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
        loads = [sum(ncars[lo:hi]) for lo, hi in parts]
        assert max(loads) - min(loads) <= max(ncars)  # within one ring of perfect balance


def test_nccl_init_summary(tmp_path):
    log = tmp_path / "nccl.log"
    log.write_text("box:1:1 [0] NCCL INFO NCCL version 2.28.9+cuda12.8\n"
                   "box:1:9 [0] NCCL INFO comm 0x55 rank 0 nRanks 8 nNodes 1 localRanks 8 localRank 0\n"
                   "box:1:9 [0] NCCL INFO ncclCommInitRank comm 0x55 rank 0 nranks 8 - Init COMPLETE\n"
                   "box:1:9 [0] NCCL INFO something else\n")
    s = bench.nccl_init_summary(str(log))
    assert s["init_lines"] == 3 and s["nranks_seen"] == [8]
    assert bench.nccl_init_summary(str(tmp_path / "missing.log")) is None


def test_gpus_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4"], env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr


def test_spawn_command(monkeypatch):
    seen = {}

    def fake_call(cmd):
        seen["cmd"] = cmd
        return 0

    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "8", "--steps", "20"])
    args = bench.argparse.Namespace(gpus=8)
    assert bench.spawn(args) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=8" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "8", "--steps", "20"]


def test_dist_identity_at_one_rank():
    d = bench.Dist(0, 1, 0)
    assert d.max(3.5) == 3.5 and d.all_true(True) and not d.all_true(False)
    assert d.bcast({"a": 1}) == {"a": 1} and d.gather(7) == [7]
    d.barrier()
    d.close()
    assert np.isclose(d.max(1.0), 1.0)
