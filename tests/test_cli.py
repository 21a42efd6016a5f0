"""The `nasch` command line (paper_2309_14311_b200/bin/nasch), checked the
way the reference checks its own (/root/reference/proj/tests/cli_tests.sh:
exit codes, thread precedence, output files, verify/bench tables).

Argument, parameter-file and precedence errors are decided before any
simulation is built, so those cases run without a GPU; everything that
steps a ring is marked gpu.  The pinned checksum is the reference's
(test_engine.cpp:114, test_capi.cpp:116) for the same base.params.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NASCH = os.path.join(ROOT, "paper_2309_14311_b200", "bin", "nasch")
BASE = "length = 50\nncars = 10\nvmax = 3\np = 0.5\nsteps = 20\nseed = 1\n"
PINNED = format(6917392272001519308, "016x")  # reference test_capi.cpp:116


def run(args, cwd, env=None):
    e = dict(os.environ)
    e.pop("NASCH_THREADS", None)
    e.update(env or {})
    p = subprocess.run([NASCH] + args, cwd=cwd, env=e, capture_output=True, text=True, timeout=300)
    return p.returncode, p.stdout, p.stderr


@pytest.fixture
def work(tmp_path):
    if not os.path.exists(NASCH):
        pytest.fail("nasch CLI not built (make -C paper_2309_14311_b200/csrc)")
    (tmp_path / "base.params").write_text(BASE)
    return tmp_path


def checksum_of(out):
    m = re.search(r"^checksum = ([0-9a-f]{16})$", out, re.M)
    assert m, out
    return m.group(1)


# ---- no GPU needed -------------------------------------------------------

def test_usage_errors(work):
    assert run(["run", "--params", "base.params", "--threads", "0"], work)[0] == 1
    assert run(["run"], work)[0] == 1
    assert run(["frobnicate"], work)[0] == 1
    assert run([], work)[0] == 1
    assert run(["run", "--params", "base.params", "--output", "gif"], work)[0] == 1
    assert run(["run", "--params", "base.params", "--threads", "-2"], work)[0] == 1
    assert run(["run", "--params", "base.params", "--bogus"], work)[0] == 1
    assert run(["verify", "--params", "base.params"], work)[0] == 1
    assert run(["verify", "--params", "base.params", "--max-threads", "0"], work)[0] == 1
    assert run(["bench", "--params", "base.params"], work)[0] == 1
    assert run(["bench", "--params", "base.params", "--threads-list", "1,0"], work)[0] == 1
    assert run(["bench", "--params", "base.params", "--threads-list", "1", "--repeats", "0"], work)[0] == 1


def test_garbage_env_threads_is_usage_error(work):
    assert run(["run", "--params", "base.params"], work, {"NASCH_THREADS": "potato"})[0] == 1


def test_param_file_errors(work):
    (work / "broken.params").write_text("length = 50\nwheels = 3\n")
    code, _, err = run(["run", "--params", "broken.params"], work)
    assert code == 1 and "error:" in err
    code, _, err = run(["run", "--params", "does_not_exist.params"], work)
    assert code == 3 and "does_not_exist.params" in err
    (work / "bad.params").write_text("length = 5\nncars = 9\n")  # N > L: invalid
    assert run(["run", "--params", "bad.params"], work)[0] == 1


def test_help(work):
    for args in (["--help"], ["run", "--help"], ["verify", "--help"], ["bench", "--help"]):
        code, out, _ = run(args, work)
        assert code == 0 and "Usage" in out


# ---- on the GPU ----------------------------------------------------------

@pytest.mark.gpu
def test_run_checksum_and_threads(work):
    code, out, _ = run(["run", "--params", "base.params"], work)
    assert code == 0
    assert checksum_of(out) == PINNED
    assert "threads=1" in out
    for line in ("density = 0.200000", "mean_velocity = ", "flow = "):
        assert line in out
    for t in ("2", "3", "8"):
        for eng in ("cuda", "agent"):
            c, o, _ = run(["run", "--params", "base.params", "--threads", t, "--engine", eng], work)
            assert c == 0 and checksum_of(o) == PINNED


@pytest.mark.gpu
def test_thread_precedence(work):
    _, out, _ = run(["run", "--params", "base.params"], work, {"NASCH_THREADS": "3"})
    assert "threads=3" in out
    _, out, _ = run(["run", "--params", "base.params", "--threads", "2"], work, {"NASCH_THREADS": "3"})
    assert "threads=2" in out
    (work / "t.params").write_text(BASE + "threads = 4\n")
    _, out, _ = run(["run", "--params", "t.params"], work)
    assert "threads=4" in out


@pytest.mark.gpu
def test_output_files(work):
    assert run(["run", "--params", "base.params", "--output", "pgm", "--out", "road.pgm"], work)[0] == 0
    assert (work / "road.pgm").read_bytes()[:2] == b"P5"
    code, out, _ = run(["run", "--params", "base.params", "--output", "ascii", "--out", "road.txt"], work)
    assert code == 0 and "wrote road.txt (20 frames)" in out
    assert len((work / "road.txt").read_text().splitlines()) == 20
    assert run(["run", "--params", "base.params", "--output", "ascii", "--out", "wide.txt",
                "--threads", "8"], work)[0] == 0
    assert (work / "road.txt").read_bytes() == (work / "wide.txt").read_bytes()
    assert run(["run", "--params", "base.params", "--output", "none", "--out", "never.txt"], work)[0] == 0
    assert not (work / "never.txt").exists()
    run(["run", "--params", "base.params", "--output", "pgm"], work)
    assert (work / "traffic.pgm").exists()
    run(["run", "--params", "base.params", "--output", "ascii"], work)
    assert (work / "traffic.txt").exists()


@pytest.mark.gpu
def test_overrides(work):
    c1 = checksum_of(run(["run", "--params", "base.params", "--seed", "2"], work)[1])
    c2 = checksum_of(run(["run", "--params", "base.params", "--seed", "2"], work)[1])
    assert c1 == c2 != PINNED
    assert "steps=5" in run(["run", "--params", "base.params", "--steps", "5"], work)[1]


@pytest.mark.gpu
def test_verify(work):
    code, out, _ = run(["verify", "--params", "base.params", "--max-threads", "6"], work)
    assert code == 0, out
    assert "OK: all checksums identical" in out
    assert len(re.findall(r"^workers \d+: checksum " + PINNED + "$", out, re.M)) == 6
    assert "grid reference: checksum " + PINNED in out


@pytest.mark.gpu
def test_verify_segmented_ring(work):
    # large enough that workers 2..4 really split the ring into segments
    (work / "seg.params").write_text("length = 4000\nncars = 1500\nvmax = 5\np = 0.3\nsteps = 60\nseed = 9\n")
    code, out, _ = run(["verify", "--params", "seg.params", "--max-threads", "4"], work)
    assert code == 0, out
    sums = set(re.findall(r"checksum ([0-9a-f]{16})", out))
    assert len(sums) == 1


@pytest.mark.gpu
def test_bench_table_matches_csv(work):
    code, out, _ = run(["bench", "--params", "base.params", "--threads-list", "1,2", "--repeats", "2"], work)
    assert code == 0, out
    assert "workers,wall_time_s,speedup,efficiency,checksum" in out
    csv = {l.split(",")[0]: l for l in out.splitlines() if re.match(r"^\d+,", l)}
    assert csv["1"].split(",")[2] == "1.0000"
    assert csv["1"].split(",")[4] == PINNED
    for w in ("1", "2"):
        row = next(l for l in out.splitlines() if re.match(r"^ +%s " % w, l))
        assert ",".join(row.split()) == csv[w]
    code, out, _ = run(["bench", "--params", "base.params", "--threads-list", "2", "--repeats", "1"], work)
    assert code == 0 and re.search(r"^1,", out, re.M)
    with open(work / "base.params", "a") as f:
        f.write("output = ascii\n")
    code, out, _ = run(["bench", "--params", "base.params", "--threads-list", "1", "--repeats", "1",
                        "--no-output"], work)
    assert code == 0
    assert next(l for l in out.splitlines() if l.startswith("1,")).split(",")[4] == PINNED
