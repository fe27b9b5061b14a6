"""GPU: the CLI drop-in (the reference's own CTest cases, tests/CMakeLists.txt:28-35,
plus the stdout/stderr/trace formats of tools/synchro.cpp:210-221) and the
step-by-step engine C-ABI (sw_engine_*, replacing detail::BibfsEngine)."""
import json
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def cli(gpu, *args, stdin=None):
    return subprocess.run([gpu.CLI_PATH, *args], capture_output=True, text=True, input=stdin, timeout=600)


def test_ctest_cli_exact_cerny4(gpu):
    r = cli(gpu, "exact", "--gen", "cerny:4")
    assert r.returncode == 0 and re.search("threshold 9", r.stdout)


def test_ctest_cli_heuristic_smoke(gpu):
    r = cli(gpu, "heuristic", "--gen", "cerny:5", "--algorithm", "adaptive")
    assert r.returncode == 0 and re.search("bound ", r.stdout)


def test_ctest_cli_oracle_smoke(gpu):
    r = cli(gpu, "oracle", "--gen", "cerny:4")
    assert r.returncode == 0 and re.search("threshold 9", r.stdout)


def test_cli_exact_formats_and_trace(gpu, ref, tmp_path):
    case = json.load(open(os.path.join(GOLDEN, "solve_medium.json")))[1]  # random:300,2,1
    tp = tmp_path / "t.txt"
    r = cli(gpu, "exact", "--gen", case["spec"], "--track-word", "--trace", str(tp))
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert lines[0] == f"threshold {case['threshold']}"
    word = [int(x) for x in lines[1].split()[1:]]
    a = gpu.from_spec(case["spec"])
    assert lines[1].startswith("word ") and len(word) == case["threshold"]
    assert ref.is_reset_word(a.n, a.k, a.delta, word)
    err = r.stderr.strip().splitlines()[-1]
    m = re.fullmatch(r"time_s=\S+ peak_mem_bytes=(\d+) upper_bound=(\d+) iterations=(\d+) "
                     r"bfs_steps=(\d+) ibfs_steps=(\d+) dfs=([01])", err)
    assert m, err
    assert [int(x) for x in m.groups()] == [case["peak_memory"], case["upper_bound"], case["iterations"],
                                            case["bfs_steps"], case["ibfs_steps"], int(case["used_dfs"])]
    assert tp.read_text().splitlines() == case["trace"]


def test_cli_exact_stdin_and_errors(gpu):
    r = cli(gpu, "exact", "--input", "-", stdin="4 2\n1 1\n2 1\n3 2\n0 3\n")
    assert r.returncode == 0 and r.stdout == "threshold 9\n"
    assert cli(gpu, "exact", "--input", "-", stdin="3 2\n1 0\n2 1\n0 2\n").returncode == 2
    assert cli(gpu, "exact", "--gen", "random:100,2,1", "--memory", "2000").returncode == 4
    assert cli(gpu, "exact", "--gen", "random:300,2,0", "--time-limit", "0.001").returncode == 6
    assert cli(gpu, "exact", "--gen", "cerny:6", "--dfs-shard", "2/2").returncode != 0


def test_cli_schedules(gpu):
    for sched in ("auto", "bfs", "ibfs", "dfs"):
        r = cli(gpu, "exact", "--gen", "random:50,2,0", "--schedule", sched)
        assert r.returncode == 0 and r.stdout == "threshold 16\n", (sched, r.stderr)


def test_engine_step_api_replays_golden_schedule(gpu):
    """Drive the engine through sw_engine_* exactly like solve_exact's loop and
    compare the per-iteration list sizes with the golden trace."""
    case = json.load(open(os.path.join(GOLDEN, "solve_small.json")))[24]  # random:100,2,0
    a = gpu.from_spec(case["spec"])
    eng = gpu.Engine(a, case["upper_bound"])
    lines = [l for l in case["trace"] if " step=" in l and "handoff" not in l]
    for line in lines:
        fields = dict(kv.split("=") for kv in line.split())
        r = int(fields["iter"])
        kind = eng.choose(r)
        assert kind == fields["step"]
        st = eng.stats()
        assert (st.lbfs, st.libfs, st.hbfs, st.hibfs) == tuple(int(fields[x]) for x in
                                                               ("lbfs", "libfs", "hbfs", "hibfs"))
        eng.step(kind)
        assert not eng.meet()
    r_dfs = int(case["trace"][-2].split()[0].split("=")[1])
    assert eng.choose(r_dfs) == "DFS"
    assert eng.dfs(r_dfs) == case["threshold"]
    eng.close()


SHIM = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref",
                    "shim_driver")
# spec memory track_word upper_bound dfs_largest history_growth beam_initial
# beam_cost_fraction reduction_of_reduction set_cost
SHIM_CASES = [
    "cerny:16 4294967296 1 0 20000 1.5 0 0.05 0 512",
    "cerny:12 4294967296 0 0 20000 3.0 0 0.05 0 512",
    "random:200,2,1 4294967296 0 0 500 2.0 0 0.05 0 512",
    "random:200,2,1 16777216 1 0 3000 2.0 0 0.05 0 512",
    "random:200,2,1 4194304 0 37 20000 2.0 0 0.05 0 512",
    "random:100,2,5 4294967296 0 0 20000 2.0 0 0.05 0.3 512",
    "random:150,2,4 4294967296 1 0 20000 2.0 100 0.2 0 256",
    "random:100,3,2 4294967296 0 0 20000 2.0 16 0.01 0 512",
]


@pytest.mark.skipif(not os.path.exists(SHIM), reason="shim driver not built (needs the reference)")
def test_reference_side_shim_matches_reference_solve(gpu):
    """include/synchro_b200_shim.hpp compiled against the unmodified reference
    headers (oracle/Makefile `shim`): synchro::solve_exact_b200 with every
    EngineTuning / TuningParams field forwarded returns the reference's
    SolveResult (bibfs_engine.hpp:50-59) and the same trace as the reference's
    own synchro::solve_exact, on non-default dfs_largest, history_growth,
    beam_initial, beam_cost_fraction, reduction_of_reduction and set_cost."""
    r = subprocess.run([SHIM], input="\n".join(SHIM_CASES) + "\n", capture_output=True, text=True,
                       timeout=1200)
    assert r.returncode == 0, r.stderr
    lines = r.stdout.splitlines()
    assert len(lines) == len(SHIM_CASES)
    for line in lines:
        spec, ref_part, b200_part, flags = [x.strip() for x in line.split("|")]
        assert ref_part[4:] == b200_part[5:], line
        assert flags == "1 1", line
