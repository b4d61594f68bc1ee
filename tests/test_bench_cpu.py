"""bench.py's CPU legs (no GPU): the --impl reference arm (the fp64 oracle on the host cores) prints
the contract's JSON line, on every host core even after a 1-thread measurement in the same process."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line_and_cores(tmp_path):
    env = dict(os.environ, AD2_BENCH_CACHE=str(tmp_path))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "1",
                        "--steps", "2", "--warmup", "1", "--cpu-budget", "1"], capture_output=True, text=True,
                       env=env, timeout=600)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "entry-iter/s" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    import oracle
    assert line["cpu_baseline"]["cores"] == oracle.max_threads()


def test_cpu_baseline_keeps_all_cores_after_one_thread_leg():
    sys.path.insert(0, ROOT)
    import bench
    import oracle
    from paper_1510_00012_b200 import workloads as wl
    b = wl.make_config(1)
    n0 = bench.host_cores()
    a = bench.cpu_baseline(b, budget_s=0.01, one_thread=True)       # runs the 1-thread leg last
    assert a["cores"] == n0 and "value_1thread" in a
    c = bench.cpu_baseline(b, n_clusters=1)
    assert c["cores"] == n0
    assert oracle.max_threads() in (1, n0)                            # the OpenMP setting itself may be 1 now
