"""bench.py's CPU-side contract: --impl reference prints one JSON line with the
oracle's throughput (no GPU needed)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_reference_arm_json():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--workload", "c1", "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "updates/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["workload"] == "c1"


def test_bench_reference_nonzero_rank_is_silent():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--workload", "c1", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_operating_points_map_to_asaga_options():
    """Every bench operating point translates into keyword options the binding accepts (a
    renamed option would otherwise only fail on the GPU box)."""
    import inspect

    import bench
    from paper_1606_04809_b200 import Asaga

    params = inspect.signature(Asaga.__init__).parameters
    assert set(bench.OPERATING_POINT) == {"c1", "c2", "c3", "c4"}
    for name, op in bench.OPERATING_POINT.items():
        kw = bench.asaga_options(op)
        for k in kw:
            assert k in params, (name, k)
        assert op["W"] > 0 and 0.0 < op["gscale"] <= 1.0
    assert bench.default_workload(1) == "c4" and bench.default_workload(8) == "c3"
