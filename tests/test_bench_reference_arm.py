"""bench.py --impl reference (the driver's reference arm) on CPU: it prints one JSON line with the
contract's keys, times the reference's algorithm on the oracle, and never maps the B200 library
(bench.py:mapped_product_libraries)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line_and_no_product_library():
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "0", "--cpu-budget", "1"],
                         capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["higher_is_better"] is False and d["unit"] == "s/system"
    assert d["product_libraries_mapped"] == []
    assert d["config"]["row_sum"] == "ordered" and d["config"]["orthogonalization"] == "mgs"
    assert d["config"]["factor_solve"] == "sweep"
    assert d["e2e"]["value"] == d["value"] and d["cpu_baseline"]["kind"] == "port"
    assert d["value"] > 0 and d["per_iteration_s"] > 0
