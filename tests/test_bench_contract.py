"""bench.py's reference arm keeps the driver's one-JSON-line contract (CPU: the
reference arm needs no GPU; small workload)."""
import json
import os
import subprocess
import sys

import pytest

from oracle import ref

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref (the compiled reference) is not built")
def test_reference_arm_prints_one_json_line():
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--per-rank-mib", "2", "--cpu-seconds", "0.2"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, res.stdout
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        assert d["metric"] == json.load(f)["metric"]


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref (the compiled reference) is not built")
def test_reference_arm_loads_no_product_code():
    """The reference arm (matrix generation included) runs the reference's own
    code only: no product module imported, no product library mapped."""
    code = ("import sys, argparse, bench\n"
            "a = argparse.Namespace(steps=1, warmup=3, per_rank_mib=1, ratio=0.7, cpu_seconds=0.1, fresh_matrix=False)\n"
            "line = bench.run_reference(a)\n"
            "maps = open('/proc/self/maps').read()\n"
            "assert 'libnimble_b200' not in maps, 'product library mapped'\n"
            "assert not any(m.startswith('paper_2604_00317_b200') for m in sys.modules), 'product imported'\n"
            "assert line['config'] == bench.config_of(8, a)\n"
            "print('ok')\n")
    res = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert res.returncode == 0 and "ok" in res.stdout, res.stderr[-2000:]
