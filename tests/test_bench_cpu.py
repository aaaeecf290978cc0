"""CPU checks of the benchmark harness: the reference arm (oracle port on host
cores) prints one contract-shaped JSON line, and the roofline helpers are
consistent.  No GPU needed."""

import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_prints_contract_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--cpu-views", "1"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["unit"] == "GUPS" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def test_gather_roofline_fractions():
    sys.path.insert(0, str(ROOT))
    import bench

    g = bench.gather_roofline(32.0 * 1e12, 1000.0, 16.0 * 1e12, 500.0, {"sm_mhz": 1965.0})
    # peak = measured LDG.128 bytes/clk/SM (profiles/l1_peak_*.json) x 148 SMs x clock
    per_clk = json.loads(sorted((ROOT / "profiles").glob("l1_peak_*.json"))[-1].read_text())["ldg128_bytes_per_clk_sm"]
    peak = per_clk * 148 * 1965.0 * 1e6 / 1e9
    assert 120.0 <= per_clk <= 128.0 and "measured" in g["peak_source"]
    assert g["peak"] == pytest.approx(peak, abs=0.1)
    assert g["forward"]["achieved"] == pytest.approx(32.0e12 / 1.0 / 1e9, abs=0.1)
    assert g["back"]["frac"] == pytest.approx(16.0e12 / 0.5 / 1e9 / peak, rel=1e-3)
