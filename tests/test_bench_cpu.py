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


def test_roofline_names_the_binding_bound():
    """`roofline` puts the dominant kernel against the L1 load path (the bound
    that binds a gather kernel), and reports its HBM position separately on
    algorithmic HBM bytes -- never L1-served bytes over the HBM peak."""
    sys.path.insert(0, str(ROOT))
    import bench

    l1 = {"ldg128_gbs": 36000.0, "lds32_gbs": 31000.0, "source": "test"}
    r = bench.roofline(samples=1e12, fp_ms=1000.0, fp_views=720, bp_updates=1e11, bp_ms=100.0, l1=l1)
    assert r["bound"] == "l1_load_path" and r["unit"] == "GB/s" and r["peak"] == 36000.0
    assert r["achieved"] == pytest.approx(32.0e12 / 1.0 / 1e9, abs=0.1)
    assert r["frac"] == pytest.approx(32.0e3 / 36000.0, rel=1e-3)
    alg = 4.0 * (512 ** 3 + 720 * 1024 * 1024)
    assert r["hbm"]["algorithmic_bytes_per_launch"] == alg
    assert r["hbm"]["frac"] == pytest.approx(alg / 1.0 / 1e9 / r["hbm"]["peak"], rel=1e-2)
    assert r["back"]["frac"] == pytest.approx(16.0e11 / 0.1 / 1e9 / 36000.0, rel=1e-3)


def test_ncu_traffic_takes_the_newest_capture(tmp_path, monkeypatch):
    """The roofline's `traffic` comes from the newest committed cfg4 capture: round-letter
    order (r02aq after r02k), and a capture of a view-subset launch is scaled to the
    whole call the bench times."""
    sys.path.insert(0, str(ROOT))
    import bench

    prof = tmp_path / "profiles" / "r02"
    prof.mkdir(parents=True)
    k = bench.FP_KERNEL
    (prof / "ncu_r02k_old.json").write_text(json.dumps({k: {"dram_bytes_per_launch": 1.0, "config": "cfg4-full"}}))
    (prof / "ncu_r02aq_new.json").write_text(json.dumps({k: {"dram_bytes_per_launch": 2.0, "config": "cfg4-full"}}))
    (prof / "ncu_r02zz_probe.json").write_text(json.dumps({k: {"dram_bytes_per_launch": 9.0,
                                                               "config": "cfg4-probe1"}}))
    (prof / "ncu_r02ap_bp.json").write_text(json.dumps({"bpk": {"dram_bytes_per_launch": 3.0, "views": 360,
                                                                 "config": "cfg4-full"}}))
    monkeypatch.setattr(bench, "ROOT", tmp_path)
    traffic, src = bench.ncu_traffic(k)
    assert traffic == 2.0 and src.endswith("ncu_r02aq_new.json")
    traffic, _ = bench.ncu_traffic("bpk")
    assert traffic == 3.0 * bench.VIEWS / 360
