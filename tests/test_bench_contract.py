"""bench.py's JSON contract, checked on CPU through the reference (oracle) arm, and the
graft entry points' presence."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_prints_one_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e", "impl"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "doubles/s"
    assert d["higher_is_better"] is True and d["steps"] == 2
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and "sample" in cb
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_reference_arm_nonzero_rank_exits_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--gpus", "2"], capture_output=True, text=True, timeout=120, cwd=ROOT,
                         env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_clock_rejection_rule():
    """Timing rules: hw_slowdown / hw_thermal_slowdown / sw_thermal_slowdown, or SM clocks far
    below max with no reason (a leftover lock), reject the timed region; sw_power_cap does not."""
    sys.path.insert(0, ROOT)
    import bench
    ok = {"sm_mhz": 1965, "sm_max_mhz": 1965, "reasons": [], "samples": 20}
    assert not bench.clocks_rejected(ok)
    assert not bench.clocks_rejected(dict(ok, sm_mhz=1560, reasons=["sw_power_cap"]))
    for r in ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"):
        assert bench.clocks_rejected(dict(ok, reasons=[r]))
    assert bench.clocks_rejected(dict(ok, sm_mhz=1000))
    assert not bench.clocks_rejected(dict(ok, samples=0, sm_mhz=None))


def test_graft_entry_has_build_and_smoke():
    sys.path.insert(0, ROOT)
    import __graft_entry__ as g
    assert callable(g.build) and callable(g.smoke)


def _json_line(stdout: str) -> dict:
    lines = [l for l in stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, stdout[-2000:]
    return json.loads(lines[0])


@pytest.mark.gpu
def test_our_arm_one_gpu_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "5", "--warmup", "3",
                          "--config", "c1", "--e2e-steps", "1"], capture_output=True, text=True, timeout=900,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = _json_line(out.stdout)
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] >= 3 and d["value"] > 0
    assert d["gpu_launches"] == 5                       # one fused launch per step
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["peak"] > 0 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    # achieved = algorithmic bytes per launch (8 per summand) / the kernel's average duration
    assert r["algorithmic_bytes_per_launch"] == 8 * d["config"]["n_per_gpu"]
    assert abs(r["achieved"] - r["algorithmic_bytes_per_launch"] / (r["kernel_ms"] * 1e6)) < 1e-6 * r["achieved"]
    assert d["e2e"]["h2d_bytes_per_step"] == 8 * d["config"]["n_per_gpu"] and d["e2e"]["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["clocks"]["sm_max_mhz"]
    assert len(d["result"]["value_hex"]) == 16 and len(d["result"]["image_sha256"]) == 64


@pytest.mark.gpu
def test_our_arm_two_ranks_host_path_on_one_gpu():
    """The N>1 host path of bench.py (launch, barrier, max over ranks, e2e, cross-rank result
    check) with 2 ranks sharing one GPU over gloo; no fused exchange (its kernels would wait on
    each other, which must not run as separate launches on one GPU)."""
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", "29571", os.path.join(ROOT, "bench.py"),
                          "--gpus", "2", "--steps", "3", "--warmup", "3", "--config", "c1", "--dist-backend", "gloo",
                          "--e2e-steps", "1"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    d = _json_line(out.stdout)
    assert d["n_gpus"] == 2 and d["config"]["n_total"] == 2 * d["config"]["n_per_gpu"]
    assert d["gpu_launches"] == 6 and d["e2e"]["h2d_bytes_per_step"] == 2 * 8 * d["config"]["n_per_gpu"]


def test_bench_faithful_check():
    """bench.faithful (the c2cs / c3cs line's check): y is RD or RU of the exact A * 2^-1074."""
    import math
    sys.path.insert(0, ROOT)
    import bench
    one = 1 << 1074                                        # 1.0 in units of 2^-1074
    ulp = 1 << (1074 - 52)
    assert bench.faithful(1.0, one)
    assert bench.faithful(1.0, one + ulp // 3) and bench.faithful(1.0, one + ulp - 1)
    assert not bench.faithful(1.0, one + ulp)              # S = succ(1.0): only succ is faithful
    assert bench.faithful(math.nextafter(1.0, 2.0), one + ulp // 3)
    assert bench.faithful(1.0, one - ulp // 4) and not bench.faithful(1.0, one - ulp // 2)   # gap below is ulp/2
    assert not bench.faithful(math.inf, one) and not bench.faithful(math.nan, one)
    assert bench.faithful(-1.0, -one - 1) and not bench.faithful(-1.0, one)
