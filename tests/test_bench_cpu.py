"""CPU: the host side of bench.py that the driver depends on — the one-line
JSON contract of the reference arm (rank 0 prints, other ranks exit 0
silently), the read:write mix ceiling next to the roofline, and the NUMA
binding helper's no-op paths.  The reference arm runs the compiled
reference (oracle/_ref) on a bounded sample: a few seconds here."""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402

REQUIRED = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
            "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"}


def _ref_built() -> bool:
    return any((ROOT / "oracle" / "_ref").glob("*.so"))


def test_mix_ceiling_picks_the_kernels_mix():
    phi, n = 2651553280, 266118400
    k23 = {"bytes": 2 * phi + 28 * n, "write_bytes": 12 * n + 2 * phi}
    k23["GBps"] = k23["bytes"] / 2.24e-3 / 1e9
    m = bench.mix_ceiling(k23)
    assert m["mix"].startswith("1:2") and 0.9 < m["frac"] < 1.0
    k1 = {"bytes": 2 * phi + 4 * n, "write_bytes": 2 * n}
    k1["GBps"] = k1["bytes"] / 0.98e-3 / 1e9
    assert bench.mix_ceiling(k1)["mix"] == "read"
    assert bench.mix_ceiling({"bytes": 1, "GBps": 1.0}) is None  # no write split: not reported


def test_numa_binding_is_a_no_op_without_nvml(monkeypatch):
    if not hasattr(os, "sched_getaffinity"):
        pytest.skip("no affinity API")
    before = os.sched_getaffinity(0)
    monkeypatch.setenv("SAMO_BENCH_NUMA", "0")
    with bench.gpu_local_cpus(0):
        assert os.sched_getaffinity(0) == before
    monkeypatch.setenv("SAMO_BENCH_NUMA", "1")
    with bench.gpu_local_cpus(0):  # no GPU / NVML here: left to the OS
        pass
    assert os.sched_getaffinity(0) == before


def test_clock_sampler_summaries(monkeypatch):
    """The clocks object: off / non-zero ranks sample nothing; nvidia-smi rows
    and NVML samples reduce to the contract's keys, reasons as a union."""
    monkeypatch.setenv("SAMO_BENCH_CLOCKS", "off")
    with bench.ClockSampler("0") as clk:
        pass
    assert not clk.active() and clk.summary()["samples"] == 0
    with bench.ClockSampler(None) as clk:  # ranks other than 0
        clk.sample_now()
    assert clk.summary()["samples"] == 0 and clk.in_region == 0
    clk = bench.ClockSampler("0")
    clk.lines = ["1965, 1965, 350.5, Not Active, Not Active, Not Active, Active, 3996",
                 "1950, 1965, 360.0, Not Active, Not Active, Not Active, Not Active, 3996", "garbage"]
    clk.samples = [(1965.0, 1965.0, 3996.0, None, {"hw_slowdown"})]
    s = clk.summary()
    assert s["sm_mhz"] == 1965.0 and s["sm_max_mhz"] == 1965.0 and s["samples"] == 3
    assert s["reasons"] == ["hw_slowdown", "sw_power_cap"]
    assert s["mem_mhz"] == 3996.0 and s["power_w_max"] == 360.0


@pytest.mark.skipif(not _ref_built(), reason="oracle/_ref not built")
def test_reference_arm_prints_one_json_line():
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, res.stdout[-2000:]
    d = json.loads(lines[0])
    assert REQUIRED <= set(d), REQUIRED - set(d)
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.skipif(not _ref_built(), reason="oracle/_ref not built")
def test_reference_arm_other_ranks_exit_silently():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    res = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300,
                         cwd=ROOT, env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    assert res.stdout.strip() == ""


@pytest.mark.parametrize("name,p,tensors,phi,nnz", [
    ("gpt-2.7b", 0.9, 388, 2_651_553_280, 266_118_400),
    ("gpt-1.3b", 0.8, 292, 1_315_723_264, 263_659_096),   # config 3
    ("gpt-1.3b", 0.9, 292, 1_315_723_264, 132_151_096),
    ("gpt-1.3b", 0.95, 292, 1_315_723_264, 66_397_096),
])
def test_workloads_match_the_survey(oracle, name, p, tensors, phi, nnz):
    """The bench's synthetic GPT parameter sets: tensor
    count, dense parameters and kept elements under the reference's
    unpruned_count (prune.hpp:76-79; 1-D LN/bias tensors non-prunable)."""
    from paper_2302_05045_b200 import workloads
    wl = workloads.get(name, p)
    assert len(wl.tensors) == tensors and wl.phi == phi
    kept = sum(oracle.unpruned_count(p, t.numel) if t.prunable else t.numel for t in wl.tensors)
    assert kept == nnz
