"""CPU checks of bench.py's roofline accounting (no GPU).

The whole-step roofline divides 4·D/N algorithmic HBM bytes (append r+w, ring-put read,
incoming replica writes) and D/N NVLink bytes by the step time;
the step kernel's roofline pairs every timed launch with its own bytes, and its traffic comes
from the committed ncu launch list of the same command.
"""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_under_test", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_step_roofline_one_gpu(bench):
    # D = 19.1 MB replicated per step for 400 steps at 19.1 us per step
    D, steps, us = 19.1e6, 400, 19.1
    r = bench.step_roofline(D * steps, us * steps * 1e-3, 1, 6541.5, "measured")
    assert r["hbm"]["achieved"] == pytest.approx(4 * D / (us * 1e-6) / 1e9, rel=1e-3)
    assert r["hbm"]["frac"] == pytest.approx(r["hbm"]["achieved"] / 6541.5, abs=1e-4)
    assert "nvlink" not in r


def test_step_roofline_is_per_gpu(bench):
    # weak scaling: N GPUs move N times the bytes in the same time -> same per-GPU figures
    one = bench.step_roofline(1e9, 1.0, 1, 6541.5, "m")
    four = bench.step_roofline(4e9, 1.0, 4, 6541.5, "m")
    assert four["hbm"]["achieved"] == pytest.approx(one["hbm"]["achieved"])
    assert four["nvlink"]["achieved"] == pytest.approx(1e9 / 1.0e-3 / 1e9)
    assert four["nvlink"]["peak"] == bench.NVLINK_PEAK_GBS


def test_step_kernel_timed_region_traffic(bench):
    """The committed traffic of kv_step_kernel is the average over the 20 launches of the
    driver's timed region (ncu launch list of the same command), every launch listed."""
    pop = bench.traffic_ref("decode_population", "kv_step_kernel")
    assert pop is not None and pop["n_launches"] == len(pop["launches"]) == 20
    per = [x["dram_read"] + x["dram_write"] for x in pop["launches"]]
    assert pop["traffic"] == int(sum(per) / len(per))
    assert pop["dram_read"] + pop["dram_write"] == pytest.approx(pop["traffic"], abs=2)


def _log(app, rep):
    return [{"app_bytes": a, "rep_bytes": r} for a, r in zip(app, rep)]


def test_launch_bytes(bench):
    r = {"app_bytes": 10, "rep_bytes": 7}
    assert bench.launch_bytes(r, 1) == (2 * 10 + 2 * 7, 0)      # loopback: all through HBM
    assert bench.launch_bytes(r, 2) == (2 * 10 + 7, 7)          # the replica writes cross NVLink


def test_timed_roofline_pairs_bytes_with_the_region(bench):
    # three launches with different mixes in a 30 us region: achieved = sum of their own
    # bytes / the region (not the step mean of another window, not a sampled launch time)
    log = _log([4e6, 0, 8e6], [2e6, 5e6, 1e6])
    rec = {"log": log, "ms": 0.030}
    r = bench.timed_roofline(rec, 1, 6550.1, "measured")
    hb = sum(2 * a + 2 * p for a, p in zip([4e6, 0, 8e6], [2e6, 5e6, 1e6]))
    assert r["launches"] == 3 and r["avg_launch_us"] == pytest.approx(10.0)
    assert r["achieved"] == pytest.approx(hb / 30e-6 / 1e9, rel=1e-3)
    assert r["frac"] == pytest.approx(r["achieved"] / 6550.1, abs=1e-4)
    assert r["algorithmic_bytes_per_launch"] == int(hb / 3)
    r2 = bench.timed_roofline(rec, 2, 6550.1, "measured")
    assert r2["bound"] == "nvlink" and r2["peak"] == bench.NVLINK_PEAK_GBS
    assert r2["achieved"] == pytest.approx(8e6 / 30e-6 / 1e9, rel=1e-3)
