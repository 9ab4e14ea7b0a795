"""CPU checks of bench.py's roofline accounting (no GPU).

The whole-step roofline divides 4·D/N algorithmic HBM bytes (append r+w, ring-put read,
incoming replica writes) and D/N NVLink bytes by the step time;
the copy-node traffic comes from the committed ncu population capture.
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


def test_copy_node_population_traffic(bench):
    pop = bench.traffic_ref("decode_population", "kv_ring_put_copy_kernel")
    assert pop is not None and pop["n_launches"] >= 8
    assert pop["traffic"] == pop["dram_read"] + pop["dram_write"]
    # the kernel requests each payload byte once: L2 writes = D, L2 reads = D + descriptors
    assert pop["algorithmic_rw"] == 2 * pop["l2_write_requested"]
    assert 0 <= pop["l2_read_requested"] - pop["l2_write_requested"] < 0.01 * pop["l2_write_requested"]
    # no re-reads from DRAM: read traffic within 1 % of the requested reads
    assert pop["dram_read"] <= 1.01 * pop["l2_read_requested"]
    assert pop["traffic_over_algorithmic"] == pytest.approx(pop["traffic"] / pop["algorithmic_rw"], abs=1e-3)
