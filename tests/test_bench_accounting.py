"""CPU checks of bench.py's roofline accounting: the numbers a reader
recomputes from the bench line, SURVEY §8(d)'s per-unit costs and the committed peak measurements."""
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.fixture(scope="module")
def bench():
    import bench as B
    return B


WORK = {"tested": 3800.0, "units": 340.0, "cells_aggregated": 300.0, "rows": 60.0, "runs": 200.0}


def test_l2_roofline_bytes_and_fracs(bench):
    peaks = json.load(open(os.path.join(ROOT, "profiles", "r2j_l2_peak.json")))["results"]
    seq = max(r["GBps"] for r in peaks if r["pattern"] == "seq_cg")
    runs = {r["run_records"]: r["GBps"] for r in peaks if r["pattern"] == "runs" and r.get("warps_per_sm") == 64}
    n_info, ms = 1000, 0.01
    out = bench.l2_roofline(n_info, WORK, ms, {"l2_read_bytes": 2.0e9})
    bpw = 16 * 3800 + 16 * 2 * (340 + 300) + 16 * 60 + 32      # record, table entries, row starts, pose
    assert out["bytes_per_wp"] == pytest.approx(bpw)
    assert out["achieved"] == pytest.approx(n_info * bpw / (ms / 1e3) / 1e9)
    assert out["peak"] == seq and out["frac"] == pytest.approx(out["achieved"] / seq)
    # mean run 19 records: the pattern roof is the one measured at runs of 16
    assert out["mean_run_records"] == pytest.approx(19.0)
    assert out["pattern_peak"] == runs[16]
    assert out["frac_of_pattern_peak"] == pytest.approx(out["achieved"] / runs[16])
    assert out["algorithmic_share_of_l2_reads"] == pytest.approx(n_info * bpw / 2.0e9)


def test_l2_roofline_counted_table_bytes(bench):
    w = dict(WORK, unit_table_entries=700.0, row_table_bytes=1500.0)
    out = bench.l2_roofline(1000, w, 0.01, None)
    assert out["bytes_per_wp"] == pytest.approx(16 * 3800 + 16 * 700 + 1500 + 32)


def test_l2_pattern_roof_follows_run_length(bench):
    peaks = json.load(open(os.path.join(ROOT, "profiles", "r2j_l2_peak.json")))["results"]
    runs = {r["run_records"]: r["GBps"] for r in peaks if r["pattern"] == "runs" and r.get("warps_per_sm") == 64}
    w = dict(WORK, runs=WORK["tested"] / 9.0)
    assert bench.l2_roofline(10, w, 1.0, None)["pattern_peak"] == runs[8]
    w = dict(WORK, runs=WORK["tested"] / 2.0)       # shorter than any measured run: the shortest
    assert bench.l2_roofline(10, w, 1.0, None)["pattern_peak"] == runs[min(runs)]
    # longer runs read faster (the pattern's roof rises with the run length)
    ks = sorted(runs)
    assert all(runs[a] <= runs[b] * 1.02 for a, b in zip(ks, ks[1:]))


def test_alu_roofline_uses_survey_units(bench):
    class WL:
        T, N, K = 100, 1000, 10

    w = dict(WORK)
    out = bench.roofline("visibility_gain", 2.0, WL, 10, 1, "culled", {"sm_mhz": 1965.0}, 6544.0, w, None)
    lane = 10 * 100 * (10 * 3800 + 25 * 340 + 25 * 60)      # SURVEY.md:709: 10 / 25 / 25 per test / unit / row
    alu = out["alu"]
    assert alu["bound"] == "alu"
    assert alu["achieved"] == pytest.approx(lane / 2e-3 / 1e12)
    assert alu["peak"] == pytest.approx(148 * 128 * 1965e6 / 1e12)
    assert alu["frac"] == pytest.approx(alu["achieved"] / alu["peak"])
    assert out["l2"]["bound"] == "l2"


def test_primary_roof_is_survey_min_roof(bench):
    """frac = achieved / min(FP32 peak, arithmetic intensity x bandwidth); the culled gain
    kernel's bandwidth is the measured L2 roof, and with SURVEY's per-unit costs (10 lane instructions per
    16-byte record) its product with the intensity is the smaller roof."""
    class WL:
        T, N, K = 100, 1000, 10

    out = bench.roofline("visibility_gain", 2.0, WL, 10, 1, "culled", {"sm_mhz": 1965.0}, 6544.0, dict(WORK), None)
    rule, alu, l2 = out["roof_rule"], out["alu"], out["l2"]
    n_info = 10 * 100
    lane = n_info * (10 * 3800 + 25 * 340 + 25 * 60)
    ai = lane / (n_info * l2["bytes_per_wp"])
    assert rule["ai_lane_instr_per_byte"] == pytest.approx(ai)
    assert rule["l2_roof"] == pytest.approx(ai * l2["peak"] * 1e9 / 1e12)
    assert rule["fp32_roof"] == pytest.approx(alu["peak"])
    assert rule["binding"] == "l2" and rule["l2_roof"] < rule["fp32_roof"]
    # the primary fields are the L2 roof's; its fraction equals achieved lane instructions over AI x L2 peak
    assert out["bound"] == "l2" and out["unit"] == "GB/s"
    assert out["achieved"] == pytest.approx(l2["achieved"]) and out["peak"] == pytest.approx(l2["peak"])
    assert out["frac"] == pytest.approx(alu["achieved"] / rule["l2_roof"])
    assert out["frac"] == pytest.approx(min(1.0, alu["achieved"] / min(rule["fp32_roof"], rule["l2_roof"])))
