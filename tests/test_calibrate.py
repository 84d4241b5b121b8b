"""Calibration loop on CPU: the profile CSV this repo writes is the
reference's ProfileRecord format, and the reference's own fit recovers known coefficients
from records shaped like the B200 profiler's output."""
import sys
from pathlib import Path

import pytest

from paper_2412_01523_b200 import calibrate

ROOT = Path(__file__).resolve().parent.parent
for cand in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if cand.is_dir() and str(cand) not in sys.path:
        sys.path.append(str(cand))
seqplan = pytest.importorskip("seqplan")


def _synthetic(coeffs, loads):
    rows = []
    for d, lens in loads:
        v = 1e15 if d == 1 else 7.7e11
        comp = sum(coeffs["alpha1"] * s * s + coeffs["alpha2"] * s for s in lens) / d + coeffs["beta1"]
        comm = sum(coeffs["alpha3"] * s for s in lens) / (d * v) + coeffs["beta2"]
        mem = sum(lens) / d * coeffs["m_token"] + coeffs["m_ms"]
        rows.append(calibrate.GroupMeasurement(tuple(lens), d, v, comp, comm, mem))
    return rows


def test_profile_csv_round_trips_through_reference_reader(tmp_path):
    from seqplan.cost_model import read_profile_csv
    rows = [calibrate.GroupMeasurement((5, 7, 9), 2, 7.7e11, 1e-3, 2e-4, 1.5e6),
            calibrate.GroupMeasurement((100,), 1, 1e15, 3e-3, 0.0, 2.5e6)]
    path = tmp_path / "p.csv"
    calibrate.write_profile_csv(path, rows)
    recs = read_profile_csv(path)
    assert [(r.token_lengths, r.degree, r.bandwidth, r.measured_comp_time, r.measured_comm_time,
             r.measured_peak_memory) for r in recs] == \
        [(r.token_lengths, r.degree, r.bandwidth, r.comp_s, r.comm_s, r.mem_bytes) for r in rows]


def test_fit_recovers_coefficients():
    truth = {"alpha1": 6e-11, "alpha2": 2.5e-8, "beta1": 1e-4, "alpha3": 65536.0,
             "beta2": 3e-5, "m_token": 2e5, "m_ms": 2e9}
    lengths = [1024 + 37 * i * i for i in range(40)]
    loads = calibrate.group_loads(lengths, [1, 2, 4], per_degree=5)
    fr, merged = calibrate.fit(_synthetic(truth, loads))
    got = merged.to_json_dict()
    for k, v in truth.items():
        assert got[k] == pytest.approx(v, rel=1e-6), k
    assert fr.comp_rel_error < 1e-9
    pred = calibrate.predict(merged, _synthetic(truth, loads))
    assert pred["comm_rel_error_d_ge_2"] < 1e-9


def test_group_loads_are_deterministic_and_distinct():
    lengths = [3, 900, 40, 4096, 7, 123, 2048, 55]
    a = calibrate.group_loads(lengths, [1, 2], per_degree=4)
    assert a == calibrate.group_loads(lengths, [1, 2], per_degree=4)
    for d in (1, 2):
        totals = {sum(l) for dd, l in a if dd == d}
        assert len(totals) >= 3


def test_step_bytes_scale_with_degree():
    b1 = calibrate.step_bytes_per_device([4096, 1024], 1, 32, 128)
    b4 = calibrate.step_bytes_per_device([4096, 1024], 4, 32, 128)
    assert b4 < b1
