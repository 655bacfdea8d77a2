"""CPU: bench.py's CSV rows use the reference report schema
(proj/src/bench.cpp:151-163) with the reference's statistics — best_ns = the
fastest step, mean_ns = the mean step, gbps = input bytes / best_ns (decimal
GB/s), error_margin_pct = 100 (mean - best) / best (bench.cpp:77-87) — and
parse, exactly, with the reference's OWN parse_csv (bench.cpp:172-203, built
from /root/reference into oracle/_ref). A mixed GPU + CPU report parses."""
import os
import sys

import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

pytestmark = pytest.mark.skipif(O.ref() is None, reason="oracle/_ref (the reference build) is not present")


def test_rows_round_trip_through_reference_parse_csv(tmp_path):
    path = str(tmp_path / "report.csv")
    gpu_steps = [2_461_903, 2_458_117, 2_470_550, 2_459_001]           # ns per step (CUDA events)
    bench.write_csv(path, [("cuda-sm100a-copy", 1 << 32, gpu_steps, None),
                           ("cuda-sm100a-inplace", 1 << 32, [1_861_000, 1_902_345], None)])
    bench.write_csv(path, [("reference-bitmask-x16-copy", 1 << 27, [5_123_456], 5_500_000.25)])   # appended
    rows = O.ref_parse_csv(path)
    assert [r[0] for r in rows] == ["cuda-sm100a-copy", "cuda-sm100a-inplace", "reference-bitmask-x16-copy"]
    impl, units, nbytes, best, mean, gbps, margin = rows[0]
    assert (units, nbytes, best) == (1 << 32, 2 << 32, min(gpu_steps))
    assert mean == sum(gpu_steps) / len(gpu_steps)
    assert gbps == (2 << 32) / min(gpu_steps)
    assert margin == 100.0 * (mean - best) / best
    assert rows[2][3:5] == (5_123_456, 5_500_000.25)
    with open(path) as f:
        lines = f.read().splitlines()
    assert lines[0] == "impl,input_units,bytes,best_ns,mean_ns,gbps,error_margin_pct"
    assert len(lines) == 4 and all(l.count(",") == 6 for l in lines)


def test_reference_rejects_the_round1_cpu_row_format(tmp_path):
    """The round-1 CPU rows left cells empty; the reference parser throws on
    them (stoull of ""), which is why every row is now complete."""
    p = tmp_path / "old.csv"
    p.write_text("impl,input_units,bytes,best_ns,mean_ns,gbps,error_margin_pct\nreference-reference,,,,,61.058,\n")
    with pytest.raises(ValueError):
        O.ref_parse_csv(str(p))


def test_reference_arm_appends_parseable_rows(tmp_path):
    path = str(tmp_path / "ref.csv")
    import subprocess

    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c0",
                        "--steps", "3", "--warmup", "3", "--csv", path], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    rows = O.ref_parse_csv(path)
    assert len(rows) == 1 and rows[0][1] == 1 << 24 and rows[0][3] > 0 and rows[0][6] >= 0
