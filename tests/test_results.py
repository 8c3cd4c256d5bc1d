"""The bench reporting format: ResultRow and its CSV /
JSON writers byte for byte like proj/src/bench.cpp:222-263, and (gpu) the
ADR integrator order study of bench.cpp:131-179 on the device."""
import json
import math

import pytest

import paper_2509_26475_b200 as P
from paper_2509_26475_b200 import results as R


def rows():
    a = R.make_row("adr", "grid=50", 0.000244140625, 1.25e-9, 0.5,
                   P.RunRecord(3, 41, [], 1234), math.nan)
    b = R.make_row("gallery", "zero_8", 1.0, 0.0, 1e-05, P.RunRecord(1, 2, [5, 6], 7), 1e-12)
    b.order = 4.0
    c = R.make_row("x", "big", 2.0, 3e-11, 0.25, P.RunRecord(), 1e-12)
    return [a, b, c]


def test_make_row_ok_rule():
    a, b, c = rows()
    assert a.ok and b.ok and not c.ok          # NaN bound never fails; error > bound fails
    assert b.sweeps == 2 and b.matvecs == 7 and b.s_effective == 1


def test_csv_format():
    txt = R.rows_to_csv(rows())
    lines = txt.splitlines()
    assert lines[0] == ("experiment,label,t,error,order,seconds,s_eff,series_len_S,sweeps,"
                        "matvecs,bound,ok")
    # ostream precision(17): %.17g, nan for unset order / bound
    assert lines[1] == ("adr,grid=50,0.000244140625,1.25e-09,nan,0.5,3,41,0,1234,"
                        "nan,1")
    assert lines[2] == "gallery,zero_8,1,0,4,1.0000000000000001e-05,1,2,2,7,9.9999999999999998e-13,1"
    assert lines[3].endswith(",0") and txt.endswith("\n")


def test_json_format():
    txt = R.rows_to_json(rows())
    arr = json.loads(txt)
    assert "order" not in arr[0] and "bound" not in arr[0]   # non-finite fields omitted
    assert arr[1]["order"] == 4.0 and arr[1]["bound"] == 1e-12
    # nlohmann::json objects are std::map: keys in sorted order
    assert list(arr[1].keys()) == sorted(arr[1].keys())
    assert txt.startswith('[\n  {\n    "error": 1.25e-09,') and txt.endswith("]\n")


def test_write_rows(tmp_path):
    cfg = R.BenchConfig(out_path=str(tmp_path / "r.json"), format="json")
    R.write_rows(rows(), cfg)
    assert (tmp_path / "r.json").read_text() == R.rows_to_json(rows())
    cfg = R.BenchConfig(out_path=str(tmp_path / "r.csv"))
    R.write_rows(rows(), cfg)
    assert (tmp_path / "r.csv").read_text() == R.rows_to_csv(rows())
    assert not R.all_within_bounds(rows())


@pytest.mark.gpu
def test_adr_order_study_on_device():
    """bench.cpp:131-179 at a reduced grid: observed order >= 3.5 on every
    refinement row (the rows' ok), as the reference's acceptance run."""
    out = R.run_adr(R.BenchConfig(adr_nx=24, adr_ny=24))
    assert len(out) == 4
    for r in out[1:]:
        assert r.order >= 3.5 and r.ok, R.rows_to_csv(out)
    assert all(r.matvecs > 0 and r.s_effective >= 1 for r in out)


def test_reference_writer_checks(tmp_path):  # test_bench.cpp:42-73
    row = R.ResultRow(experiment="gallery", label="identity_10", t=1.0, error=1e-16,
                      seconds=0.01, s_effective=1, series_len_S=7, sweeps=0, matvecs=42,
                      bound=1e-13)
    csv = R.rows_to_csv([row])
    assert csv.startswith("experiment,label,t,error") and "identity_10" in csv
    assert '"matvecs": 42' in R.rows_to_json([row])
    cfg = R.BenchConfig(out_path=str(tmp_path / "bench_rows_test.csv"), format="csv")
    R.write_rows([row], cfg)
    assert (tmp_path / "bench_rows_test.csv").read_text() == csv

