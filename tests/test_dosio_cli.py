"""dosio formats, the CLI and the scaling harness.

Modelled on the reference's tests/test_dosio.py, test_cli.py and
test_bench.py.  The CPU tests use golden tables (no enumeration); the
`gpu` tests run the commands that enumerate or evaluate thermodynamics.
"""

import subprocess
import sys

import numpy as np
import pytest

import paper_1110_2561_b200 as isd
from paper_1110_2561_b200 import bench as bench_mod
from paper_1110_2561_b200.cli import main
from paper_1110_2561_b200.dosio import parse_dos_csv, parse_dos_json
from paper_1110_2561_b200.workloads import workloads
from golden_io import GOLDEN, read_csv_table, read_json_table

ROOT = __import__("os").path.dirname(GOLDEN.rstrip("/").rsplit("/", 1)[0])


def _dos(name):
    rows, cols, depth, j, table = read_csv_table(name)
    return isd.DoSHistogram(isd.LatticeSpec(rows, cols, depth, j), table)


@pytest.fixture
def dos4x4():
    return _dos("dos_4x4x1_J1.csv")


@pytest.fixture
def dos2x2():
    return _dos("dos_2x2x1_J1.csv")


# -- dosio (CPU) ---------------------------------------------------------------

def test_csv_is_byte_identical_to_reference_files():
    # the goldens were written by the reference's write_dos
    for name in ("dos_4x4x1_J1.csv", "dos_3x3x1_Jm2.csv", "dos_3x4x1_J0p5.csv",
                 "dos_2x2x3_J1.csv"):
        text = open(f"{GOLDEN}/{name}").read()
        assert isd.format_dos_csv(isd.parse_dos(text)) == text


def test_csv_header(dos2x2):
    lines = isd.format_dos_csv(dos2x2).splitlines()
    assert lines[0] == "# rows=2 cols=2 depth=1 J=1 N=4 B=8 version=1"
    assert lines[1] == "count,M,E"


def test_round_trips(tmp_path, dos4x4):
    assert parse_dos_csv(isd.format_dos_csv(dos4x4)) == dos4x4
    assert parse_dos_json(isd.format_dos_json(dos4x4)) == dos4x4
    assert isd.parse_dos(isd.format_dos_json(dos4x4)) == dos4x4
    p = tmp_path / "d.csv"
    isd.write_dos(dos4x4, str(p))
    assert isd.read_dos(str(p)) == dos4x4
    p = tmp_path / "d.json"
    isd.write_dos(dos4x4, str(p), as_json=True)
    assert isd.read_dos(str(p)) == dos4x4


@pytest.mark.parametrize("fname,name", [("c1_4x4_free.json", "c1"),
                                        ("c4_6x6_pmJ_seed1234.json", "c4"),
                                        ("c3_6x6_free.json", "c3")])
def test_extended_lattices_round_trip(fname, name):
    _, table = read_json_table(fname)
    spec = workloads()[name].spec
    dos = isd.DoSHistogram(spec, table)
    text = isd.format_dos_csv(dos)
    assert "version=2" in text.splitlines()[0]
    back = isd.parse_dos(text)
    assert back == dos and back.spec == spec
    assert isd.parse_dos(isd.format_dos_json(dos)) == dos


def _lines(dos):
    return isd.format_dos_csv(dos).splitlines()


def test_parse_errors_carry_lines(dos2x2):
    with pytest.raises(isd.DosFileError) as err:
        parse_dos_csv("\n".join(_lines(dos2x2)[1:]))
    assert err.value.line == 1
    lines = _lines(dos2x2)
    lines[0] = lines[0].replace("version=1", "version=9")
    with pytest.raises(isd.DosFileError, match="version"):
        parse_dos_csv("\n".join(lines))
    lines = _lines(dos2x2)
    lines[0] = lines[0].replace("B=8", "B=10")
    with pytest.raises(isd.DosFileError, match="B=10"):
        parse_dos_csv("\n".join(lines))
    lines = _lines(dos2x2)
    lines[3] = "x,2,0"
    with pytest.raises(isd.DosFileError) as err:
        parse_dos_csv("\n".join(lines))
    assert err.value.line == 4
    lines = _lines(dos2x2)
    lines.append(lines[2])
    with pytest.raises(isd.DosFileError, match="duplicate"):
        parse_dos_csv("\n".join(lines))
    lines = _lines(dos2x2)
    lines[2] = "1,4,-7"
    with pytest.raises(isd.DosFileError, match="grid"):
        parse_dos_csv("\n".join(lines))


def test_extended_header_validation(dos2x2):
    spec = isd.LatticeSpec(2, 2, bond_signs=(1, -1) * 4)
    text = isd.format_dos_csv(isd.DoSHistogram(spec, dos2x2.counts))
    bad = text.replace("signs=+-+-+-+-", "signs=+-+")
    with pytest.raises(isd.DosFileError, match="bond_signs"):
        parse_dos_csv(bad)
    bad = text.replace("signs=+-+-+-+-", "signs=+x+-+-+-")
    with pytest.raises(isd.DosFileError, match="signs"):
        parse_dos_csv(bad)


# -- CLI (CPU paths) -------------------------------------------------------------

def test_cli_verify_pass_and_fail(tmp_path, capsys, dos4x4):
    good = tmp_path / "g.csv"
    isd.write_dos(dos4x4, str(good))
    assert main(["verify", str(good)]) == 0
    assert "PASS total-count" in capsys.readouterr().out
    bad = dos4x4.counts.copy()
    bad[8, 16] += 1
    badp = tmp_path / "b.csv"
    isd.write_dos(isd.DoSHistogram(dos4x4.spec, bad), str(badp))
    assert main(["verify", str(badp)]) == 1
    err = capsys.readouterr().err
    assert err.startswith("error: check-failed: total-count,binomial-marginals")


def test_cli_validation_and_io_errors(tmp_path, capsys):
    assert main(["dos", "--rows", "1", "--cols", "5", "--out", "-"]) == 1
    assert "error: validation: degenerate periodic axis" in capsys.readouterr().err
    assert main(["dos", "--rows", "5", "--cols", "9", "--out", "-"]) == 1
    assert "cap of 40" in capsys.readouterr().err
    assert main(["verify", str(tmp_path / "missing.csv")]) == 3
    assert "error: io:" in capsys.readouterr().err
    p = tmp_path / "junk.csv"
    p.write_text("garbage\n")
    assert main(["verify", str(p)]) == 1
    assert "error: parse: line 1" in capsys.readouterr().err
    with pytest.raises(SystemExit) as exc:
        main(["dos", "--rows", "2"])
    assert exc.value.code == 2


def test_cli_thermo_rejects_bad_grid(tmp_path, capsys, dos2x2):
    p = tmp_path / "d.csv"
    isd.write_dos(dos2x2, str(p))
    assert main(["thermo", str(p), "--tmin", "1", "--tmax", "2",
                 "--tstep", "0"]) == 1
    assert "tstep" in capsys.readouterr().err
    assert main(["thermo", str(p), "--tmin", "3", "--tmax", "2"]) == 1
    assert "tmax" in capsys.readouterr().err


def test_scaling_report_round_trip():
    rec = [bench_mod.BenchRecord(isd.LatticeSpec(4, 4), w, 0.5 / w, [0.1] * w,
                                 float(w)) for w in (1, 2, 4)]
    text = bench_mod.emit_scaling_report(rec)
    rows = bench_mod.parse_scaling_report(text)
    assert [r["workers"] for r in rows] == [1, 2, 4]
    assert rows[2]["wall_seconds"] == 0.125 and rows[2]["speedup"] == 4.0
    with pytest.raises(ValueError):
        bench_mod.parse_scaling_report("nope\n")
    with pytest.raises(ValueError):
        bench_mod.run_bench(isd.LatticeSpec(2, 2), [])
    with pytest.raises(ValueError):
        bench_mod.run_bench(isd.LatticeSpec(2, 2), [0])


def test_run_bench_detects_mismatch(monkeypatch, dos2x2):
    # the harness must refuse a corrupted run (test_bench.py:47-61)
    calls = {"n": 0}

    def fake(spec, workers=None):
        calls["n"] += 1
        counts = dos2x2.counts.copy()
        if calls["n"] > 1:
            counts[2, 4] += 1
        return isd.DoSHistogram(spec, counts), 0.01, [0.01] * (workers or 1)

    monkeypatch.setattr(bench_mod, "full_dos_timed", fake)
    with pytest.raises(isd.ResultMismatchError):
        bench_mod.run_bench(isd.LatticeSpec(2, 2), [1, 2], repeats=1)


# -- GPU: commands that enumerate / evaluate -------------------------------------

@pytest.mark.gpu
def test_cli_dos_and_thermo(tmp_path, capsys):
    out = tmp_path / "dos.csv"
    assert main(["dos", "--rows", "3", "--cols", "3", "--workers", "2",
                 "--out", str(out)]) == 0
    assert "N=9 spins, B=18 bonds, 512 configurations" in capsys.readouterr().out
    assert isd.read_dos(str(out)) == _dos("dos_3x3x1_J1.csv")
    assert main(["dos", "--rows", "2", "--cols", "2", "--out", "-"]) == 0
    cap = capsys.readouterr()
    assert "configurations" in cap.err
    assert isd.parse_dos(cap.out) == _dos("dos_2x2x1_J1.csv")
    assert main(["thermo", str(out), "--tmin", "0.5", "--tmax", "2.5",
                 "--tstep", "0.5", "--field", "0.2"]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert lines[0] == "T,h,log_Z,F,U,C,M_mean,chi" and len(lines) == 6
    free = tmp_path / "free.csv"
    assert main(["dos", "--rows", "4", "--cols", "4", "--boundary", "free",
                 "--out", str(free)]) == 0
    _, want = read_json_table("c1_4x4_free.json")
    assert np.array_equal(isd.read_dos(str(free)).counts, want)


@pytest.mark.gpu
def test_run_bench_on_gpu():
    recs = bench_mod.run_bench(isd.LatticeSpec(5, 5), [1, 2, 4], repeats=2)
    assert [r.num_workers for r in recs] == [1, 2, 4]
    assert all(r.wall_seconds > 0 and r.configs_per_second > 0 for r in recs)
    assert all(len(r.per_worker_seconds) == r.num_workers for r in recs)


@pytest.mark.gpu
def test_run_bench_extended_record_and_report(tmp_path, capsys):
    spec = isd.LatticeSpec(3, 3, 4)  # c5: the hoisted kernel's roofline
    recs = bench_mod.run_bench(spec, [1, 2], repeats=1, roofline=True)
    for r in recs:
        assert r.num_gpus == 1
        assert 0.3 < r.roofline_fraction < 1.05, r.roofline_fraction
        assert 500 < r.sm_clock_mhz < 3000
    rows = bench_mod.parse_scaling_report(bench_mod.emit_extended_report(recs))
    assert [row["workers"] for row in rows] == [1, 2]
    assert rows[0]["roofline_fraction"] == recs[0].roofline_fraction
    # the CLI flag
    assert main(["bench", "--rows", "3", "--cols", "3", "--workers", "1,2",
                 "--repeats", "1", "--extended"]) == 0
    out = capsys.readouterr().out
    assert out.splitlines()[0] == bench_mod.EXTENDED_HEADER


def test_extended_report_round_trip_without_gpu():
    spec = isd.LatticeSpec(2, 2)
    recs = [bench_mod.BenchRecord(spec, 1, 0.5, [0.5], 1.0, 32.0, 1, 0.9,
                                  1965.0),
            bench_mod.BenchRecord(spec, 2, 0.25, [0.2, 0.25], 2.0, 64.0, 1)]
    text = bench_mod.emit_extended_report(recs)
    assert text.splitlines()[0] == (
        "rows,cols,depth,N,workers,wall_seconds,speedup,"
        "gpus,configs_per_second,roofline_fraction,sm_mhz")
    rows = bench_mod.parse_scaling_report(text)
    assert rows[0]["roofline_fraction"] == 0.9 and rows[0]["sm_mhz"] == 1965.0
    assert rows[1]["roofline_fraction"] is None and rows[1]["sm_mhz"] is None
    # the reference report is unchanged
    assert bench_mod.emit_scaling_report(recs).splitlines()[0] == \
        bench_mod.REPORT_HEADER


@pytest.mark.gpu
def test_console_module_runs(tmp_path):
    out = tmp_path / "d.csv"
    r = subprocess.run([sys.executable, "-m", "paper_1110_2561_b200.cli", "dos",
                        "--rows", "2", "--cols", "3", "--out", str(out)],
                       capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    assert isd.read_dos(str(out)) == _dos("dos_2x3x1_J1.csv")
