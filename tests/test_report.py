"""Reference-format bench reports and compare."""
import csv

import pytest

from conftest import GOLDEN
from paper_2305_10553_b200.report import BENCH_COLUMNS, Report, ReportError, compare, main, read_bench_medians

REF_BENCH = GOLDEN / "reference_bench_sh03b_desk.csv"


def test_reads_the_reference_bench_report():
    med = read_bench_medians(str(REF_BENCH))
    assert set(med) == {("sh03b-desk", k) for k in ("field", "stream", "shear", "collision", "nonlinear")}
    assert all(v > 0 for v in med.values())


def test_compare_ratios_and_overall(tmp_path):
    before = {("c", "a"): 2.0, ("c", "b"): 6.0}
    after = {("c", "a"): 1.0, ("c", "b"): 2.0}
    rep = compare(before, after)
    rows = {(r[0], r[1]): float(r[4]) for r in rep.rows}
    assert rows[("c", "a")] == 2.0 and rows[("c", "b")] == 3.0 and rows[("all", "overall")] == 8.0 / 3.0
    with pytest.raises(ReportError):
        compare(before, {("c", "a"): 1.0})


def test_report_csv_and_atomic_write(tmp_path):
    rep = Report(BENCH_COLUMNS, [("x", "field", "optimized", 3, "1.0", "0.5", "abc", "dev")], {"tool": "t"})
    path = tmp_path / "r.csv"
    rep.write(str(path))
    text = path.read_text()
    assert text.startswith("# tool=t\n")
    rows = list(csv.DictReader(line for line in text.splitlines() if not line.startswith("#")))
    assert rows[0]["kernel"] == "field" and rows[0]["median_s"] == "1.0"
    assert [p.name for p in tmp_path.iterdir()] == ["r.csv"]  # no temp file left behind
    assert read_bench_medians(str(path)) == {("x", "field"): 1.0}


def test_cli_compare_rejects_non_reports(tmp_path, capsys):
    bad = tmp_path / "bad.csv"
    bad.write_text("a,b\n1,2\n")
    assert main(["compare", "--before", str(bad), "--after", str(REF_BENCH)]) == 2


@pytest.mark.gpu
def test_gpu_bench_report_checksums_match_reference_bitwise_kernels(tmp_path):
    """Bench rows carry output checksums: shear and stream 'original' are
    bitwise-equal to the reference, so their checksums equal the reference CLI's."""
    from paper_2305_10553_b200.report import bench_report
    rep = bench_report("sh03b-desk", ["stream", "shear"], ("original",), reps=3, seed=1234)
    ours = {r[1]: r[6] for r in rep.rows}
    with open(REF_BENCH) as fh:
        ref = {r["kernel"]: r["checksum"] for r in csv.DictReader(ln for ln in fh if not ln.startswith("#"))}
    assert ours["shear"] == ref["shear"]
    assert ours["stream"] == ref["stream"]
    path = tmp_path / "gpu.csv"
    rep.write(str(path))
    assert set(read_bench_medians(str(path))) == {("sh03b-desk", "stream"), ("sh03b-desk", "shear")}


@pytest.mark.gpu
def test_gpu_fft_bench_prime_size_elimination():
    """test_acceptance.py:88-99 on the device: 720 (2^4 3^2 5) beats 719 (prime)."""
    from paper_2305_10553_b200.report import fft_bench_report
    rep = fft_bench_report((719, 720), batch=256, reps=5)
    rows = {r[0]: r for r in rep.rows}
    assert rows[719][1] == "719" and rows[720][1] == "2*2*2*2*3*3*5"
    assert float(rows[720][2]) <= float(rows[719][2])


def test_verify_host_checks_and_exit_code(monkeypatch, capsys):
    """`verify` mirrors the reference's (cli.py:535-776): one row per check, exit 3
    when any check fails (cli.py:75), a crashing check counts as failed."""
    from paper_2305_10553_b200 import report
    host = ["padding_minimal", "padding_overhead", "padding_examples", "factorize_product"]
    rep, code = report.verify_report("sh03b-desk", 1234, host)
    assert code == 0 and [r[0] for r in rep.rows] == host and all(r[2] == "pass" for r in rep.rows)
    assert rep.columns == ("check", "case", "status", "value", "seconds")

    def boom(case, seed):
        raise RuntimeError("no device")

    monkeypatch.setattr(report, "VERIFY_CHECKS", report.VERIFY_CHECKS + (("always_fails", lambda c, s: (False, "x")),
                                                                        ("crashes", boom)))
    rep, code = report.verify_report("sh03b-desk", 1234, host + ["always_fails", "crashes"])
    assert code == report.EXIT_VERIFY == 3
    assert [r[2] for r in rep.rows[-2:]] == ["fail", "fail"] and "RuntimeError" in rep.rows[-1][3]
    assert main(["verify", "--checks", "padding_examples"]) == 0
    assert "padding_examples" in capsys.readouterr().out


@pytest.mark.gpu
def test_gpu_verify_all_checks_pass():
    from paper_2305_10553_b200.report import VERIFY_CHECKS, verify_report
    rep, code = verify_report("sh03b-desk", 1234)
    assert code == 0, [r for r in rep.rows if r[2] != "pass"]
    assert len(rep.rows) == len(VERIFY_CHECKS)
