"""Bench reports in the reference's format.

The reference's ``gyroproxy bench`` writes a CSV with one ``#`` metadata line
and the columns ``case,kernel,variant,reps,median_s,min_s,checksum``
(cli.py:120-178, 413-423); ``gyroproxy compare`` divides the medians of two such
reports per (case, kernel) and adds an overall ratio-of-sums row (cli.py:459-507).
This module produces the same report from the GPU kernels (``time_kernel``
times device-resident calls; checksums are of the outputs, so a GPU report and
a CPU report of the same seed agree wherever the kernels agree bitwise -- shear,
stream "original") and compares a reference CPU report with a GPU one.

    python -m paper_2305_10553_b200.report bench --case sh03b-desk --reps 5 --out gpu.csv
    python -m paper_2305_10553_b200.report compare --before ref_cpu.csv --after gpu.csv
    python -m paper_2305_10553_b200.report fft-bench --sizes 719,720

Extra trailing columns (``device``) do not disturb ``compare``, which reads
columns by name.
"""

from __future__ import annotations

import argparse
import csv
import io
import os
import platform
import sys
import tempfile
from dataclasses import dataclass, field
from datetime import datetime, timezone

from . import __version__

BENCH_COLUMNS = ("case", "kernel", "variant", "reps", "median_s", "min_s", "checksum", "device")


@dataclass
class Report:
    columns: tuple
    rows: list
    meta: dict = field(default_factory=dict)

    def csv_text(self) -> str:
        out = io.StringIO()
        out.write("# " + " ".join(f"{k}={v}" for k, v in self.meta.items()) + "\n")
        w = csv.writer(out, lineterminator="\n")
        w.writerow(self.columns)
        w.writerows(self.rows)
        return out.getvalue()

    def write(self, path: str) -> None:
        """Atomic: temp file in the target directory, then rename."""
        target = os.path.abspath(path)
        fd, tmp = tempfile.mkstemp(dir=os.path.dirname(target), prefix=".gkreport-", suffix=".tmp")
        try:
            with os.fdopen(fd, "w", encoding="utf-8", newline="") as fh:
                fh.write(self.csv_text())
            os.replace(tmp, target)
        except BaseException:
            if os.path.exists(tmp):
                os.unlink(tmp)
            raise

    def plain(self) -> str:
        cells = [tuple(map(str, r)) for r in self.rows]
        width = [max([len(c)] + [len(r[i]) for r in cells]) for i, c in enumerate(self.columns)]
        fmt = lambda r: "  ".join(v.ljust(width[i]) for i, v in enumerate(r)).rstrip()  # noqa: E731
        return "\n".join([fmt(self.columns)] + [fmt(r) for r in cells])


def _meta(command: str, **extra) -> dict:
    meta = {"tool": "paper_2305_10553_b200", "version": __version__, "command": command}
    meta.update(extra)
    meta["timestamp"] = datetime.now(timezone.utc).strftime("%Y-%m-%dT%H:%M:%SZ")
    meta["host"] = f"{platform.node()} {platform.system()} {platform.machine()}"
    return meta


def bench_report(case: str, kernels=None, variants=("optimized",), reps: int = 5, seed: int = 1234) -> Report:
    import torch

    from .grid import make_case
    from .kernels import KERNEL_NAMES, time_kernel

    shape = make_case(case)
    dev = torch.cuda.get_device_name(torch.cuda.current_device())
    rows = []
    for kernel in kernels or KERNEL_NAMES:
        for variant in variants:
            t = time_kernel(kernel, variant, shape, reps, seed)
            rows.append((case, kernel, variant, reps, repr(t.median_s), repr(t.min_s), t.checksum, dev))
    return Report(BENCH_COLUMNS, rows, _meta("bench", case=case, reps=reps, seed=seed))


def fft_bench_report(sizes=(719, 720), batch: int = 256, reps: int = 9, seed: int = 1234) -> Report:
    """GPU analogue of ``gyroproxy fft-bench`` (cli.py:386-410): median/min time of a
    batched complex-to-real inverse transform of each size (substream 5 inputs,
    standard normal), with the size's prime factorisation -- the padding story
    (a 7-smooth 720 vs the prime 719) on the device FFT: smooth sizes run the
    radix kernels, a large prime falls to the generic O(p^2) pass."""
    import statistics
    import time

    import torch

    from .grid import substream
    from .padding import factorize
    from .spectral import to_real

    rows = []
    for n in sizes:
        gen = substream(seed, 5)
        spec = gen.standard_normal((batch, n // 2 + 1)) + 1j * gen.standard_normal((batch, n // 2 + 1))
        dspec = torch.from_numpy(spec.reshape(batch, n // 2 + 1, 1)).cuda()
        to_real(dspec, 1, n)  # warm-up (plan, workspace)
        times = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            to_real(dspec, 1, n)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
        rows.append((n, "*".join(map(str, factorize(n))), repr(statistics.median(times)), repr(min(times))))
    return Report(("size", "factors", "median_seconds", "min_seconds"), rows,
                  _meta("fft-bench", batch=batch, reps=reps, seed=seed))


class ReportError(ValueError):
    pass


def read_bench_medians(path: str) -> dict:
    """(case, kernel) -> median seconds of a bench report (ours or the reference's)."""
    with open(path, encoding="utf-8", newline="") as fh:
        body = [ln for ln in fh if not ln.startswith("#")]
    rd = csv.DictReader(body)
    if rd.fieldnames is None or not {"case", "kernel", "median_s"} <= set(rd.fieldnames):
        raise ReportError(f"{path}: not a bench report (needs case, kernel, median_s)")
    med = {}
    for row in rd:
        key = (row["case"], row["kernel"])
        if key in med:
            raise ReportError(f"{path}: duplicate rows for {key}; one variant per report")
        med[key] = float(row["median_s"])
    if not med:
        raise ReportError(f"{path}: no rows")
    return med


def compare(before: dict, after: dict) -> Report:
    """Per-kernel before/after ratio (before / after = speed-up) and overall ratio of sums."""
    if set(before) != set(after):
        raise ReportError(f"reports cover different (case, kernel) sets: "
                          f"only before {sorted(set(before) - set(after))}, "
                          f"only after {sorted(set(after) - set(before))}")
    rows = [(c, k, repr(before[(c, k)]), repr(after[(c, k)]), repr(before[(c, k)] / after[(c, k)]))
            for c, k in sorted(before)]
    tb, ta = sum(before.values()), sum(after.values())
    rows.append(("all", "overall", repr(tb), repr(ta), repr(tb / ta)))
    return Report(("case", "kernel", "before_s", "after_s", "ratio"), rows, _meta("compare"))


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2305_10553_b200.report")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench")
    b.add_argument("--case", required=True)
    b.add_argument("--kernels", default=None, help="comma list (default: all five)")
    b.add_argument("--variants", default="optimized")
    b.add_argument("--reps", type=int, default=5)
    b.add_argument("--seed", type=int, default=1234)
    b.add_argument("--out")
    f = sub.add_parser("fft-bench")
    f.add_argument("--sizes", default="719,720")
    f.add_argument("--batch", type=int, default=256)
    f.add_argument("--reps", type=int, default=9)
    f.add_argument("--out")
    c = sub.add_parser("compare")
    c.add_argument("--before", required=True)
    c.add_argument("--after", required=True)
    c.add_argument("--out")
    a = ap.parse_args(argv)
    try:
        if a.cmd == "bench":
            rep = bench_report(a.case, a.kernels.split(",") if a.kernels else None, tuple(a.variants.split(",")),
                               a.reps, a.seed)
        elif a.cmd == "fft-bench":
            rep = fft_bench_report(tuple(int(x) for x in a.sizes.split(",")), a.batch, a.reps)
        else:
            rep = compare(read_bench_medians(a.before), read_bench_medians(a.after))
    except (ReportError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    if a.out:
        rep.write(a.out)
    print(rep.plain())
    return 0


if __name__ == "__main__":
    sys.exit(main())
