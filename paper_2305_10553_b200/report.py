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
    python -m paper_2305_10553_b200.report verify --case sh03b-desk   # exit 3 on a failed check

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


# ------------------------------------------------------------------ verify
# The reference's `gyroproxy verify` (cli.py:535-776) runs 19 named checks and
# exits 3 when one fails.  Here the hot-path checks run on the GPU kernels as
# self-consistency checks between independent paths (int8-slice vs fp64 DMMA
# collision, pipelined host-buffer step vs the monolithic step, per-slice bracket
# vs the batched nonlinear term, device vs host generator, ...) plus the host-side
# planner/generator checks.  Comparisons against the reference's CPU oracles live
# with the tests (tools/verify_oracle.py): the product package never imports them.

EXIT_VERIFY = 3
VERIFY_COLUMNS = ("check", "case", "status", "value", "seconds")


def _max_rel(got, want) -> float:
    import numpy as np

    got, want = np.asarray(got), np.asarray(want)
    scale = float(np.max(np.abs(want))) if want.size else 0.0
    diff = float(np.max(np.abs(got - want))) if want.size else 0.0
    return diff if scale == 0.0 else diff / scale


def _v_padding_minimal(case, seed):
    """Planner == smallest 7-smooth size >= ceil(3n/2), found independently."""
    from .padding import plan_padded_size

    def smooth(m):
        for p in (2, 3, 5, 7):
            while m % p == 0:
                m //= p
        return m == 1

    bad = 0
    for n in range(1, 769):
        m = (3 * n + 1) // 2
        while not smooth(m):
            m += 1
        bad += plan_padded_size(n).n_padded != m
    return bad == 0, str(bad)


def _v_padding_overhead(case, seed):
    from .padding import plan_padded_size

    worst = max(p.n_padded / p.n_min for p in map(plan_padded_size, range(8, 4097)))
    return worst <= 1.25, repr(worst)


def _v_padding_examples(case, seed):
    from .padding import cost_score, factorize, naive_padded_size, plan_padded_size

    ok = (plan_padded_size(48).n_padded == 72 and plan_padded_size(479).n_padded == 720
          and naive_padded_size(477) == 716 and factorize(716) == [2, 2, 179]
          and plan_padded_size(477).n_padded == 720 and cost_score([2, 2, 2, 3, 3]) == 12)
    return ok, "5 cases"


def _v_factorize(case, seed):
    import math

    from .grid import substream
    from .padding import factorize

    for n in map(int, substream(seed, 5).integers(1, 10**6, 200)):
        f = factorize(n)
        if math.prod(f) != n or any(p < 2 or any(p % d == 0 for d in range(2, math.isqrt(p) + 1)) for p in f):
            return False, str(n)
    return True, "200 values"


def _v_rng_device(case, seed):
    import numpy as np

    from .grid import component_mean_abs, make_case, random_state, random_state_device

    shape = make_case(case)
    d1 = random_state_device(shape, seed).cpu().numpy()
    if not np.array_equal(d1, random_state_device(shape, seed).cpu().numpy()):
        return False, "nondeterministic"
    if not np.array_equal(d1, random_state(shape, seed)):
        return False, "device generator != host generator"
    peak = max(float(np.max(np.abs(d1.real))), float(np.max(np.abs(d1.imag))))
    mean_abs = component_mean_abs(d1)
    return peak <= 1.0 and 0.3 < mean_abs < 0.7, repr(mean_abs)


def _v_roundtrip(case, seed):
    from .grid import substream
    from .spectral import to_real, to_spectrum

    n, worst = 72, 0.0
    for k in range(3):
        x = substream(seed + k, 5).uniform(-1.0, 1.0, (n, n))
        worst = max(worst, _max_rel(to_real(to_spectrum(x, n, n // 2 + 1), n, n), x))
    return worst <= 1e-12, repr(worst)


def _v_parseval(case, seed):
    import numpy as np

    from .grid import substream
    from .spectral import to_spectrum

    n, worst = 72, 0.0
    for k in range(3):
        x = substream(seed + k, 5).uniform(-1.0, 1.0, (n, n))
        spec = to_spectrum(x, n, n // 2 + 1)
        w = np.full(spec.shape[0], 2.0)
        w[0] = w[-1] = 1.0  # ky = 0 and the unpaired Nyquist row count once
        power = float(w @ np.sum(np.abs(spec) ** 2, axis=1))
        ref = float(np.mean(x**2))
        worst = max(worst, abs(power - ref) / ref)
    return worst <= 1e-12, repr(worst)


def _v_bracket_self(case, seed):
    import numpy as np

    from .grid import substream
    from .spectral import bracket, bracket_plans, random_spectrum

    worst = 0.0
    for k in range(3):
        f = random_spectrum(8, 4, substream(seed + k, 5))
        worst = max(worst, float(np.max(np.abs(bracket(f, f, *bracket_plans(8, 4))))))
    return worst == 0.0, repr(worst)


def _v_bracket_antisymmetry(case, seed):
    import numpy as np

    from .grid import substream
    from .spectral import bracket, bracket_plans, random_spectrum

    for n_kx, n_ky in ((8, 4), (7, 3), (16, 8)):
        gen = substream(seed, 5)
        f, g = random_spectrum(n_kx, n_ky, gen), random_spectrum(n_kx, n_ky, gen)
        p = bracket_plans(n_kx, n_ky)
        if not np.array_equal(bracket(f, g, *p), -bracket(g, f, *p)):
            return False, f"{n_kx}x{n_ky}"
    return True, "exact"


def _case_inputs(case, seed):
    from .grid import make_case, random_state
    from .kernels import make_kernel_inputs

    shape = make_case(case)
    return shape, random_state(shape, seed), make_kernel_inputs(shape, seed)


def _v_stream_variants(case, seed):
    from .kernels import stream_kernel

    worst = 0.0
    for k in range(3):
        _, h, inp = _case_inputs(case, seed + k)
        worst = max(worst, _max_rel(stream_kernel(h, inp["stencil"], "optimized"),
                                    stream_kernel(h, inp["stencil"], "original")))
    return worst <= 1e-13, repr(worst)


def _v_shear_variants(case, seed):
    import numpy as np

    from .kernels import shear_kernel

    for k in range(3):
        _, h, inp = _case_inputs(case, seed + k)
        a = shear_kernel(h, inp["shifts"], "optimized")
        if not np.array_equal(a, shear_kernel(h, inp["shifts"], "original")):
            return False, "variants differ"
        s = np.asarray(inp["shifts"])
        # shift each ky row back: every value that stayed in range returns bitwise
        back = shear_kernel(a, -s, "optimized")
        R = h.shape[-1]
        keep = np.array([[0 <= kx - sy < R for kx in range(R)] for sy in s])
        if not np.array_equal(back[..., keep], h[..., keep]):
            return False, "inverse shift"
    return True, "0.0"


def _v_collision_modes(case, seed):
    from . import _lib
    from .kernels import collision_kernel

    _, h, inp = _case_inputs(case, seed)
    lib = _lib.load()
    prev = lib.gk_collision_mode(-1)
    try:
        lib.gk_collision_mode(1)
        dmma = collision_kernel(h, inp["matrices"])
        lib.gk_collision_mode(2)
        i8 = collision_kernel(h, inp["matrices"])
    finally:
        lib.gk_collision_mode(prev)
    err = _max_rel(i8, dmma)
    return err <= 1e-12, repr(err)


def _v_nonlinear_slices(case, seed):
    import numpy as np

    from .kernels import nonlinear_kernel
    from .spectral import bracket

    shape, h, inp = _case_inputs(case, seed)
    got = nonlinear_kernel(h, inp["phi"], inp["plans"])
    if not np.array_equal(got, nonlinear_kernel(h, inp["phi"], inp["plans"], threads=2)):
        return False, "thread count changed values"
    want = np.empty_like(h)
    for idx in np.ndindex(*shape.dims[:3]):
        want[idx] = bracket(h[idx], inp["phi"], *inp["plans"])
    err = _max_rel(got, want)
    return err <= 1e-13, repr(err)


def _v_step_host_pipeline(case, seed):
    import numpy as np
    import torch

    from .step import Stepper

    shape, h, inp = _case_inputs(case, seed)
    st = Stepper(shape, inp, dt=1e-3)
    dev = torch.device("cuda", torch.cuda.current_device())
    hd = torch.from_numpy(h).to(dev)
    want = st.step(hd).cpu().numpy()
    h_host = torch.from_numpy(h).pin_memory()
    o_host = torch.empty_like(h_host).pin_memory()
    chunks = max(1, min(4, shape.n_theta // 2))
    st.step_host(h_host, o_host, torch.empty_like(hd), torch.empty_like(hd), chunks=chunks)
    torch.cuda.synchronize()
    return bool(np.array_equal(o_host.numpy(), want)), f"{chunks} chunks, bitwise"


def _v_kernel_checksums(case, seed):
    from .grid import make_case
    from .kernels import KERNEL_NAMES, checksum, run_kernel, time_kernel

    shape, h, inp = _case_inputs(case, seed)
    for kernel in KERNEL_NAMES:
        t = time_kernel(kernel, "optimized", make_case(case), 3, seed)
        if t.checksum != checksum(run_kernel(kernel, h, inp, "optimized")):
            return False, kernel
    return True, f"{len(KERNEL_NAMES)} kernels"


VERIFY_CHECKS = (
    ("padding_minimal", _v_padding_minimal),
    ("padding_overhead", _v_padding_overhead),
    ("padding_examples", _v_padding_examples),
    ("factorize_product", _v_factorize),
    ("rng_device_vs_host", _v_rng_device),
    ("transform_roundtrip", _v_roundtrip),
    ("transform_parseval", _v_parseval),
    ("bracket_self_zero", _v_bracket_self),
    ("bracket_antisymmetry", _v_bracket_antisymmetry),
    ("stream_variants", _v_stream_variants),
    ("shear_variants", _v_shear_variants),
    ("collision_int8_vs_fp64", _v_collision_modes),
    ("nonlinear_slices", _v_nonlinear_slices),
    ("step_host_pipeline", _v_step_host_pipeline),
    ("kernel_checksums", _v_kernel_checksums),
)


def verify_report(case: str = "sh03b-desk", seed: int = 1234, checks=None) -> tuple:
    """Run the checks; returns (Report, exit code 0 or EXIT_VERIFY)."""
    import time

    rows, failures = [], 0
    for name, fn in VERIFY_CHECKS:
        if checks and name not in checks:
            continue
        t0 = time.perf_counter()
        try:
            ok, value = fn(case, seed)
        except Exception as e:  # a crashing check is a failed check, reported as such
            ok, value = False, f"{type(e).__name__}: {e}"
        failures += 0 if ok else 1
        rows.append((name, case, "pass" if ok else "fail", value, f"{time.perf_counter() - t0:.6f}"))
    return Report(VERIFY_COLUMNS, rows, _meta("verify", case=case, seed=seed, checks=len(rows))), \
        (EXIT_VERIFY if failures else 0)


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
    v = sub.add_parser("verify")
    v.add_argument("--case", default="sh03b-desk")
    v.add_argument("--seed", type=int, default=1234)
    v.add_argument("--checks", default=None, help="comma list (default: all)")
    v.add_argument("--out")
    c = sub.add_parser("compare")
    c.add_argument("--before", required=True)
    c.add_argument("--after", required=True)
    c.add_argument("--out")
    a = ap.parse_args(argv)
    try:
        if a.cmd == "bench":
            rep = bench_report(a.case, a.kernels.split(",") if a.kernels else None, tuple(a.variants.split(",")),
                               a.reps, a.seed)
        elif a.cmd == "verify":
            rep, code = verify_report(a.case, a.seed, a.checks.split(",") if a.checks else None)
            if a.out:
                rep.write(a.out)
            print(rep.plain())
            return code
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
