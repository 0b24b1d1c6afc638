"""The oracle half of the reference's `verify` (cli.py:621-704): GPU kernels vs the
reference's transform-free CPU oracles restated in oracle/direct.py.  Test
infrastructure (imports oracle/); the product-side checks are
`python -m paper_2305_10553_b200.report verify`.

    python tools/verify_oracle.py [--case sh03b-desk] [--seed 1234]    # exit 3 on a failure
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import direct  # noqa: E402
from paper_2305_10553_b200.grid import make_case, random_state, substream  # noqa: E402
from paper_2305_10553_b200.kernels import make_kernel_inputs, run_kernel, stream_kernel, shear_kernel  # noqa: E402
from paper_2305_10553_b200.report import EXIT_VERIFY, VERIFY_COLUMNS, Report, _max_rel, _meta  # noqa: E402
from paper_2305_10553_b200.spectral import bracket, bracket_plans, random_spectrum  # noqa: E402


def field_oracle(case, seed):
    shape = make_case(case)
    h, inp = random_state(shape, seed), make_kernel_inputs(shape, seed)
    err = _max_rel(run_kernel("field", h, inp), direct.field_loop(h, inp["weights"]))
    return err <= 1e-13, repr(err)


def stream_oracle(case, seed):
    shape, worst = make_case(case), 0.0
    for k in range(3):
        h, inp = random_state(shape, seed + k), make_kernel_inputs(shape, seed + k)
        worst = max(worst, _max_rel(stream_kernel(h, inp["stencil"]), direct.stream_loop(h, inp["stencil"])))
    return worst <= 1e-13, repr(worst)


def shear_oracle(case, seed):
    shape = make_case(case)
    for k in range(3):
        h, inp = random_state(shape, seed + k), make_kernel_inputs(shape, seed + k)
        if not np.array_equal(shear_kernel(h, inp["shifts"]), direct.shear_loop(h, inp["shifts"])):
            return False, "oracle differs"
    return True, "0.0"


def collision_oracle(case, seed):
    shape = make_case(case)
    h, inp = random_state(shape, seed), make_kernel_inputs(shape, seed)
    err = _max_rel(run_kernel("collision", h, inp), direct.collision_loop(h, inp["matrices"]))
    return err <= 1e-12, repr(err)


def bracket_oracle(case, seed):
    worst = 0.0
    for n_kx, n_ky in ((8, 4), (7, 3)):
        for k in range(3):
            gen = substream(seed + k, 5)
            f, g = random_spectrum(n_kx, n_ky, gen), random_spectrum(n_kx, n_ky, gen)
            worst = max(worst, _max_rel(bracket(f, g, *bracket_plans(n_kx, n_ky)), direct.bracket_convolution(f, g)))
    return worst <= 1e-12, repr(worst)


CHECKS = (("field_oracle", field_oracle), ("stream_oracle", stream_oracle), ("shear_oracle", shear_oracle),
          ("collision_oracle", collision_oracle), ("bracket_oracle", bracket_oracle))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="sh03b-desk")
    ap.add_argument("--seed", type=int, default=1234)
    a = ap.parse_args()
    rows, fails = [], 0
    for name, fn in CHECKS:
        t0 = time.perf_counter()
        ok, value = fn(a.case, a.seed)
        fails += not ok
        rows.append((name, a.case, "pass" if ok else "fail", value, f"{time.perf_counter() - t0:.6f}"))
    print(Report(VERIFY_COLUMNS, rows, _meta("verify-oracle", case=a.case)).plain())
    return EXIT_VERIFY if fails else 0


if __name__ == "__main__":
    sys.exit(main())
