"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports gyroproxy from /root/reference/pkg/src (read-only, unmodified),
runs the reference's own functions on seeded inputs and writes their outputs
to tests/golden/*.npz / *.json.  These fixtures pin both the CPU oracle
(oracle/) and the CUDA path; nothing at test time reads /root/reference.
"""

from __future__ import annotations

import csv
import json
import shutil
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent

C1 = (16, 8, 8, 8, 4, 2)
SMALL = (12, 4, 5, 3, 2, 2)
STEP_DT = 1e-3
STEP_N = 10


def main():
    sys.path.insert(0, str(REF))
    from gyroproxy import grid, kernels, padding, spectral

    out = {}

    # --- kernels on SMALL (every kernel, both stream variants) and on C1
    for tag, dims, seed in (("small", SMALL, 21), ("c1", C1, 7)):
        shape = grid.GridShape(*dims)
        h = grid.random_state(shape, seed)
        inp = kernels.make_kernel_inputs(shape, seed)
        out[f"{tag}_field"] = kernels.field_kernel(h, inp["weights"])
        out[f"{tag}_nonlinear"] = kernels.nonlinear_kernel(h, inp["phi"], inp["plans"])
        out[f"{tag}_collision"] = kernels.collision_kernel(h, inp["matrices"])
        if tag == "small":
            out[f"{tag}_stream_original"] = kernels.stream_kernel(h, inp["stencil"], "original")
            out[f"{tag}_stream_optimized"] = kernels.stream_kernel(h, inp["stencil"], "optimized")
            out[f"{tag}_shear"] = kernels.shear_kernel(h, inp["shifts"])
            out[f"{tag}_h_head"] = h.reshape(-1)[:64]
            out[f"{tag}_shifts"] = np.asarray(inp["shifts"])
        else:
            out[f"{tag}_h_head"] = h.reshape(-1)[:64]
            # builder-defined step composed from reference functions only
            x = h.copy()
            for _ in range(STEP_N):
                phi = kernels.field_kernel(x, inp["weights"])
                rhs = (kernels.stream_kernel(x, inp["stencil"])
                       + kernels.nonlinear_kernel(x, phi, inp["plans"])
                       + kernels.collision_kernel(x, inp["matrices"]))
                x = kernels.shear_kernel(x + STEP_DT * rhs, inp["shifts"])
            out[f"{tag}_step{STEP_N}"] = x

    # --- bracket on random representable spectra (spectral tests' grids)
    for n_kx, n_ky in ((8, 4), (7, 3), (16, 8)):
        plans = spectral.bracket_plans(n_kx, n_ky)
        for seed in (1, 2, 3):
            gen = grid.substream(seed, 0)
            f = spectral.random_spectrum(n_kx, n_ky, gen)
            g = spectral.random_spectrum(n_kx, n_ky, gen)
            key = f"br_{n_kx}x{n_ky}_s{seed}"
            out[key + "_f"], out[key + "_g"] = f, g
            out[key + "_out"] = spectral.bracket(f, g, *plans)
    gen = grid.substream(24, 0)
    f = spectral.random_spectrum(8, 4, gen)
    g = spectral.random_spectrum(8, 4, gen)
    out["br_loose_f"], out["br_loose_g"] = f, g
    out["br_loose_out"] = spectral.bracket(f, g, 32, 30)
    # non-representable (raw random) input: the c2r projection must match too
    gen = grid.substream(77, 0)
    f = gen.uniform(-1, 1, (5, 10)) + 1j * gen.uniform(-1, 1, (5, 10))
    g = gen.uniform(-1, 1, (5, 10)) + 1j * gen.uniform(-1, 1, (5, 10))
    out["br_raw_f"], out["br_raw_g"] = f, g
    out["br_raw_out"] = spectral.bracket(f, g, *spectral.bracket_plans(10, 5))

    # --- standalone transforms
    gen = grid.substream(31, 0)
    spec = gen.uniform(-1, 1, (2, 3, 8)) + 1j * gen.uniform(-1, 1, (2, 3, 8))
    out["tr_spec"] = spec
    out["tr_real_12x9"] = spectral.to_real(spec, 12, 9)
    out["tr_real_8x4"] = spectral.to_real(spec, 8, 4)  # same-size x, Nyquist row in y
    field = gen.uniform(-1, 1, (2, 10, 9))
    out["tr_field"] = field
    out["tr_spec_9x6"] = spectral.to_spectrum(field, 9, 6)
    out["tr_spec_8x4"] = spectral.to_spectrum(field, 8, 4)

    np.savez_compressed(HERE / "reference_outputs.npz", **out)

    # --- integer tables: plans, kx tables
    tables = {
        "plan_padded": [padding.plan_padded_size(n).n_padded for n in range(1, 4097)],
        "naive_padded": [padding.naive_padded_size(n) for n in range(1, 513)],
        "factorize_720": padding.factorize(720),
        "kx_values": {str(n): spectral.kx_values(n).tolist() for n in range(1, 21)},
        "kx_derivative_values": {str(n): spectral.kx_derivative_values(n).tolist() for n in range(1, 21)},
        "bracket_plans": {f"{a},{b}": [p.n_padded for p in spectral.bracket_plans(a, b)]
                          for a, b in ((16, 8), (480, 48), (1344, 288), (1344, 160), (2688, 576),
                                       (48, 8), (96, 16), (12, 4), (8, 4), (7, 3))},
        "shifts_small_21": [int(s) for s in kernels.make_kernel_inputs(grid.GridShape(*SMALL), 21)["shifts"]],
        "step": {"dt": STEP_DT, "n": STEP_N, "dims": C1, "seed": 7},
    }
    (HERE / "reference_tables.json").write_text(json.dumps(tables, indent=0))

    # a bench report written by the reference's own CLI (format + checksums; the
    # timings are this container's and only serve as a compare() input)
    from gyroproxy.cli import RunConfig, run
    rep, code = run(RunConfig(command="bench", case="sh03b-desk", kernels=kernels.KERNEL_NAMES,
                              variants=("original",), reps=3, seed=1234))
    assert code == 0
    rep.write(str(HERE / "reference_bench_sh03b_desk.csv"))

    # the reference's own RNG golden statistics (data file, pkg/tests/data)
    shutil.copyfile(REF.parent / "tests" / "data" / "generator_stats.csv", HERE / "generator_stats.csv")
    with open(HERE / "generator_stats.csv", newline="") as fh:
        assert len(list(csv.DictReader(fh))) == 9
    print("wrote", sorted(p.name for p in HERE.iterdir()))


if __name__ == "__main__":
    main()
