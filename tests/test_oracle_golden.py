"""Pin the CPU oracle (oracle/) against the reference's own outputs (CPU).

The fixtures were produced by importing the unmodified reference package
(tests/golden/make_golden.py).  The port oracle follows the reference's numpy
calls one for one, so it must agree bitwise; the direct-summation oracles are
independent and agree to the reference's tolerances.
"""
import numpy as np
import pytest

from conftest import rel_err, rel_l2
from oracle import direct, port
from paper_2305_10553_b200.grid import GridShape, random_state
from paper_2305_10553_b200.kernels import make_kernel_inputs

SMALL = (12, 4, 5, 3, 2, 2)
C1 = (16, 8, 8, 8, 4, 2)


@pytest.fixture(scope="module")
def small():
    shape = GridShape(*SMALL)
    return random_state(shape, 21), make_kernel_inputs(shape, 21)


@pytest.fixture(scope="module")
def c1():
    shape = GridShape(*C1)
    return random_state(shape, 7), make_kernel_inputs(shape, 7)


def test_port_kernels_bitwise_small(small, golden):
    h, inp = small
    nx, ny = (p.n_padded for p in inp["plans"])
    assert np.array_equal(port.field(h, inp["weights"]), golden["small_field"])
    assert np.array_equal(port.stream(h, inp["stencil"], "original"), golden["small_stream_original"])
    assert np.array_equal(port.stream(h, inp["stencil"], "optimized"), golden["small_stream_optimized"])
    assert np.array_equal(port.shear(h, inp["shifts"]), golden["small_shear"])
    assert np.array_equal(port.collision(h, inp["matrices"]), golden["small_collision"])
    assert np.array_equal(port.nonlinear(h, inp["phi"], nx, ny), golden["small_nonlinear"])


def test_port_kernels_bitwise_c1(c1, golden):
    h, inp = c1
    nx, ny = (p.n_padded for p in inp["plans"])
    assert np.array_equal(port.field(h, inp["weights"]), golden["c1_field"])
    assert np.array_equal(port.collision(h, inp["matrices"]), golden["c1_collision"])
    assert np.array_equal(port.nonlinear(h, inp["phi"], nx, ny), golden["c1_nonlinear"])


def test_port_step_matches_reference_composition(c1, golden, tables):
    h, inp = c1
    nx, ny = (p.n_padded for p in inp["plans"])
    x = h
    for _ in range(tables["step"]["n"]):
        x, _ = port.step(x, inp["weights"], inp["stencil"], inp["matrices"], inp["shifts"],
                         tables["step"]["dt"], nx, ny)
    assert np.array_equal(x, golden["c1_step10"])


def test_direct_oracles_agree_with_reference(small, golden):
    h, inp = small
    assert rel_err(direct.field_loop(h, inp["weights"]), golden["small_field"]) < 1e-13
    assert rel_err(direct.stream_loop(h, inp["stencil"]), golden["small_stream_original"]) < 1e-13
    assert np.array_equal(direct.shear_loop(h, inp["shifts"]), golden["small_shear"])
    assert rel_err(direct.collision_loop(h, inp["matrices"]), golden["small_collision"]) < 1e-12


@pytest.mark.parametrize("key", ["8x4_s1", "8x4_s2", "7x3_s1", "16x8_s3"])
def test_convolution_oracle_agrees_with_reference_bracket(golden, key):
    f, g = golden[f"br_{key}_f"], golden[f"br_{key}_g"]
    assert rel_err(direct.bracket_convolution(f, g), golden[f"br_{key}_out"]) < 1e-12


def test_port_bracket_and_transforms_bitwise(golden):
    for key in ("8x4_s1", "7x3_s2", "16x8_s3"):
        f, g = golden[f"br_{key}_f"], golden[f"br_{key}_g"]
        ny_, nx_ = f.shape
        nx, ny = port.plan_sizes(nx_, ny_)
        assert np.array_equal(port.poisson_bracket(f, g, nx, ny), golden[f"br_{key}_out"])
    assert np.array_equal(port.poisson_bracket(golden["br_loose_f"], golden["br_loose_g"], 32, 30),
                          golden["br_loose_out"])
    assert np.array_equal(port.synth(golden["tr_spec"], 12, 9), golden["tr_real_12x9"])
    assert np.array_equal(port.analyse(golden["tr_field"], 9, 6), golden["tr_spec_9x6"])


def test_direct_dft_pair():
    gen = np.random.default_rng(0)
    field = gen.uniform(-1, 1, (6, 9))
    assert rel_err(direct.idft2(direct.dft2(field), 6), field) < 1e-13
    spec = direct.random_spectrum(7, 4, gen)
    assert rel_err(port.synth(spec, 7, 6), direct.idft2(spec, 6) * 42) < 1e-13
    assert rel_l2(port.analyse(field, 9, 4), direct.dft2(field)[:4] / 54) < 1e-13
