"""GPU parity for the five kernels through the C-ABI (libgk.so).

Re-points the reference's own contract tests (pkg/tests/test_kernels.py) at the
B200 package and adds golden-vector and oracle comparisons on identical seeded
inputs.  Tolerances are the reference's (test_kernels.py:32-36): 1e-13 for
stream/field/per-slice nonlinear, 1e-12 for collision and bracket-vs-oracle,
exact for shear, zero-field, self-bracket and determinism.
"""
import numpy as np
import pytest
import torch

from conftest import rel_err
from paper_2305_10553_b200 import _lib
from oracle import direct, port
from paper_2305_10553_b200.grid import GridShape, make_case, random_state, substream
from paper_2305_10553_b200.kernels import (DEFAULT_STENCIL, KERNEL_NAMES, VARIANTS, KernelTiming, checksum,
                                           collision_kernel, field_kernel, make_kernel_inputs,
                                           nonlinear_kernel, run_kernel, shear_kernel, stream_kernel,
                                           time_kernel)
from paper_2305_10553_b200.spectral import bracket, bracket_plans, is_hermitian, random_spectrum

pytestmark = pytest.mark.gpu

SMALL = GridShape(n_radial=12, n_toroidal=4, n_theta=5, n_xi=3, n_energy=2, n_species=2)
C1 = GridShape(16, 8, 8, 8, 4, 2)


def seeded(shape, seed):
    return random_state(shape, seed), make_kernel_inputs(shape, seed)


# ---------------------------------------------------------------- golden vectors (reference outputs)

def test_golden_small_all_kernels(golden):
    h, inp = seeded(SMALL, 21)
    assert rel_err(field_kernel(h, inp["weights"]), golden["small_field"]) < 1e-13
    # original variant reproduces the reference's rounding sequence exactly
    assert np.array_equal(stream_kernel(h, inp["stencil"], "original"), golden["small_stream_original"])
    assert rel_err(stream_kernel(h, inp["stencil"], "optimized"), golden["small_stream_optimized"]) < 1e-13
    assert np.array_equal(shear_kernel(h, inp["shifts"]), golden["small_shear"])
    assert rel_err(collision_kernel(h, inp["matrices"]), golden["small_collision"]) < 1e-12
    assert rel_err(nonlinear_kernel(h, inp["phi"], inp["plans"]), golden["small_nonlinear"]) < 1e-13


def test_golden_c1(golden):
    h, inp = seeded(C1, 7)
    assert rel_err(field_kernel(h, inp["weights"]), golden["c1_field"]) < 1e-13
    assert rel_err(collision_kernel(h, inp["matrices"]), golden["c1_collision"]) < 1e-12
    got = nonlinear_kernel(h, inp["phi"], inp["plans"])
    # per-slice tolerance as in the reference's nonlinear checks
    want = golden["c1_nonlinear"]
    worst = max(rel_err(got[idx], want[idx]) for idx in np.ndindex(C1.dims[:4]))
    assert worst < 1e-13


# ---------------------------------------------------------------- field

def test_field_uniform_weights_sum_velocity_space():
    out = field_kernel(np.ones(SMALL.dims, dtype=complex), np.ones(SMALL.dims[:3]))
    assert out.shape == SMALL.dims[3:] and np.all(out == SMALL.velocity_size)


def test_field_zero_weights():
    h, inp = seeded(SMALL, 3)
    assert np.all(field_kernel(h, np.zeros_like(inp["weights"])) == 0.0)


def test_field_matches_loop_oracle():
    for seed in (1, 2, 3):
        h, inp = seeded(SMALL, seed)
        assert rel_err(field_kernel(h, inp["weights"]), direct.field_loop(h, inp["weights"])) < 1e-13


# ---------------------------------------------------------------- stream

@pytest.mark.parametrize("variant", VARIANTS)
def test_stream_identity_stencil(variant):
    h = random_state(SMALL, 4)
    assert np.array_equal(stream_kernel(h, (1.0,), variant), h)


@pytest.mark.parametrize("variant", VARIANTS)
def test_stream_centered_difference_of_constant_is_zero(variant):
    assert np.all(stream_kernel(np.full(SMALL.dims, 2.0 - 1.0j), (-0.5, 0.0, 0.5), variant) == 0.0)


def test_stream_wraps_periodically():
    h = np.zeros(SMALL.dims, dtype=complex)
    h[..., 0, :, :] = 1.0
    out = stream_kernel(h, DEFAULT_STENCIL)
    hit = np.nonzero(np.any(out != 0.0, axis=(0, 1, 2, 4, 5)))[0]
    assert list(hit) == [1, 2, SMALL.n_theta - 2, SMALL.n_theta - 1]


def test_stream_variants_and_oracle_sh03b_desk():
    shape = make_case("sh03b-desk")
    for seed in (1, 2, 3):
        h = random_state(shape, seed)
        a = stream_kernel(h, DEFAULT_STENCIL, "original")
        b = stream_kernel(h, DEFAULT_STENCIL, "optimized")
        assert rel_err(b, a) < 1e-13
        assert np.array_equal(a, port.stream(h, DEFAULT_STENCIL, "original"))
        assert rel_err(b, port.stream(h, DEFAULT_STENCIL, "optimized")) < 1e-13


@pytest.mark.parametrize("width", [3, 7, 9, 11])
def test_stream_other_widths(width):
    shape = GridShape(6, 2, 13, 2, 1, 1)
    h = random_state(shape, 40 + width)
    c = substream(width, 5).uniform(-1, 1, width)
    assert np.array_equal(stream_kernel(h, c, "original"), port.stream(h, c, "original"))
    assert rel_err(stream_kernel(h, c, "optimized"), direct.stream_loop(h, c)) < 1e-13


@pytest.mark.parametrize("width, n_theta", [(33, 40), (41, 41), (65, 67)])
def test_stream_wide_widths(width, n_theta):
    """Any odd width <= n_theta, as the reference accepts (kernels.py:65-68), incl. w == n_theta."""
    shape = GridShape(6, 2, n_theta, 2, 1, 1)
    h = random_state(shape, width)
    c = substream(width, 9).uniform(-1, 1, width)
    assert np.array_equal(stream_kernel(h, c, "original"), port.stream(h, c, "original"))
    assert rel_err(stream_kernel(h, c, "optimized"), direct.stream_loop(h, c)) < 1e-13
    with pytest.raises(ValueError):
        stream_kernel(h, np.ones(n_theta + 2), "original")


# ---------------------------------------------------------------- shear

@pytest.mark.parametrize("variant", VARIANTS)
def test_shear_zero_shift_is_identity(variant):
    h = random_state(SMALL, 7)
    out = shear_kernel(h, np.zeros(SMALL.n_toroidal, dtype=int), variant)
    assert np.array_equal(out, h) and out is not h


@pytest.mark.parametrize("variant", VARIANTS)
def test_shear_full_shift_clears_everything(variant):
    h = random_state(SMALL, 8)
    shifts = np.full(SMALL.n_toroidal, SMALL.n_radial)
    assert np.all(shear_kernel(h, shifts, variant) == 0.0)
    assert np.all(shear_kernel(h, -shifts, variant) == 0.0)


def test_shear_gathers_with_zero_fill():
    h = random_state(SMALL, 9)
    out = shear_kernel(h, np.array([2, -1, 0, 3]))
    n = SMALL.n_radial
    assert np.array_equal(out[..., 0, : n - 2], h[..., 0, 2:]) and np.all(out[..., 0, n - 2:] == 0.0)
    assert np.array_equal(out[..., 1, 1:], h[..., 1, : n - 1]) and np.all(out[..., 1, :1] == 0.0)


def test_shear_variants_agree_bitwise():
    shape = make_case("sh03b-desk")
    for seed in (1, 2, 3):
        h, inp = seeded(shape, seed)
        a = shear_kernel(h, inp["shifts"], "original")
        assert np.array_equal(a, shear_kernel(h, inp["shifts"], "optimized"))
        assert np.array_equal(a, direct.shear_loop(h, inp["shifts"]))


# ---------------------------------------------------------------- collision

@pytest.fixture
def coll_mode():
    """Switch the collision arithmetic (gk_collision_mode) for one test, then restore it."""
    lib = _lib.load()
    prev = lib.gk_collision_mode(-1)
    yield lib
    lib.gk_collision_mode(prev)


def test_collision_identity_and_zero(coll_mode):
    coll_mode.gk_collision_mode(1)  # fp64 DMMA: identity is exact
    h = random_state(SMALL, 11)
    m = SMALL.velocity_size
    eye = np.broadcast_to(np.eye(m), (SMALL.n_theta, m, m)).copy()
    assert np.array_equal(collision_kernel(h, eye), h)
    assert np.all(collision_kernel(h, np.zeros((SMALL.n_theta, m, m))) == 0.0)


def test_collision_matches_loop_oracle():
    for seed in (1, 2):
        h, inp = seeded(SMALL, seed)
        assert rel_err(collision_kernel(h, inp["matrices"]), direct.collision_loop(h, inp["matrices"])) < 1e-12


@pytest.mark.parametrize("dims", [(48, 8, 8, 6, 4, 3), (96, 16, 6, 6, 4, 3), (10, 3, 3, 5, 7, 1),
                                  (33, 2, 4, 9, 8, 3),
                                  # M % 16 == 0: the pipelined v2 DGEMM (M = 576 sh03b, 432 em04b, 48, 64)
                                  (8, 2, 2, 24, 8, 3), (10, 3, 2, 18, 8, 3), (12, 2, 3, 4, 4, 3),
                                  (200, 3, 2, 8, 4, 2)])
def test_collision_shapes_vs_port(dims):
    shape = GridShape(*dims)
    h, inp = seeded(shape, 5)
    assert rel_err(collision_kernel(h, inp["matrices"]), port.collision(h, inp["matrices"])) < 1e-12


# int8 tensor-core path (collision_i8.cu): fp64 GEMM as exact int8 slice products.
# Same tolerance as the reference's collision checks (1e-12); measured ~5e-14.

@pytest.mark.parametrize("dims", [(48, 8, 8, 6, 4, 3), (10, 3, 3, 5, 7, 1), (33, 2, 4, 9, 8, 3),
                                  (12, 2, 3, 4, 4, 3), (200, 3, 2, 8, 4, 2), (480, 48, 2, 2, 1, 1),
                                  # large M: 4, 2 and 1 column pairs per slicing CTA, warp-padded CTAs
                                  (6, 5, 1, 20, 8, 5), (4, 3, 2, 30, 8, 7), (2, 3, 1, 25, 10, 13)])
def test_collision_int8_slices_vs_port(dims, coll_mode):
    coll_mode.gk_collision_mode(2)
    shape = GridShape(*dims)
    h, inp = seeded(shape, 5)
    assert rel_err(collision_kernel(h, inp["matrices"]), port.collision(h, inp["matrices"])) < 1e-12


def test_collision_int8_identity_zero_determinism(coll_mode):
    coll_mode.gk_collision_mode(2)
    shape = GridShape(64, 8, 3, 8, 4, 2)  # M = 64, N = 1024 reals
    h = random_state(shape, 11)
    m = shape.velocity_size
    eye = np.broadcast_to(np.eye(m), (shape.n_theta, m, m)).copy()
    # sparse rows cannot be certified from the magnitude product (the dropped slice
    # pairs are bounded per nonzero): such tiles come back recomputed in fp64
    assert rel_err(collision_kernel(h, eye), h) < 1e-13
    assert np.all(collision_kernel(h, np.zeros((shape.n_theta, m, m))) == 0.0)
    A = make_kernel_inputs(shape, 3)["matrices"]
    assert np.array_equal(collision_kernel(h, A), collision_kernel(h, A))


def test_collision_int8_wide_dynamic_range(coll_mode):
    """Rows of A over 16 decades, columns of h over 10: per-row/column power-of-two
    scales keep the error relative to the result."""
    shape = GridShape(100, 10, 3, 4, 4, 4)
    h, inp = seeded(shape, 9)
    m = shape.velocity_size
    A = inp["matrices"] * np.logspace(-8, 8, m)[None, :, None]
    h = h * np.logspace(-5, 5, shape.n_radial * shape.n_toroidal).reshape(1, 1, 1, 1, shape.n_toroidal, -1)
    coll_mode.gk_collision_mode(2)
    got = collision_kernel(h, A)
    assert rel_err(got, port.collision(h, A)) < 1e-12


def test_collision_int8_propagates_non_finite(coll_mode):
    """A NaN/Inf in a column of h or a row of A poisons that output column / row,
    as a GEMM does (the slicing scales must not silently drop it)."""
    shape = GridShape(40, 3, 2, 4, 4, 4)
    h, inp = seeded(shape, 4)
    A = inp["matrices"].copy()
    h = h.copy()
    h.reshape(shape.velocity_size, shape.n_theta, -1)[5, 1, 7] = np.nan
    A[0, 3, 9] = np.inf
    coll_mode.gk_collision_mode(2)
    got = collision_kernel(h, A).reshape(shape.velocity_size, shape.n_theta, -1)
    assert np.all(np.isnan(got[:, 1, 7]))                     # column of h with the NaN
    assert not np.any(np.isfinite(got[3, 0, :]))             # row of A with the Inf
    ok = np.ones(got.shape, bool)
    ok[:, 1, 7] = False
    ok[3, 0, :] = False
    assert np.all(np.isfinite(got[ok]))


def _fixups(lib):
    import ctypes as C
    v = C.c_int64()
    assert lib.gk_collision_fixups(C.byref(v)) == 0
    return v.value


def _componentwise_bound_ok(got, h, A, tau=2.0 ** -37):
    """|C - A B| <= tau * |A| |B| elementwise (the int8 path's certificate), with
    the exact product taken in extended precision."""
    m = h.shape[0] * h.shape[1] * h.shape[2]
    T = h.shape[3]
    B = h.reshape(m, T, -1)
    C = got.reshape(m, T, -1)
    for t in range(T):
        Al = A[t].astype(np.longdouble)
        for part in (np.real, np.imag):
            Bt = part(B[:, t]).astype(np.longdouble)
            exact = Al @ Bt
            P = np.abs(Al) @ np.abs(Bt)
            err = np.abs(part(C[:, t]).astype(np.longdouble) - exact)
            if not np.all(err <= tau * P + 1e-300):
                return False
    return True


@pytest.mark.parametrize("kind", ["graded_h_banded_A", "inversely_graded"])
def test_collision_int8_graded_velocity_axis_is_certified(coll_mode, kind):
    """grading along the K (velocity) axis -- h spanning 12 decades over
    velocity, A banded or inversely graded -- breaks the int8 slicing's normwise
    accuracy (rows off by 1e-3 relative).  The certificate (magnitude-slice product
    Q) must flag those tiles and the fp64 recompute must fix them: componentwise
    error <= 2^-37 sum_k |A_ik||B_kj|, and tiles were recomputed."""
    shape = GridShape(40, 4, 2, 16, 8, 1)  # M = 128, N = 320 reals, T = 2
    m = shape.velocity_size
    h, inp = seeded(shape, 21)
    grade = np.logspace(0, -12, m)
    h = h * grade.reshape(1, 8, 16, 1, 1, 1)  # velocity index = (energy, xi) flattened, C order
    rng = np.random.default_rng(4)
    if kind == "graded_h_banded_A":
        A = np.zeros((shape.n_theta, m, m))
        for d in range(-3, 4):
            idx = np.arange(max(0, -d), min(m, m - d))
            A[:, idx, idx + d] = rng.uniform(-1, 1, (shape.n_theta, idx.size))
    else:
        A = rng.uniform(-1, 1, (shape.n_theta, m, m)) / grade[None, None, :]
    coll_mode.gk_collision_mode(2)
    n0 = _fixups(coll_mode)
    got = collision_kernel(h, A)
    assert _fixups(coll_mode) > n0
    assert _componentwise_bound_ok(got, h, A)
    # and the rows of small magnitude are right relative to themselves
    want = port.collision(h, A).reshape(m, shape.n_theta, -1)
    g = got.reshape(m, shape.n_theta, -1)
    row_err = np.max(np.abs(g - want), axis=(1, 2)) / np.max(np.abs(want), axis=(1, 2))
    assert np.max(row_err) < 1e-10


@pytest.mark.parametrize("zeros", [False, True])
def test_collision_int8_certificate_passes_regular_data(coll_mode, zeros):
    """On the benchmark's kind of data (U[-1,1] state and matrices) every tile
    certifies: no fp64 recompute, and the bound holds -- also with the exact-zero
    columns a step's shear leaves at the radial edges and a zero row of A (the
    bound counts only nonzero products, so zeros cost nothing)."""
    coll_mode.gk_collision_mode(2)
    shape = GridShape(480, 4, 2, 8, 8, 2)  # M = 128
    h, inp = seeded(shape, 8)
    A = inp["matrices"].copy()
    if zeros:
        h = shear_kernel(h, np.array([3, -2, 0, 1]))  # zero-filled radial edges
        A[1, 17, :] = 0.0
    n0 = _fixups(coll_mode)
    got = collision_kernel(h, A)
    assert _fixups(coll_mode) == n0
    assert _componentwise_bound_ok(got, h, A)
    if zeros:
        assert np.all(got[..., 0, -3:] == 0.0) and np.all(got.reshape(128, 2, -1)[17, 1] == 0.0)


def test_collision_auto_mode_uses_int8_at_benchmark_width(coll_mode):
    shape = GridShape(480, 48, 6, 4, 4, 4)  # M = 64, N = 46080 (sh03b's width), M^2 N T >= 2^30
    h, inp = seeded(shape, 2)
    coll_mode.gk_collision_mode(0)
    auto = collision_kernel(h, inp["matrices"])
    coll_mode.gk_collision_mode(2)
    assert np.array_equal(auto, collision_kernel(h, inp["matrices"]))
    coll_mode.gk_collision_mode(1)
    assert rel_err(auto, collision_kernel(h, inp["matrices"])) < 1e-12


def test_collision_auto_mode_keeps_dmma_for_tiny_gemms(coll_mode):
    """Below 2^30 multiply-adds (C1-sized) the fp64 DMMA path is faster and exact
    for the identity: auto must pick it."""
    coll_mode.gk_collision_mode(0)
    h = random_state(C1, 3)
    m = C1.velocity_size
    eye = np.broadcast_to(np.eye(m), (C1.n_theta, m, m)).copy()
    assert np.array_equal(collision_kernel(h, eye), h)


def test_int8_peak_probe(coll_mode):
    import ctypes as C
    v = C.c_double()
    assert coll_mode.gk_probe_i8_peak(C.byref(v)) == 0
    assert 1000.0 < v.value < 6000.0  # dense int8 TOPS on one B200 (nominal 4500)


# ---------------------------------------------------------------- nonlinear

def test_nonlinear_zero_field_moment():
    h, inp = seeded(SMALL, 14)
    assert np.all(nonlinear_kernel(h, np.zeros_like(inp["phi"]), inp["plans"]) == 0.0)


def test_nonlinear_state_equal_to_moment_vanishes():
    _, inp = seeded(SMALL, 15)
    h = np.broadcast_to(inp["phi"], SMALL.dims).copy()
    assert np.all(nonlinear_kernel(h, inp["phi"], inp["plans"]) == 0.0)


def test_nonlinear_is_per_slice_bracket():
    shape = GridShape(16, 8, 2, 2, 1, 1)
    h, inp = seeded(shape, 17)
    out = nonlinear_kernel(h, inp["phi"], inp["plans"])
    for idx in np.ndindex(shape.dims[:3]):
        for t in range(shape.n_theta):
            want = bracket(h[idx][t], inp["phi"][t], *inp["plans"])
            assert rel_err(out[idx][t], want) < 1e-13


def test_nonlinear_slice_matches_convolution_oracle():
    shape = GridShape(16, 8, 2, 1, 1, 1)
    gen = substream(18, 0)
    h = np.zeros(shape.dims, dtype=complex)
    for t in range(shape.n_theta):
        h[0, 0, 0, t] = random_spectrum(16, 8, gen)
    phi = np.stack([random_spectrum(16, 8, gen) for _ in range(shape.n_theta)])
    out = nonlinear_kernel(h, phi, bracket_plans(16, 8))
    for t in range(shape.n_theta):
        assert rel_err(out[0, 0, 0, t], direct.bracket_convolution(h[0, 0, 0, t], phi[t])) < 1e-12


def test_nonlinear_thread_count_does_not_change_results():
    h, inp = seeded(SMALL, 19)
    one = nonlinear_kernel(h, inp["phi"], inp["plans"], threads=1)
    assert np.array_equal(one, nonlinear_kernel(h, inp["phi"], inp["plans"], threads=4))


def test_nonlinear_preserves_representability():
    shape = GridShape(8, 4, 2, 2, 1, 1)
    gen = substream(20, 0)
    h = np.zeros(shape.dims, dtype=complex)
    for idx in np.ndindex(shape.dims[:4]):
        h[idx] = random_spectrum(8, 4, gen)
    phi = np.stack([random_spectrum(8, 4, gen) for _ in range(shape.n_theta)])
    out = nonlinear_kernel(h, phi, bracket_plans(8, 4))
    for idx in np.ndindex(shape.dims[:4]):
        assert is_hermitian(out[idx]) and np.all(out[idx][:, 4] == 0.0)


@pytest.mark.parametrize("case", ["sh03b-desk", "em04b-desk"])
def test_nonlinear_desk_cases_vs_port(case):
    shape = make_case(case)
    h, inp = seeded(shape, 1234)
    nx, ny = (p.n_padded for p in inp["plans"])
    got = nonlinear_kernel(h, inp["phi"], inp["plans"])
    want = port.nonlinear(h, inp["phi"], nx, ny)
    worst = max(rel_err(got[idx], want[idx]) for idx in np.ndindex(shape.dims[:4]))
    assert worst < 1e-13


# ---------------------------------------------------------------- shared contracts

@pytest.mark.parametrize("kernel", ["field", "stream", "shear", "collision"])
def test_linear_kernels_are_linear(kernel):
    f, inp = seeded(SMALL, 21)
    g = random_state(SMALL, 22)
    lhs = run_kernel(kernel, 2.0 * f - 0.5j * g, inp)
    rhs = 2.0 * run_kernel(kernel, f, inp) - 0.5j * run_kernel(kernel, g, inp)
    assert rel_err(lhs, rhs) < 1e-12


def test_single_implementation_kernels_agree_across_variants():
    h, inp = seeded(SMALL, 33)
    for kernel in ("field", "collision", "nonlinear"):
        assert np.array_equal(run_kernel(kernel, h, inp, "original"), run_kernel(kernel, h, inp, "optimized"))


def test_kernel_names_cover_dispatch():
    h, inp = seeded(SMALL, 34)
    for kernel in KERNEL_NAMES:
        out = run_kernel(kernel, h, inp)
        assert out.shape == (SMALL.dims[3:] if kernel == "field" else SMALL.dims)


def test_time_kernel_contract():
    t = time_kernel("shear", "optimized", SMALL, reps=3, seed=7)
    assert isinstance(t, KernelTiming) and t.reps == 3 and t.median_s >= t.min_s > 0.0
    h, inp = seeded(SMALL, 7)
    assert t.checksum == checksum(run_kernel("shear", h, inp, "optimized"))
    assert time_kernel("shear", "optimized", SMALL, reps=4, seed=7).checksum == t.checksum


def test_kernel_checksums_deterministic():
    """cli.py:750-762: bitwise run-to-run identity and cross-variant identity."""
    shape = make_case("sh03b-desk")
    for kernel in KERNEL_NAMES:
        a = time_kernel(kernel, "optimized", shape, 3, 1234)
        h, inp = seeded(shape, 1234)
        assert a.checksum == checksum(run_kernel(kernel, h, inp, "optimized"))
        if kernel != "stream":
            assert time_kernel(kernel, "original", shape, 3, 1234).checksum == a.checksum


def test_device_tensors_stay_on_device():
    h, inp = seeded(SMALL, 35)
    ht = torch.from_numpy(h).cuda()
    out = run_kernel("collision", ht, inp)
    assert isinstance(out, torch.Tensor) and out.is_cuda
    assert np.array_equal(out.cpu().numpy(), collision_kernel(h, inp["matrices"]))


@pytest.mark.parametrize("dims", [(480, 48, 3, 1, 1, 2),     # sh03b slices: 720 x 144 plan
                                  (1344, 288, 2, 1, 1, 1),   # em04b slices: 2016 x 864 plan
                                  (1344, 160, 2, 1, 1, 1),   # C5a slices: 2016 x 480 plan
                                  # y plans of the rectangular YCOL below their n_ky maximum
                                  # (empty bins inside the staged slots, fewer kept outputs)
                                  (480, 159, 2, 1, 1, 1),    # 720 x 480, n_ky 159 < 160
                                  (480, 287, 1, 1, 1, 1)])   # 720 x 864, n_ky 287 < 288
def test_nonlinear_benchmark_slice_shapes_vs_port(dims):
    """The compile-time-specialised FFT path (fixed radices) against the oracle."""
    shape = GridShape(*dims)
    h, inp = seeded(shape, 99)
    nx, ny = (p.n_padded for p in inp["plans"])
    got = nonlinear_kernel(h, inp["phi"], inp["plans"])
    want = port.nonlinear(h, inp["phi"], nx, ny)
    worst = max(rel_err(got[idx], want[idx]) for idx in np.ndindex(shape.dims[:4]))
    assert worst < 1e-13
    # exact-zero contract on the fixed path: every slice equal to phi[theta]
    hz = np.broadcast_to(inp["phi"], shape.dims).copy()
    assert np.all(nonlinear_kernel(hz, inp["phi"], inp["plans"]) == 0.0)


@pytest.mark.parametrize("dist", ["gauss", "lognormal"])
def test_collision_int8_certificate_passes_heavy_tailed_data(coll_mode, dist):
    """Gaussian operands (row and column maxima several times the typical entry)
    still certify -- the dropped-pair bound uses the digits' actual magnitudes;
    log-normal ones (maxima ~30x the typical entry) may fall back on some tiles.
    Either way the componentwise bound holds."""
    coll_mode.gk_collision_mode(2)
    shape = GridShape(480, 4, 2, 8, 8, 2)  # M = 128
    rng = np.random.default_rng(17)
    if dist == "gauss":
        h = rng.normal(size=shape.dims) + 1j * rng.normal(size=shape.dims)
        A = rng.normal(size=(shape.n_theta, 128, 128))
    else:
        h = rng.lognormal(0, 1, shape.dims) * np.sign(rng.normal(size=shape.dims)) + 1j * rng.normal(size=shape.dims)
        A = rng.lognormal(0, 1, (shape.n_theta, 128, 128)) * np.sign(rng.normal(size=(shape.n_theta, 128, 128)))
    n0 = _fixups(coll_mode)
    got = collision_kernel(h, A)
    if dist == "gauss":
        assert _fixups(coll_mode) == n0
    assert _componentwise_bound_ok(got, h, A)


@pytest.mark.parametrize("k", [-600, 400, -985, 1008])
def test_collision_int8_power_of_two_scaling_is_exact(k, coll_mode):
    """collision(2^k h) == 2^k collision(h) bit for bit: the epilogue's exponent-add
    fast scaling (moderate scales) and its general path (k = -985 / 1008 push the
    output exponents out of the fast range) both apply the power-of-two scales
    exactly."""
    coll_mode.gk_collision_mode(2)
    shape = GridShape(48, 10, 2, 6, 4, 2)  # M = 48, 960 reals per theta
    h, inp = seeded(shape, 23)
    A = inp["matrices"]
    base = collision_kernel(h, A)
    got = collision_kernel(h * np.ldexp(1.0, k), A)
    assert np.array_equal(got, base * np.ldexp(1.0, k))


def test_collision_int8_cta_pair_is_bit_identical(tmp_path, coll_mode):
    """GK_I8_PAIR=1 runs the GEMM as tcgen05 cta_group::2 MMAs (CTA pairs, stage
    copies through tensor maps completing on the leader's barrier): same slices,
    same integer sums, so the same bits as the one-CTA kernel -- including an odd
    number of column blocks (the pair's spare block) and certificate fallbacks."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    coll_mode.gk_collision_mode(2)
    shapes = [(480, 48, 2, 4, 4, 2), (40, 20, 3, 4, 4, 2)]  # 46080 reals (even ncb); 1600 reals: 13 blocks
    for n, dims in enumerate(shapes):
        shape = GridShape(*dims)
        h, inp = seeded(shape, 31 + n)
        np.save(tmp_path / f"h{n}.npy", h)
        np.save(tmp_path / f"a{n}.npy", inp["matrices"])
    script = f"""
import sys, numpy as np
sys.path.insert(0, {str(root)!r})
from paper_2305_10553_b200 import _lib
from paper_2305_10553_b200.kernels import collision_kernel
_lib.load().gk_collision_mode(2)
for n in range({len(shapes)}):
    h = np.load({str(tmp_path)!r} + f"/h{{n}}.npy"); A = np.load({str(tmp_path)!r} + f"/a{{n}}.npy")
    np.save({str(tmp_path)!r} + f"/c{{n}}.npy", collision_kernel(h, A))
    if n == 1:
        np.save({str(tmp_path)!r} + "/g.npy", collision_kernel(h, A * np.logspace(-6, 6, A.shape[1])[None, :, None]))
"""
    res = subprocess.run([sys.executable, "-c", script], env=dict(os.environ, GK_I8_PAIR="1"),
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    for n in range(len(shapes)):
        h, A = np.load(tmp_path / f"h{n}.npy"), np.load(tmp_path / f"a{n}.npy")
        assert np.array_equal(np.load(tmp_path / f"c{n}.npy"), collision_kernel(h, A)), n
    h, A = np.load(tmp_path / "h1.npy"), np.load(tmp_path / "a1.npy")
    graded = A * np.logspace(-6, 6, A.shape[1])[None, :, None]  # graded rows: some tiles recomputed
    assert np.array_equal(np.load(tmp_path / "g.npy"), collision_kernel(h, graded))


def test_pipelined_b_slicing_is_bit_identical(tmp_path, coll_mode):
    """GK_SB_PIPE=1 (the warp-specialised, tensor-copy-pipelined B slicing) gives
    slice_b's bits: collision outputs (slices, certificate stats) at awkward shapes
    and the step's h' and phi (the fused field moment)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    from paper_2305_10553_b200.step import Stepper
    root = Path(__file__).resolve().parents[1]
    coll_mode.gk_collision_mode(2)
    shapes = [(40, 20, 3, 4, 4, 2), (33, 7, 2, 9, 8, 3), (480, 48, 3, 8, 8, 1)]
    for n, dims in enumerate(shapes):
        shape = GridShape(*dims)
        h, inp = seeded(shape, 61 + n)
        np.save(tmp_path / f"h{n}.npy", h)
        np.save(tmp_path / f"a{n}.npy", inp["matrices"])
    step_shape = GridShape(480, 48, 8, 8, 8, 1)
    script = f"""
import sys, numpy as np
sys.path.insert(0, {str(root)!r})
from paper_2305_10553_b200 import _lib
from paper_2305_10553_b200.grid import GridShape, random_state
from paper_2305_10553_b200.kernels import collision_kernel, make_kernel_inputs
from paper_2305_10553_b200.step import Stepper
_lib.load().gk_collision_mode(2)
d = {str(tmp_path)!r}
for n in range({len(shapes)}):
    np.save(d + f"/c{{n}}.npy", collision_kernel(np.load(d + f"/h{{n}}.npy"), np.load(d + f"/a{{n}}.npy")))
shape = GridShape(480, 48, 8, 8, 8, 1)
st = Stepper(shape, make_kernel_inputs(shape, 67), 1e-4)
np.save(d + "/s.npy", st.run(random_state(shape, 67), 1))
np.save(d + "/phi.npy", st.phi.cpu().numpy())
"""
    res = subprocess.run([sys.executable, "-c", script], env=dict(os.environ, GK_SB_PIPE="1"),
                         capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    for n in range(len(shapes)):
        h, A = np.load(tmp_path / f"h{n}.npy"), np.load(tmp_path / f"a{n}.npy")
        assert np.array_equal(np.load(tmp_path / f"c{n}.npy"), collision_kernel(h, A)), n
    st = Stepper(step_shape, make_kernel_inputs(step_shape, 67), 1e-4)
    want = st.run(random_state(step_shape, 67), 1)
    assert np.array_equal(np.load(tmp_path / "s.npy"), want)
    assert np.array_equal(np.load(tmp_path / "phi.npy"), st.phi.cpu().numpy())


def test_collision_int8_uncertified_tiles_get_dmma_bits(coll_mode):
    """When every tile fails the certificate (h graded over 12 decades in velocity
    and A graded inversely, so the products are of equal size), the recompute runs
    the DMMA collision's 64 x 128 tile: the int8 path then returns the DMMA path's
    bits exactly."""
    import ctypes
    shape = GridShape(128, 8, 4, 8, 4, 2)  # M = 64, 2048 reals per theta
    h, inp = seeded(shape, 71)
    m = shape.velocity_size
    h = h * np.logspace(-6, 6, m).reshape(shape.n_species, shape.n_energy, shape.n_xi, 1, 1, 1)
    A = inp["matrices"] * np.logspace(6, -6, m)[None, None, :]
    lib = coll_mode
    n0, n1 = ctypes.c_int64(0), ctypes.c_int64(0)
    lib.gk_collision_mode(2)
    lib.gk_collision_fixups(ctypes.byref(n0))
    got = collision_kernel(h, A)
    lib.gk_collision_fixups(ctypes.byref(n1))
    assert n1.value > n0.value  # tiles were recomputed
    lib.gk_collision_mode(1)
    assert np.array_equal(got, collision_kernel(h, A))
