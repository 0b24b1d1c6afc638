"""GPU parity for the spectral API (to_real / to_spectrum / bracket).

Re-points the reference's pkg/tests/test_spectral.py contracts at the B200
package and compares against reference golden vectors and the transform-free
convolution oracle.
"""
import numpy as np
import pytest

from conftest import rel_err
from oracle import direct, port
from paper_2305_10553_b200.grid import substream
from paper_2305_10553_b200.spectral import (bracket, bracket_plans, hermitian_ky0, is_hermitian,
                                            random_spectrum, to_real, to_spectrum)

pytestmark = pytest.mark.gpu


def test_golden_brackets(golden):
    for key in [k[:-4] for k in golden.files if k.startswith("br_") and k.endswith("_out")]:
        f, g, want = golden[key + "_f"], golden[key + "_g"], golden[key + "_out"]
        n_ky, n_kx = f.shape
        plans = (32, 30) if "loose" in key else bracket_plans(n_kx, n_ky)
        assert rel_err(bracket(f, g, *plans), want) < 1e-13, key


def test_golden_transforms(golden):
    spec, field = golden["tr_spec"], golden["tr_field"]
    assert rel_err(to_real(spec, 12, 9), golden["tr_real_12x9"]) < 1e-13
    assert rel_err(to_real(spec, 8, 4), golden["tr_real_8x4"]) < 1e-13
    assert rel_err(to_spectrum(field, 9, 6), golden["tr_spec_9x6"]) < 1e-13
    assert rel_err(to_spectrum(field, 8, 4), golden["tr_spec_8x4"]) < 1e-13


def test_to_real_zero_spectrum():
    assert np.all(to_real(np.zeros((3, 8), dtype=complex), 12, 12) == 0.0)


@pytest.mark.parametrize("n_x, n_y", [(8, 6), (12, 9), (16, 12)])
def test_to_real_single_mode_amplitude(n_x, n_y):
    spec = np.zeros((3, 8), dtype=complex)
    spec[1, 2] = 1.0
    y, x = np.meshgrid(np.arange(n_y), np.arange(n_x), indexing="ij")
    assert rel_err(to_real(spec, n_x, n_y), 2 * np.cos(2 * np.pi * (2 * x / n_x + y / n_y))) < 1e-13


def test_to_real_matches_oracle_scaled():
    spec = random_spectrum(7, 4, substream(3, 0))
    assert rel_err(to_real(spec, 7, 6), direct.idft2(spec, 6) * 42) < 1e-13


def test_to_spectrum_constant_and_oracle():
    spec = to_spectrum(np.full((9, 12), 1.5), 8, 4)
    assert spec[0, 0] == pytest.approx(1.5)
    spec[0, 0] = 0
    assert np.max(np.abs(spec)) < 1e-14
    field = substream(4, 0).uniform(-1, 1, (10, 9))
    assert rel_err(to_spectrum(field, 9, 6), direct.dft2(field) / 90) < 1e-13


@pytest.mark.parametrize("n_kx, n_ky", [(8, 3), (7, 4), (16, 8), (1, 1), (480, 48)])
def test_transform_roundtrip_padded(n_kx, n_ky):
    spec = random_spectrum(n_kx, n_ky, substream(n_kx * 31 + n_ky, 0))
    px, py = bracket_plans(n_kx, n_ky)
    assert rel_err(to_spectrum(to_real(spec, px.n_padded, py.n_padded), n_kx, n_ky), spec) < 1e-13


def test_transform_roundtrip_same_size_and_batch():
    field = substream(8, 0).uniform(-1, 1, (10, 12))
    assert rel_err(to_real(to_spectrum(field, 12, 6), 12, 10), field) < 1e-13
    spec = np.stack([random_spectrum(8, 3, substream(s, 0)) for s in range(4)]).reshape(2, 2, 3, 8)
    f = to_real(spec, 12, 9)
    assert f.shape == (2, 2, 9, 12)
    assert rel_err(to_spectrum(f, 8, 3), spec) < 1e-13


def test_transforms_match_port_on_raw_batches():
    gen = substream(91, 0)
    spec = gen.uniform(-1, 1, (5, 6, 20)) + 1j * gen.uniform(-1, 1, (5, 6, 20))
    for nx, ny in ((30, 16), (20, 10), (35, 11), (22, 13)):
        assert rel_err(to_real(spec, nx, ny), port.synth(spec, nx, ny)) < 1e-13
        field = gen.uniform(-1, 1, (3, ny, nx))
        assert rel_err(to_spectrum(field, 20, 6), port.analyse(field, 20, 6)) < 1e-13


def test_size_checks_raise():
    spec = np.zeros((3, 8), dtype=complex)
    for args in ((7, 12), (12, 3)):
        with pytest.raises(ValueError):
            to_real(spec, *args)
    with pytest.raises(ValueError):
        to_spectrum(np.zeros((6, 8)), 9, 3)
    with pytest.raises(ValueError):
        to_spectrum(np.zeros((6, 8)), 8, 5)


def test_nyquist_column_dropped_on_size_change():
    spec = np.zeros((3, 8), dtype=complex)
    spec[1, 4] = 1 + 2j
    assert np.max(np.abs(to_real(spec, 12, 9))) == 0.0
    assert np.max(np.abs(to_real(spec, 8, 9))) > 0.1
    out = to_spectrum(substream(6, 0).uniform(-1, 1, (9, 12)), 8, 3)
    assert np.all(out[:, 4] == 0.0)


def test_parseval_and_roundtrip_72():
    n = 72
    w = np.full(n // 2 + 1, 2.0)
    w[0] = w[-1] = 1.0
    for seed in range(10):
        field = substream(2000 + seed, 0).uniform(-1.0, 1.0, (n, n))
        spec = to_spectrum(field, n, n // 2 + 1)
        assert rel_err(to_real(spec, n, n), field) <= 1e-12
        lhs, rhs = float(np.mean(field ** 2)), float(np.sum(w[:, None] * np.abs(spec) ** 2))
        assert abs(lhs - rhs) / abs(lhs) <= 1e-12


def test_bracket_of_unit_cosines():
    f = np.zeros((3, 8), dtype=complex)
    f[0, 1] = f[0, -1] = 0.5
    g = np.zeros((3, 8), dtype=complex)
    g[1, 0] = 0.5
    want = np.zeros((3, 8), dtype=complex)
    want[1, 1], want[1, -1] = -0.25, 0.25
    assert rel_err(bracket(f, g, *bracket_plans(8, 3)), want) < 1e-13


def test_bracket_self_is_exactly_zero():
    for seed in range(5):
        f = random_spectrum(8, 4, substream(21 + seed, 0))
        assert np.all(bracket(f, f, *bracket_plans(8, 4)) == 0.0)
    raw = substream(5, 0).uniform(-1, 1, (48, 480)) + 1j * substream(6, 0).uniform(-1, 1, (48, 480))
    assert np.all(bracket(raw, raw, *bracket_plans(480, 48)) == 0.0)


def test_bracket_antisymmetric_bilinear():
    gen = substream(22, 0)
    f, g = random_spectrum(8, 4, gen), random_spectrum(8, 4, gen)
    plans = bracket_plans(8, 4)
    assert rel_err(bracket(f, g, *plans), -bracket(g, f, *plans)) < 1e-13
    gen = substream(23, 0)
    f1, f2, g = (random_spectrum(7, 3, gen) for _ in range(3))
    plans = bracket_plans(7, 3)
    lhs = bracket(2.0 * f1 - 0.5 * f2, g, *plans)
    assert rel_err(lhs, 2.0 * bracket(f1, g, *plans) - 0.5 * bracket(f2, g, *plans)) < 1e-12


@pytest.mark.parametrize("n_kx, n_ky", [(8, 4), (7, 3), (16, 8), (12, 5), (9, 2), (2, 1), (1, 1)])
def test_bracket_matches_convolution_oracle(n_kx, n_ky):
    for seed in (1, 2, 3):
        gen = substream(seed, 0)
        f, g = random_spectrum(n_kx, n_ky, gen), random_spectrum(n_kx, n_ky, gen)
        assert rel_err(bracket(f, g, *bracket_plans(n_kx, n_ky)), direct.bracket_convolution(f, g)) < 1e-12


def test_bracket_quadratic_oracle_battery():
    """test_acceptance.py:102-123: 102 seeds on grids up to 16x8, 1e-12."""
    worst = worst_self = 0.0
    for n_kx, n_ky in ((8, 4), (7, 3), (16, 8)):
        plans = bracket_plans(n_kx, n_ky)
        gen_pairs = [(random_spectrum(n_kx, n_ky, g), random_spectrum(n_kx, n_ky, g))
                     for g in (substream(1000 + s, 0) for s in range(34))]
        f = np.stack([p[0] for p in gen_pairs])
        g = np.stack([p[1] for p in gen_pairs])
        got = bracket(f, g, *plans)
        for i in range(len(gen_pairs)):
            worst = max(worst, rel_err(got[i], direct.bracket_convolution(f[i], g[i])))
        worst_self = max(worst_self, float(np.max(np.abs(bracket(f, f, *plans)))))
    assert worst <= 1e-12 and worst_self <= 1e-12


def test_bracket_insensitive_to_extra_padding_and_int_plans():
    gen = substream(24, 0)
    f, g = random_spectrum(8, 4, gen), random_spectrum(8, 4, gen)
    tight = bracket(f, g, *bracket_plans(8, 4))
    for plans in ((32, 30), (13, 11), (17, 19), (22, 23)):  # 13, 17, 11, 19, 23: generic prime radices
        assert rel_err(bracket(f, g, *plans), tight) < 1e-12, plans


def test_bracket_output_representable_and_rejects():
    gen = substream(25, 0)
    f, g = random_spectrum(8, 4, gen), random_spectrum(8, 4, gen)
    out = bracket(f, g, *bracket_plans(8, 4))
    assert is_hermitian(out) and np.all(out[:, 4] == 0.0)
    with pytest.raises(ValueError):
        bracket(f, f, 11, 30)
    with pytest.raises(ValueError):
        bracket(f, f, 12, 9)
    with pytest.raises(ValueError):
        bracket(f, random_spectrum(8, 3, gen), 16, 16)


def test_bracket_broadcasting_vs_port():
    gen = substream(29, 0)
    f = gen.uniform(-1, 1, (2, 1, 4, 10)) + 1j * gen.uniform(-1, 1, (2, 1, 4, 10))
    g = gen.uniform(-1, 1, (3, 4, 10)) + 1j * gen.uniform(-1, 1, (3, 4, 10))
    nx, ny = (p.n_padded for p in bracket_plans(10, 4))
    got = bracket(f, g, nx, ny)
    assert got.shape == (2, 3, 4, 10)
    want = port.poisson_bracket(f, g, nx, ny)
    for idx in np.ndindex(2, 3):
        assert rel_err(got[idx], want[idx]) < 1e-13
    # f broadcast against a batch of g (f smaller)
    got2 = bracket(f[0, 0], g, nx, ny)
    assert rel_err(got2, port.poisson_bracket(f[0, 0], g, nx, ny)) < 1e-12


def test_hermitian_projection_helper():
    gen = substream(12, 0)
    spec = gen.uniform(-1, 1, (3, 8)) + 1j * gen.uniform(-1, 1, (3, 8))
    fixed = hermitian_ky0(spec)
    assert not is_hermitian(spec) and is_hermitian(fixed)
    assert np.array_equal(fixed[1:], spec[1:]) and np.array_equal(hermitian_ky0(fixed), fixed)
