"""On-device reference generator: bit-identical to the
reference's numpy Philox substreams, pinned by the reference's golden
generator statistics."""
import csv
import math

import numpy as np
import pytest
import torch

from conftest import GOLDEN
from paper_2305_10553_b200.grid import (GridShape, component_mean_abs, make_case, random_complex_device,
                                        random_state, random_state_device, substream, uniform_device)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed, stream, dims", [(1234, 0, (3, 5, 7)), (7, 4, (33,)), (2**64 - 1, 5, (2, 9)),
                                                (0, 1, (1,)), (2026, 3, (4, 4, 4, 4))])
def test_random_complex_bitwise(seed, stream, dims):
    want = np.asarray(substream(seed, stream).uniform(-1, 1, 2 * math.prod(dims)))
    got = random_complex_device(seed, stream, dims).cpu().numpy().reshape(-1)
    assert np.array_equal(got.real, want[: math.prod(dims)])
    assert np.array_equal(got.imag, want[math.prod(dims):])


def test_random_state_bitwise_desk_cases():
    for name in ("sh03b-desk", "em04b-desk"):
        shape = make_case(name)
        for seed in (7, 1234):
            assert np.array_equal(random_state_device(shape, seed).cpu().numpy(), random_state(shape, seed))


def test_uniform_matrices_bitwise():
    want = substream(1234, 3).uniform(-1.0, 1.0, (4, 72, 72))
    assert np.array_equal(uniform_device(1234, 3, (4, 72, 72)).cpu().numpy(), want)
    want = substream(5, 1).uniform(0.25, 3.0, 1001)
    assert np.array_equal(uniform_device(5, 1, (1001,), 0.25, 3.0).cpu().numpy(), want)


def test_generator_golden_statistics_on_device():
    """The reference's pkg/tests/data/generator_stats.csv, from device-generated states."""
    shapes = {100000: GridShape(50, 10, 10, 10, 2, 1), 221184: make_case("sh03b-desk"),
              663552: make_case("em04b-desk")}
    with open(GOLDEN / "generator_stats.csv", newline="") as fh:
        for row in csv.DictReader(fh):
            h = random_state_device(shapes[int(row["count"])], int(row["seed"])).cpu().numpy()
            assert math.isclose(component_mean_abs(h), float(row["mean_abs"]), rel_tol=1e-12)


def test_full_sh03b_state_on_device_matches_host_prefix():
    """sh03b (6.8 GB): device generation; spot-check a prefix and a tail block
    against the host generator drawing the same raw positions."""
    shape = make_case("sh03b")
    h = random_state_device(shape, 1234)
    n = shape.cell_count
    flat = h.reshape(-1)
    gen = substream(1234, 0)
    head = gen.uniform(-1, 1, 4096)
    assert np.array_equal(flat[:4096].real.cpu().numpy(), head)
    bg = np.random.Philox(key=1234)
    bg.advance((2 * n - 4096) // 4)  # advance() counts 4-draw blocks; last 4096 imaginary parts
    tail = np.random.Generator(bg).uniform(-1, 1, 4096)
    assert np.array_equal(flat[-4096:].imag.cpu().numpy(), tail)


@pytest.mark.parametrize("G, g", [(2, 1), (4, 0), (8, 5)])
def test_state_shard_generator_equals_slice_of_full_state(G, g):
    """A rank's home shard generated in place equals that slice of random_state."""
    from paper_2305_10553_b200.grid import random_state_device, random_state_shard_device
    shape = GridShape(24, 16, 3, 2, 2, 1)
    M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
    full = random_state_device(shape, 77).reshape(M, T, Y, R)
    Yl = Y // G
    shard = random_state_shard_device(shape, 77, g * Yl, (g + 1) * Yl)
    assert torch.equal(shard, full[:, :, g * Yl:(g + 1) * Yl])
