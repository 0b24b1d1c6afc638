"""GPU parity of the builder-defined step and the
north_star acceptance bar: distribution function and fields within 1e-10
relative L2 of the reference after N steps, on identical inputs."""
import numpy as np
import pytest
import torch

from conftest import rel_err, rel_l2
from oracle import port
from paper_2305_10553_b200.grid import GridShape, make_case, random_state
from paper_2305_10553_b200.kernels import (collision_kernel, field_kernel, make_kernel_inputs,
                                           nonlinear_kernel, shear_kernel, stream_kernel)
from paper_2305_10553_b200.step import Stepper

pytestmark = pytest.mark.gpu

C1 = GridShape(16, 8, 8, 8, 4, 2)


def test_c1_ten_steps_match_reference(golden, tables):
    """Reference composition run by the reference package itself (golden)."""
    cfg = tables["step"]
    h = random_state(C1, cfg["seed"])
    inp = make_kernel_inputs(C1, cfg["seed"])
    got = Stepper(C1, inp, cfg["dt"]).run(h, cfg["n"])
    assert rel_l2(got, golden["c1_step10"]) < 1e-10


def test_c1_steps_and_fields_vs_oracle():
    h = random_state(C1, 7)
    inp = make_kernel_inputs(C1, 7)
    nx, ny = (p.n_padded for p in inp["plans"])
    st = Stepper(C1, inp, 1e-3)
    x_gpu = torch.from_numpy(h).cuda()
    x_cpu = h
    for _ in range(10):
        x_gpu = st.step(x_gpu)
        x_cpu, phi_cpu = port.step(x_cpu, inp["weights"], inp["stencil"], inp["matrices"], inp["shifts"],
                                   1e-3, nx, ny)
        assert rel_l2(st.phi.cpu().numpy(), phi_cpu) < 1e-10
    assert rel_l2(x_gpu.cpu().numpy(), x_cpu) < 1e-10


def test_step_equals_composition_of_kernels():
    """gk_step is exactly the composition of the public kernels (same rounding)."""
    shape = make_case("sh03b-desk")
    h = random_state(shape, 3)
    inp = make_kernel_inputs(shape, 3)
    dt = 1e-4
    phi = field_kernel(h, inp["weights"])
    rhs = stream_kernel(h, inp["stencil"]) + nonlinear_kernel(h, phi, inp["plans"])
    rhs = rhs + collision_kernel(h, inp["matrices"])
    want = shear_kernel(h + dt * rhs, inp["shifts"])
    got = Stepper(shape, inp, dt).run(h, 1)
    assert np.array_equal(got, want)


def test_linear_only_path():
    """C2-style single toroidal mode, no bracket (configs[1])."""
    shape = GridShape(24, 1, 8, 6, 4, 3)
    h = random_state(shape, 11)
    inp = make_kernel_inputs(shape, 11)
    got = Stepper(shape, inp, 1e-2, nonlinear=False).run(h, 5)
    x = h
    for _ in range(5):
        x, _ = port.step(x, inp["weights"], inp["stencil"], inp["matrices"], inp["shifts"], 1e-2, 0, 0,
                         nonlinear_on=False)
    assert rel_l2(got, x) < 1e-12


def test_step_deterministic_bitwise():
    shape = make_case("em04b-desk")
    h = torch.from_numpy(random_state(shape, 5)).cuda()
    st = Stepper(shape, make_kernel_inputs(shape, 5), 1e-4)
    a = st.step(h).cpu().numpy()
    b = st.step(h).cpu().numpy()
    assert np.array_equal(a, b)
    assert rel_err(a, a) == 0.0


def test_step_stages_compose_to_the_step():
    """gk_step_stage 0..3 on the step's workspace reproduce gk_step bitwise."""
    shape = make_case("sh03b-desk")
    h = torch.from_numpy(random_state(shape, 8)).cuda()
    st = Stepper(shape, make_kernel_inputs(shape, 8), 1e-4)
    want = st.step(h)
    out = torch.empty_like(h)
    for i in range(4):
        st.stage(i, h, out)
    assert torch.equal(out, want)
