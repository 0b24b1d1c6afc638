"""Full-size parity at the benchmark shape (sh03b, 6.8 GB state).

The GPU runs the whole step on the reference generator's sh03b state; the CPU
oracle then recomputes phi in full and the new state on a grid of (velocity,
theta) slices -- every term of the composition (stream, nonlinear bracket,
collision row, shear) from the reference algorithm on the same inputs."""
import numpy as np
import pytest
import torch

from conftest import rel_err, rel_l2
from oracle import port
from paper_2305_10553_b200.grid import make_case, random_state_device
from paper_2305_10553_b200.kernels import make_kernel_inputs
from paper_2305_10553_b200.step import Stepper

pytestmark = pytest.mark.gpu


def test_sh03b_step_matches_oracle_on_slices():
    shape = make_case("sh03b")
    M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
    inp = make_kernel_inputs(shape, 1234)
    dt = 1e-6
    h_dev = random_state_device(shape, 1234)
    st = Stepper(shape, inp, dt)
    out = st.step(h_dev)
    torch.cuda.synchronize()
    h = h_dev.reshape(M, T, Y, R).cpu().numpy()
    got = out.reshape(M, T, Y, R).cpu().numpy()
    phi_gpu = st.phi.cpu().numpy()
    del h_dev, out
    # phi = field(h, w): full reduction on the host (reference tensordot)
    phi = port.field(h.reshape(shape.dims), inp["weights"])
    assert rel_err(phi_gpu, phi) < 1e-13
    nx, ny = (p.n_padded for p in inp["plans"])
    c = np.asarray(inp["stencil"])
    half = len(c) // 2
    for v in (0, 289, M - 1):
        for t in (0, 17, T - 1):
            # stream term for this (v, t): original-order periodic stencil over theta
            s = sum(c[i] * h[v, (t + i - half) % T] for i in range(len(c)))
            nl = port.poisson_bracket(h[v, t], phi[t], nx, ny)
            coll = np.tensordot(inp["matrices"][t, v], h[:, t], axes=1)
            want = port.shear((h[v, t] + dt * ((s + nl) + coll))[None], inp["shifts"])[0]
            assert rel_err(got[v, t], want) < 1e-12, (v, t)


def _oracle_step_blocked(h, phi, inp, dt, nx, ny, rows=16, threads=None):
    """port.step (stream + nonlinear, then + collision; shear(h + dt rhs)) on the
    full state, the bracket and the stream sub-batched over velocity rows so the
    host holds only a few state-sized arrays (the reference's whole-batch
    temporaries would need ~75 GB at sh03b).  Same numpy calls and association
    order per element as port.step, so it equals port.step exactly."""
    import os
    M, T, Y, R = h.shape
    threads = threads or os.cpu_count() or 1
    coll = port.collision(h.reshape(M, 1, 1, T, Y, R), inp["matrices"]).reshape(h.shape)
    new = np.empty_like(h)
    for v0 in range(0, M, rows):
        blk = h[v0:v0 + rows].reshape(-1, 1, 1, T, Y, R)
        rhs = port.stream(blk, inp["stencil"])
        rhs = rhs + port.nonlinear(blk, phi, nx, ny, threads)
        rhs = rhs + coll[v0:v0 + rows].reshape(blk.shape)
        new[v0:v0 + rows] = port.shear(blk + dt * rhs, inp["shifts"]).reshape(-1, T, Y, R)
    return new


def test_sh03b_three_full_steps_match_oracle():
    """North-star bar at the headline shape itself: 3 full sh03b steps (M = 576,
    720 x 144 plan, int8 tensor-core collision, 6.8 GB state) against the CPU
    oracle run on the whole state -- h and phi within 1e-10 relative L2.
    dt = 2e-8 moves the state ~7% per step (|nl| / |h| ~ 3.5e6 at this shape)."""
    shape = make_case("sh03b")
    M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
    inp = make_kernel_inputs(shape, 1234)
    nx, ny = (p.n_padded for p in inp["plans"])
    dt = 2e-8
    x_gpu = random_state_device(shape, 1234)
    x_cpu = x_gpu.reshape(M, T, Y, R).cpu().numpy()
    h_init = x_gpu.clone()
    st = Stepper(shape, inp, dt)
    y_gpu = torch.empty_like(x_gpu)
    for _ in range(3):
        st.step(x_gpu, y_gpu)
        x_gpu, y_gpu = y_gpu, x_gpu
        phi = port.field(x_cpu.reshape(shape.dims), inp["weights"])
        assert rel_l2(st.phi.cpu().numpy(), phi) < 1e-10
        x_cpu = _oracle_step_blocked(x_cpu, phi, inp, dt, nx, ny)
    moved = float(torch.linalg.vector_norm(x_gpu - h_init) / torch.linalg.vector_norm(h_init))
    assert moved > 0.05, moved  # the state really moved
    del h_init
    got = x_gpu.reshape(M, T, Y, R).cpu().numpy()
    assert rel_l2(got, x_cpu) < 1e-10


def test_c2_ten_full_steps_match_oracle():
    """configs[1] at full size (480 x 1 x 32 x 24 x 8 x 3, linear-only: stream +
    field + collision, int8 collision at M = 576), 10 steps vs the oracle."""
    shape = make_case("c2-linear")
    M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
    inp = make_kernel_inputs(shape, 77)
    dt = 1e-2
    x_gpu = random_state_device(shape, 77)
    x_cpu = x_gpu.reshape(shape.dims).cpu().numpy()
    st = Stepper(shape, inp, dt, nonlinear=False)
    y_gpu = torch.empty_like(x_gpu)
    for _ in range(10):
        st.step(x_gpu, y_gpu)
        x_gpu, y_gpu = y_gpu, x_gpu
        x_cpu, phi = port.step(x_cpu, inp["weights"], inp["stencil"], inp["matrices"], inp["shifts"], dt, 0, 0,
                               nonlinear_on=False)
        assert rel_l2(st.phi.cpu().numpy(), phi) < 1e-10
    assert rel_l2(x_gpu.reshape(shape.dims).cpu().numpy(), x_cpu) < 1e-10
