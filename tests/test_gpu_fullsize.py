"""Full-size parity at the benchmark shape (sh03b, 6.8 GB state).

The GPU runs the whole step on the reference generator's sh03b state; the CPU
oracle then recomputes phi in full and the new state on a grid of (velocity,
theta) slices -- every term of the composition (stream, nonlinear bracket,
collision row, shear) from the reference algorithm on the same inputs."""
import numpy as np
import pytest
import torch

from conftest import rel_err
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
