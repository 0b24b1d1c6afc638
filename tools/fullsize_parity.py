"""Full-size sh03b parity over N steps (evidence run, not a test): the GPU step
(int8 tensor-core collision, 720 x 144 plan, 6.8 GB state) against the CPU oracle
on the whole state (tests/test_gpu_fullsize.py's blocked port.step), with the
relative L2 error of h and phi printed after every step.
    python tools/fullsize_parity.py [steps] [dt]"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
from conftest import rel_l2  # noqa: E402
from oracle import port  # noqa: E402
from test_gpu_fullsize import _oracle_step_blocked  # noqa: E402
from paper_2305_10553_b200.grid import make_case, random_state_device  # noqa: E402
from paper_2305_10553_b200.kernels import make_kernel_inputs  # noqa: E402
from paper_2305_10553_b200.step import Stepper  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
dt = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-8
shape = make_case("sh03b")
M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
inp = make_kernel_inputs(shape, 1234)
nx, ny = (p.n_padded for p in inp["plans"])
x_gpu = random_state_device(shape, 1234)
x_cpu = x_gpu.reshape(M, T, Y, R).cpu().numpy()
h0 = x_gpu.clone()
st = Stepper(shape, inp, dt)
y_gpu = torch.empty_like(x_gpu)
print(f"sh03b, {steps} steps, dt = {dt:g}, int8 collision mode, seed 1234", flush=True)
for n in range(1, steps + 1):
    st.step(x_gpu, y_gpu)
    x_gpu, y_gpu = y_gpu, x_gpu
    t0 = time.perf_counter()
    phi = port.field(x_cpu.reshape(shape.dims), inp["weights"])
    ephi = rel_l2(st.phi.cpu().numpy(), phi)
    x_cpu = _oracle_step_blocked(x_cpu, phi, inp, dt, nx, ny)
    eh = rel_l2(x_gpu.reshape(M, T, Y, R).cpu().numpy(), x_cpu)
    moved = float(torch.linalg.vector_norm(x_gpu - h0) / torch.linalg.vector_norm(h0))
    print(f"step {n:2d}: rel L2 h {eh:.3e}  phi {ephi:.3e}  |h - h0|/|h0| {moved:.3f}  "
          f"(oracle {time.perf_counter() - t0:.0f} s)", flush=True)
