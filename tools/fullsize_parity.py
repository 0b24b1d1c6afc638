"""Full-size parity over N steps (evidence run, not a test): the GPU step (int8
tensor-core collision) against the CPU oracle on the whole state
(tests/test_gpu_fullsize.py's blocked port.step), with the relative L2 error of h
and phi printed after every step.  sh03b: 6.8 GB state, 720 x 144 plan (host
peak ~40 GB).  Larger cases need ~5 state-sized host arrays (C5a: ~180 GB).
    python tools/fullsize_parity.py [steps] [dt] [case]"""
import sys
import time
from pathlib import Path

import numpy as np
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
case = sys.argv[3] if len(sys.argv) > 3 else "sh03b"
shape = make_case(case)
M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
inp = make_kernel_inputs(shape, 1234)
nx, ny = (p.n_padded for p in inp["plans"])
x_gpu = random_state_device(shape, 1234)
x_cpu = x_gpu.reshape(M, T, Y, R).cpu().numpy()
st = Stepper(shape, inp, dt)
y_gpu = torch.empty_like(x_gpu)
print(f"{case}, {steps} steps, dt = {dt:g}, int8 collision mode, seed 1234", flush=True)


def rel_l2_chunked(dev_t, host):
    """relative L2 of a device state against a host array, a velocity block at a time"""
    num = den = 0.0
    d = dev_t.reshape(M, T, Y, R)
    for v0 in range(0, M, 16):
        a = d[v0:v0 + 16].cpu().numpy()
        b = host[v0:v0 + 16]
        num += float(np.sum(np.abs(a - b) ** 2))
        den += float(np.sum(np.abs(b) ** 2))
    return (num / den) ** 0.5
for n in range(1, steps + 1):
    st.step(x_gpu, y_gpu)
    x_gpu, y_gpu = y_gpu, x_gpu
    t0 = time.perf_counter()
    phi = port.field(x_cpu.reshape(shape.dims), inp["weights"])
    ephi = rel_l2(st.phi.cpu().numpy(), phi)
    x_cpu = _oracle_step_blocked(x_cpu, phi, inp, dt, nx, ny)
    eh = rel_l2_chunked(x_gpu, x_cpu)
    print(f"step {n:2d}: rel L2 h {eh:.3e}  phi {ephi:.3e}  (oracle {time.perf_counter() - t0:.0f} s)", flush=True)
