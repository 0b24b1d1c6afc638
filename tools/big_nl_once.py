"""Nonlinear term on a few velocity rows of a large-grid case (C5a: 2016x480
plan, em04b: 2016x864) for launch lists / ncu.
    python tools/big_nl_once.py c5a|em04b [n_vel] [reps]"""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_10553_b200.grid import GridShape  # noqa: E402
from paper_2305_10553_b200.kernels import nonlinear_device  # noqa: E402
from paper_2305_10553_b200.spectral import bracket_plans  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "c5a"
nv = int(sys.argv[2]) if len(sys.argv) > 2 else 18
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
R, Y = {"c5a": (1344, 160), "em04b": (1344, 288)}[case]
shape = GridShape(R, Y, 24, nv, 1, 1)
dev = torch.device("cuda", 0)
h = torch.randn(shape.dims, dtype=torch.complex128, device=dev)
phi = torch.randn(shape.field_dims, dtype=torch.complex128, device=dev)
nx, ny = (p.n_padded for p in bracket_plans(R, Y))
nonlinear_device(h, phi, nx, ny)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(reps):
    nonlinear_device(h, phi, nx, ny)
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / reps
slices = nv * 24
print(f"{case} plan {nx}x{ny}: {slices} slices {dt*1e3:.2f} ms = {dt/slices*1e6:.2f} us/slice")
