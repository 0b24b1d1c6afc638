"""Run the nonlinear kernel on a sh03b-slice-shaped case (few velocity points) for profiling.
    python tools/nl_once.py [n_vel_slices] [reps]"""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_10553_b200 import _lib
from paper_2305_10553_b200.grid import GridShape
from paper_2305_10553_b200.kernels import nonlinear_device
from paper_2305_10553_b200.spectral import bracket_plans

nv = int(sys.argv[1]) if len(sys.argv) > 1 else 2
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
shape = GridShape(480, 48, 32, nv, 1, 1)
dev = torch.device("cuda", 0)
h = torch.randn(shape.dims, dtype=torch.complex128, device=dev)
phi = torch.randn(shape.field_dims, dtype=torch.complex128, device=dev)
nx, ny = (p.n_padded for p in bracket_plans(480, 48))
for _ in range(reps):
    out = nonlinear_device(h, phi, nx, ny)
torch.cuda.synchronize()
print("ok", out.shape)
