import sys
from pathlib import Path
import torch
sys.path.insert(0, "/root/repo")
sys.path.insert(0, ".")
from paper_2305_10553_b200.grid import GridShape
from paper_2305_10553_b200.kernels import nonlinear_device
from paper_2305_10553_b200.spectral import bracket_plans
shape = GridShape(1344, 160, 24, 18, 1, 1)   # C5a slices (18 velocity rows of 432)
dev = torch.device("cuda", 0)
h = torch.randn(shape.dims, dtype=torch.complex128, device=dev)
phi = torch.randn(shape.field_dims, dtype=torch.complex128, device=dev)
nx, ny = (p.n_padded for p in bracket_plans(1344, 160))
for _ in range(2):
    nonlinear_device(h, phi, nx, ny)
torch.cuda.synchronize()
print("ok", nx, ny)
