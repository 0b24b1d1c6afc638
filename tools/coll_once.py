"""One sh03b collision call (after a warm-up) for ncu."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_10553_b200 import _lib
from paper_2305_10553_b200.grid import make_case
shape = make_case(sys.argv[1] if len(sys.argv) > 1 else "sh03b")
dev = torch.device("cuda", 0)
lib = _lib.load()
M, T, Nc = shape.velocity_size, shape.n_theta, shape.n_toroidal * shape.n_radial
h = torch.randn(shape.dims, dtype=torch.complex128, device=dev)
A = torch.randn((T, M, M), dtype=torch.float64, device=dev)
out = torch.empty_like(h)
for _ in range(2):
    _lib.check(lib.gk_collision(A.data_ptr(), h.data_ptr(), out.data_ptr(), M, T, Nc, _lib.stream_of(dev)), "coll")
torch.cuda.synchronize()
print("ok")
