"""ycol phase breakdown from a -DGK_YCOL_STATS build (tools/build_variant.sh ystats -DGK_YCOL_STATS):
    GK_LIB_PATH=build/variants/libgk_ystats.so python tools/ycol_stats.py"""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_10553_b200 import _lib  # noqa: E402
from paper_2305_10553_b200.grid import GridShape  # noqa: E402
from paper_2305_10553_b200.kernels import nonlinear_device  # noqa: E402
from paper_2305_10553_b200.spectral import bracket_plans  # noqa: E402

_lib.load()
raw = C.CDLL(str(_lib.LIB_PATH))
raw.gk_ycol_stats.restype = C.POINTER(C.c_ulonglong)
shape = GridShape(480, 48, 32, 72, 1, 1)
dev = torch.device("cuda", 0)
h = torch.randn(shape.dims, dtype=torch.complex128, device=dev)
phi = torch.randn(shape.field_dims, dtype=torch.complex128, device=dev)
nx, ny = (p.n_padded for p in bracket_plans(480, 48))
nonlinear_device(h, phi, nx, ny)
torch.cuda.synchronize()
buf = raw.gk_ycol_stats()
tot = [sum(buf[4 * i + k] for i in range(296)) for k in range(4)]
s = sum(tot)
print("ycol phases (thread 0 of each CTA): wait+sync %.1f%%, inverse %.1f%%, packed forward %.1f%%, separate %.1f%%"
      % tuple(100 * t / s for t in tot))
sub = [sum(buf[4 * 296 + 3 * i + k] for i in range(296)) for k in range(3)]
print("inverse split: pass 0 (load + DFT) %.1f%%, prefetch issue %.1f%%, pass 1 (+ product) %.1f%% of all ycol"
      % tuple(100 * t / s for t in sub))
