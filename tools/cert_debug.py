"""Which int8-collision tiles fail the accuracy certificate on a given shape
(diagnostic).  python tools/cert_debug.py R Y T X E S"""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_10553_b200 import _lib  # noqa: E402
from paper_2305_10553_b200.grid import GridShape, random_state_device  # noqa: E402
from paper_2305_10553_b200.kernels import make_kernel_inputs  # noqa: E402

dims = [int(x) for x in sys.argv[1:7]]
shape = GridShape(*dims)
lib = _lib.load()
dev = torch.device("cuda", 0)
h = random_state_device(shape, 1234, dev)
A = torch.from_numpy(make_kernel_inputs(shape, 1234)["matrices"]).to(dev)
M, T, cells = shape.velocity_size, shape.n_theta, shape.n_toroidal * shape.n_radial
st = torch.cuda.current_stream().cuda_stream


def fix():
    v = C.c_int64()
    lib.gk_collision_fixups(C.byref(v))
    return v.value


out = torch.empty_like(h)
ref = torch.empty_like(h)
lib.gk_collision_mode(1)
_lib.check(lib.gk_collision(A.data_ptr(), h.data_ptr(), ref.data_ptr(), M, T, cells, st), "dmma")
lib.gk_collision_mode(2)
f0 = fix()
_lib.check(lib.gk_collision(A.data_ptr(), h.data_ptr(), out.data_ptr(), M, T, cells, st), "i8")
f1 = fix()
ncb, nib = -(-2 * cells // 128), -(-M // 64)
d = (torch.view_as_real(out) - torch.view_as_real(ref)).abs().reshape(M, T, 2 * cells)
print(dims, "tiles", T * ncb * nib, "fixups", f1 - f0,
      "max err", float(d.max() / torch.view_as_real(ref).abs().max()))
