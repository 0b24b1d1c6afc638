"""Bitwise A/B of builds / B-slicing kernels (default: slice_b, GK_SB_PIPE=1: the
pipelined slice_bp): digest of one sh03b step (h', phi) and of standalone
collisions at awkward shapes.   python tools/sb_ab.py; GK_SB_PIPE=1 python tools/sb_ab.py"""
import hashlib
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_10553_b200 import _lib  # noqa: E402
from paper_2305_10553_b200.grid import GridShape, make_case, random_state, random_state_device  # noqa: E402
from paper_2305_10553_b200.kernels import collision_kernel, make_kernel_inputs  # noqa: E402
from paper_2305_10553_b200.step import Stepper  # noqa: E402


def digest(t):
    hsh = hashlib.sha256()
    flat = t.reshape(-1)
    for i in range(0, flat.numel(), 1 << 26):
        hsh.update(flat[i:i + (1 << 26)].cpu().numpy().tobytes())
    return hsh.hexdigest()[:16]


dev = torch.device("cuda", 0)
_lib.load().gk_collision_mode(2)
for dims in [(40, 20, 3, 4, 4, 2), (33, 7, 2, 9, 8, 3), (480, 48, 2, 4, 4, 2)]:
    shape = GridShape(*dims)
    h = random_state(shape, 3)
    A = make_kernel_inputs(shape, 3)["matrices"]
    print(dims, hashlib.sha256(np.ascontiguousarray(collision_kernel(h, A)).tobytes()).hexdigest()[:16])
shape = make_case("sh03b")
st = Stepper(shape, make_kernel_inputs(shape, 1234), 1.5e-9, device=dev)
h = random_state_device(shape, 1234, dev)
out = st.step(h)
torch.cuda.synchronize()
print("sh03b h'", digest(torch.view_as_real(out)), "phi", digest(torch.view_as_real(st.phi)))
