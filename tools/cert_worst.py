"""Collision time when the accuracy certificate fails on most tiles (h graded over
12 decades along velocity, the ADVICE r1 case) vs regular data and the DMMA path,
at the sh03b GEMM size.   python tools/cert_worst.py"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_10553_b200 import _lib  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda", 0)
M, T, Nc = 576, 32, 23040
g = torch.Generator(device=dev).manual_seed(5)
h = torch.complex(torch.rand((M, T, Nc), dtype=torch.float64, device=dev, generator=g) * 2 - 1,
                  torch.rand((M, T, Nc), dtype=torch.float64, device=dev, generator=g) * 2 - 1)
A = torch.rand((T, M, M), dtype=torch.float64, device=dev, generator=g) * 2 - 1
graded = h * torch.logspace(-6, 6, M, dtype=torch.float64, device=dev)[:, None, None]
out = torch.empty_like(h)
st = _lib.stream_of(dev)
import ctypes  # noqa: E402


def fixups():
    n = ctypes.c_int64(0)
    lib.gk_collision_fixups(ctypes.byref(n))
    return n.value


def timeit(x, mode, label):
    lib.gk_collision_mode(mode)
    lib.gk_collision(A.data_ptr(), x.data_ptr(), out.data_ptr(), M, T, Nc, st)
    torch.cuda.synchronize()
    f0 = fixups()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        lib.gk_collision(A.data_ptr(), x.data_ptr(), out.data_ptr(), M, T, Nc, st)
    e1.record()
    torch.cuda.synchronize()
    tiles = (fixups() - f0) / 3
    print(f"{label}: {e0.elapsed_time(e1) / 3:.2f} ms, {tiles:.0f} of {T * 360 * 9} tiles recomputed", flush=True)


timeit(h, 2, "int8, U[-1,1] data")
timeit(graded, 2, "int8, h graded over 12 decades in velocity")
A_inv = A * torch.logspace(6, -6, M, dtype=torch.float64, device=dev)[None, None, :]
A_save = A.clone()
A.copy_(A_inv)
timeit(graded, 2, "int8, graded h and inversely graded A (products of equal size)")
A.copy_(A_save)
timeit(h, 1, "DMMA")
