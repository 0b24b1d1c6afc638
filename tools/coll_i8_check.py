"""int8-slice collision vs fp64 DMMA vs numpy on awkward shapes, then sh03b timing.
    python tools/coll_i8_check.py"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_10553_b200 import _lib  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda", 0)
st = _lib.stream_of(dev)


def run(mode, A, h, M, T, Nc):
    out = torch.empty_like(h)
    lib.gk_collision_mode(mode)
    _lib.check(lib.gk_collision(A.data_ptr(), h.data_ptr(), out.data_ptr(), M, T, Nc, st), "collision")
    torch.cuda.synchronize()
    return out


def case(M, T, Nc, seed, scale_rows=False):
    g = torch.Generator(device=dev).manual_seed(seed)
    h = torch.complex(torch.rand((M, T, Nc), dtype=torch.float64, device=dev, generator=g) * 2 - 1,
                      torch.rand((M, T, Nc), dtype=torch.float64, device=dev, generator=g) * 2 - 1)
    A = torch.rand((T, M, M), dtype=torch.float64, device=dev, generator=g) * 2 - 1
    if scale_rows:  # wide dynamic range across rows / columns
        A = A * torch.logspace(-8, 8, M, dtype=torch.float64, device=dev)[None, :, None]
        h = h * torch.logspace(-5, 5, Nc, dtype=torch.float64, device=dev)[None, None, :]
    ci8 = run(2, A, h, M, T, Nc)
    cdm = run(1, A, h, M, T, Nc)
    e = ((ci8 - cdm).abs().max() / cdm.abs().max()).item()
    # per-column relative error (the slicing scales are per column)
    col = ((ci8 - cdm).abs().amax(dim=0) / cdm.abs().amax(dim=0).clamp_min(1e-300)).max().item()
    line = f"M={M} T={T} Nc={Nc} rows_scaled={scale_rows}: max rel {e:.2e}, worst column {col:.2e}"
    if M * T * Nc <= 64 * 3 * 2000:
        hn, An = h.cpu().numpy(), A.cpu().numpy()
        ref = np.einsum("tim,mtn->itn", An, hn)
        en = np.abs(ci8.cpu().numpy() - ref).max() / np.abs(ref).max()
        line += f", vs numpy {en:.2e}"
    print(line, flush=True)
    return e


worst = 0.0
for M, T, Nc, sr in [(64, 2, 100, False), (100, 3, 77, False), (32, 1, 5, False), (576, 2, 2048, False),
                     (432, 2, 1000, False), (64, 3, 2000, True), (576, 1, 23040, False)]:
    worst = max(worst, case(M, T, Nc, 7 + M, sr))
# identity / zero
M, T, Nc = 64, 2, 300
h = torch.randn((M, T, Nc), dtype=torch.complex128, device=dev)
eye = torch.eye(M, dtype=torch.float64, device=dev).expand(T, M, M).contiguous()
o = run(2, eye, h, M, T, Nc)
print("identity max rel", ((o - h).abs().max() / h.abs().max()).item(), "zero:",
      bool((run(2, torch.zeros_like(eye), h, M, T, Nc) == 0).all()))

# timing at sh03b
M, T, Nc = 576, 32, 23040
h = torch.randn((M, T, Nc), dtype=torch.complex128, device=dev)
A = torch.randn((T, M, M), dtype=torch.float64, device=dev)
out = torch.empty_like(h)
for mode in (2, 1, 2):
    lib.gk_collision_mode(mode)
    lib.gk_collision(A.data_ptr(), h.data_ptr(), out.data_ptr(), M, T, Nc, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        lib.gk_collision(A.data_ptr(), h.data_ptr(), out.data_ptr(), M, T, Nc, st)
    e1.record()
    torch.cuda.synchronize()
    print(f"sh03b collision mode {mode}: {e0.elapsed_time(e1) / 3:.2f} ms", flush=True)
print("worst max rel", worst)
