"""Device time of the transposes' local block permutation (gk_permute_blocks) at the
sh03b per-rank sizes for G = 2, 4, 8 (the data each rank permutes per transpose:
S/G), for the multi-GPU step model in DESIGN.md §4."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_10553_b200 import _lib  # noqa: E402
from paper_2305_10553_b200.grid import make_case  # noqa: E402

lib = _lib.load()
shape = make_case("sh03b")
M, T, Y, R = shape.velocity_size, shape.n_theta, shape.n_toroidal, shape.n_radial
st = _lib.stream_of(torch.device("cuda", 0))
for G in (2, 4, 8):
    n = shape.state_bytes // 16 // G
    src = torch.zeros(n, dtype=torch.complex128, device="cuda")
    dst = torch.empty_like(src)
    # [G][M/G][T][Y/G * R] -> [M/G][T][G][Y/G * R] blocks: n_a = G, n_b = M/G * T, inner = Y/G * R
    args = (G, M // G * T, Y // G * R)
    lib.gk_permute_blocks(src.data_ptr(), dst.data_ptr(), *args, st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        lib.gk_permute_blocks(src.data_ptr(), dst.data_ptr(), *args, st)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"G={G}: {n * 16 / 1e9:.3f} GB per rank, permute {ms:.3f} ms ({2 * n * 16 / ms / 1e6:.0f} GB/s)")
