"""Time gk_collision at sh03b (device events), current collision mode.  python tools/coll_time.py"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_10553_b200 import _lib  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda", 0)
M, T, Nc = 576, 32, 23040
h = torch.randn((M, T, Nc), dtype=torch.complex128, device=dev)
A = torch.randn((T, M, M), dtype=torch.float64, device=dev)
out = torch.empty_like(h)
st = _lib.stream_of(dev)
lib.gk_collision(A.data_ptr(), h.data_ptr(), out.data_ptr(), M, T, Nc, st)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    lib.gk_collision(A.data_ptr(), h.data_ptr(), out.data_ptr(), M, T, Nc, st)
e1.record()
torch.cuda.synchronize()
print(f"collision {e0.elapsed_time(e1) / 3:.2f} ms")
