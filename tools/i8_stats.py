"""MMA-thread wait breakdown of the int8 collision GEMM (variant lib built with -DGK_I8_STATS):
    tools/build_variant.sh stats -DGK_I8_STATS
    GK_LIB_PATH=build/variants/libgk_stats.so python tools/i8_stats.py"""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_10553_b200 import _lib  # noqa: E402

lib = _lib.load()
raw = C.CDLL(str(_lib.LIB_PATH))
raw.gk_i8_stats.restype = C.POINTER(C.c_longlong)
dev = torch.device("cuda", 0)
M, T, Nc = 576, 32, 23040
h = torch.randn((M, T, Nc), dtype=torch.complex128, device=dev)
A = torch.randn((T, M, M), dtype=torch.float64, device=dev)
out = torch.empty_like(h)
for _ in range(2):
    lib.gk_collision(A.data_ptr(), h.data_ptr(), out.data_ptr(), M, T, Nc, _lib.stream_of(dev))
torch.cuda.synchronize()
st = raw.gk_i8_stats()
rows = [tuple(st[6 * i + k] for k in range(6)) for i in range(148)]
lead = [r for r in rows if r[2] > 0]  # CTA pairs (GK_I8_PAIR=1): only the leader issues MMAs
wf = sum(r[0] for r in lead) / len(lead)
we = sum(r[1] for r in lead) / len(lead)
tot = sum(r[2] for r in lead) / len(lead)
print(f"last group GEMM, MMA thread per CTA: total {tot:.0f} clk, wait full {wf / tot:.1%}, wait tmem-empty {we / tot:.1%}")
ew, ed, es = (sum(r[k] for r in rows) / 148 for k in (3, 4, 5))
print(f"epilogue warp 2: wait tfull {ew / tot:.1%}, drain {ed / tot:.1%}, store {es / tot:.1%}")
