"""Pinned-memory PCIe rates for a state-sized buffer: H2D alone, D2H alone, both at once."""
import sys
import torch

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 6794772480
hb = torch.empty(n, dtype=torch.uint8, pin_memory=True)
ob = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)
t(lambda: d1.copy_(hb, non_blocking=True))
h2d = t(lambda: d1.copy_(hb, non_blocking=True))
d2h = t(lambda: ob.copy_(d2, non_blocking=True))
def both():
    with torch.cuda.stream(s1):
        d1.copy_(hb, non_blocking=True)
    with torch.cuda.stream(s2):
        ob.copy_(d2, non_blocking=True)
bo = t(both)
print(f"bytes {n/1e9:.2f} GB: H2D {h2d:.1f} ms ({n/h2d/1e6:.1f} GB/s), D2H {d2h:.1f} ms ({n/d2h/1e6:.1f} GB/s), "
      f"both concurrently {bo:.1f} ms")
