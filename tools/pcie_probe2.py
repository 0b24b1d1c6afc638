"""Full-duplex PCIe with k streams per direction (chunks of the buffer round-robin
over the streams): does a second copy engine per direction raise the aggregate?
    python tools/pcie_probe2.py [bytes]"""
import sys

import torch

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 6794772480
hb = torch.empty(n, dtype=torch.uint8, pin_memory=True)
ob = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")


def run(k, chunks=32):
    ss = [torch.cuda.Stream() for _ in range(2 * k)]
    step = -(-n // chunks)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for c in range(chunks):
        a, b = c * step, min(n, (c + 1) * step)
        with torch.cuda.stream(ss[c % k]):
            d1[a:b].copy_(hb[a:b], non_blocking=True)
        with torch.cuda.stream(ss[k + c % k]):
            ob[a:b].copy_(d2[a:b], non_blocking=True)
    for s in ss:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


for k in (1, 2, 4, 1, 2, 4):
    ms = run(k)
    print(f"{k} stream(s)/direction: both directions {ms:.1f} ms, {2 * n / ms / 1e6:.1f} GB/s aggregate", flush=True)
