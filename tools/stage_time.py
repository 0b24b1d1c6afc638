"""Per-stage device time of the step (Stepper.stage, CUDA events), for A/B of
variant builds:  GK_LIB_PATH=build/variants/libgk_X.so python tools/stage_time.py [case] [reps]"""
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_10553_b200.grid import make_case, random_state_device  # noqa: E402
from paper_2305_10553_b200.kernels import make_kernel_inputs  # noqa: E402
from paper_2305_10553_b200.step import Stepper  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "sh03b"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
shape = make_case(case)
dev = torch.device("cuda", 0)
h = random_state_device(shape, 1234, dev)
st = Stepper(shape, make_kernel_inputs(shape, 1234), 1.5e-9, device=dev, graph=False)
out = torch.empty_like(h)
for _ in range(2):
    st.step(h, out)
torch.cuda.synchronize()
res = {}
for name, idx in (("field", 0), ("nl", 1), ("coll", 2), ("str", 3)):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st.stage(idx, h, out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    res[name] = statistics.median(ts)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    st.step(h, out)
b.record()
torch.cuda.synchronize()
print(case, {k: round(v, 3) for k, v in res.items()}, "step", round(a.elapsed_time(b) / reps, 3), "ms")
