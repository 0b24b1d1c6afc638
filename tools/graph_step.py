"""Whole-step time eager vs CUDA-graph replay (launch gaps / host overhead).
    python tools/graph_step.py [case] [steps]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_10553_b200.grid import make_case, random_state_device  # noqa: E402
from paper_2305_10553_b200.kernels import make_kernel_inputs  # noqa: E402
from paper_2305_10553_b200.step import Stepper  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "sh03b"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
shape = make_case(case)
dev = torch.device("cuda", 0)
h = random_state_device(shape, 1234, dev)
st = Stepper(shape, make_kernel_inputs(shape, 1234), dt=1e-6)
out = torch.empty_like(h)
s = torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for _ in range(3):
    st.step(h, out)
eager = timed(lambda: st.step(h, out))
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    st.step(h, out)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        st.step(h, out)
for _ in range(3):
    g.replay()
graph = timed(g.replay)
ref = out.clone()
st.step(h, out)
torch.cuda.synchronize()
print(f"{case}: eager {eager:.3f} ms/step, graph replay {graph:.3f} ms/step, same result: {torch.equal(ref, out)}")
