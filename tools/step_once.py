"""One sh03b step (after a warm-up step) through Stepper, for ncu captures of the
step's kernels (fused field + int8 slicing, x/y FFT kernels, int8 GEMM, finish).
    python tools/step_once.py [case]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_10553_b200.grid import make_case, random_state_device  # noqa: E402
from paper_2305_10553_b200.kernels import make_kernel_inputs  # noqa: E402
from paper_2305_10553_b200.step import Stepper  # noqa: E402

shape = make_case(sys.argv[1] if len(sys.argv) > 1 else "sh03b")
dev = torch.device("cuda", 0)
h = random_state_device(shape, 1234, dev)
st = Stepper(shape, make_kernel_inputs(shape, 1234), dt=1e-6)
out = torch.empty_like(h)
for _ in range(2):
    st.step(h, out)
torch.cuda.synchronize()
print("ok")
