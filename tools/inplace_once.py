"""One in-place sh03b step (after a warm-up one) for launch lists / ncu.
    python tools/inplace_once.py [case]"""
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
st = Stepper(shape, make_kernel_inputs(shape, 1234), dt=1e-6, inplace=True)
for _ in range(2):
    st.step_inplace(h)
torch.cuda.synchronize()
print("ok")
