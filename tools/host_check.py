"""gk_step_host vs gk_step, bitwise, with NaN-filled device/host output buffers
(a region the pipeline never writes or copies shows up).  GK_E2E_VBLOCKS picks the
velocity blocking.   python tools/host_check.py"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_10553_b200.grid import make_case, random_state  # noqa: E402
from paper_2305_10553_b200.kernels import make_kernel_inputs  # noqa: E402
from paper_2305_10553_b200.step import Stepper  # noqa: E402

for case, seed, dt in [("sh03b-desk", 1234, 1e-3), ("c1-tiny", 1234, 1e-3), ("em04b-desk", 3, 1e-4)]:
    shape = make_case(case)
    inp = make_kernel_inputs(shape, seed)
    h = random_state(shape, seed)
    st = Stepper(shape, inp, dt)
    hd = torch.from_numpy(h).cuda()
    want = st.step(hd).cpu().numpy()
    h_host = torch.from_numpy(h).pin_memory()
    for chunks in (1, 2, 3, 4, 5, 8, 16):
        o_host = torch.full_like(h_host, float("nan")).pin_memory()
        od = torch.full_like(hd, float("nan"))
        st.step_host(h_host, o_host, torch.empty_like(hd), od, chunks=chunks)
        torch.cuda.synchronize()
        got = o_host.numpy()
        if np.array_equal(got, want):
            print(case, "chunks", chunks, "ok")
            continue
        d = ~np.isclose(got, want, rtol=0, atol=0) | np.isnan(got)
        d = d.reshape(shape.velocity_size, shape.n_theta, -1).any(axis=2)
        vs, ts = np.nonzero(d)
        print(case, "chunks", chunks, "MISMATCH: T", shape.n_theta, "M", shape.velocity_size,
              "planes", sorted(set(ts.tolist())), "rows", (vs.min(), vs.max()), "count", int(d.sum()),
              "nan", bool(np.isnan(got).any()))
