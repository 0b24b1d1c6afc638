"""e2e (host-buffer steps, overlapped) with the pinned host buffers first-touched
from each NUMA node's CPUs in turn -- does the placement matter on this box?
    python tools/e2e_numa.py"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2305_10553_b200.grid import make_case, random_state_device  # noqa: E402
from paper_2305_10553_b200.kernels import make_kernel_inputs  # noqa: E402
from paper_2305_10553_b200.step import Stepper  # noqa: E402


def node_cpus():
    nodes = {}
    base = Path("/sys/devices/system/node")
    for d in sorted(base.glob("node[0-9]*")):
        cpus = set()
        for part in (d / "cpulist").read_text().strip().split(","):
            if "-" in part:
                a, b = part.split("-")
                cpus.update(range(int(a), int(b) + 1))
            elif part:
                cpus.add(int(part))
        nodes[int(d.name[4:])] = cpus & os.sched_getaffinity(0)
    return {k: v for k, v in nodes.items() if v}


def gpu_numa():
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        bus = pynvml.nvmlDeviceGetPciInfo(h).busId
        bus = bus.decode() if isinstance(bus, bytes) else bus
        p = Path(f"/sys/bus/pci/devices/{bus.lower()[-12:]}/numa_node")
        return int(p.read_text()) if p.exists() else None, bus
    except Exception as e:  # noqa: BLE001
        return None, str(e)


shape = make_case("sh03b")
dev = torch.device("cuda", 0)
st = Stepper(shape, make_kernel_inputs(shape, 1234), 1.5e-9, device=dev)
h = random_state_device(shape, 1234, dev)
pairs = [(torch.empty_like(h), torch.empty_like(h)) for _ in range(2)]
allcpu = os.sched_getaffinity(0)
print("gpu numa node / bus:", gpu_numa(), "nodes:", {k: len(v) for k, v in node_cpus().items()})
for node, cpus in node_cpus().items():
    os.sched_setaffinity(0, cpus)
    hh = torch.empty(h.shape, dtype=h.dtype, pin_memory=True)
    oh = torch.empty(h.shape, dtype=h.dtype, pin_memory=True)
    hh.copy_(h)
    oh.zero_()
    for rep in range(2):
        st.step_host(hh, oh, *pairs[0], overlap=True)
        st.step_host_join()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(6):
            st.step_host(hh, oh, *pairs[i % 2], overlap=True)
        st.step_host_join()
        e1.record()
        torch.cuda.synchronize()
        print(f"node {node}: e2e {e0.elapsed_time(e1) / 6:.1f} ms/step", flush=True)
    del hh, oh
os.sched_setaffinity(0, allcpu)
