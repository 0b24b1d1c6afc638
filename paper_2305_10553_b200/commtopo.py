"""Communication model of the multi-GPU step on a B200 NVSwitch node (SURVEY.md
§8 f4): the reference's analytic all-to-all / all-reduce model (commsim.py) applied
to the transposes dist.py actually performs, with a B200 topology file in the
reference's own key=value format (topologies/b200_nvswitch.txt, readable by
`gyroproxy comm-estimate --topo-file` as well).

Only the single-node case is modelled here (G <= gpus_per_node, one rank per GPU):
every peer is then on the same node and on another GPU, so the reference's
traffic split (commsim.py:270-300) puts everything in the intra-node share and a
collective moving B bytes per rank costs B / (intra fabric / active ranks)
(commsim.py:303-328) -- here additionally capped at one GPU's own link bandwidth,
since on NVSwitch a GPU never exceeds its 900 GB/s however few peers are active
(the reference's equal-share model would give 3.6 TB/s per rank at G = 2).
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path

from .grid import GridShape

TOPOLOGIES = Path(__file__).resolve().parent / "topologies"
GB = 1e9
_INTS = {"gpus_per_node", "intra_node_links", "nics_per_node", "processes_per_gpu"}
_FLOATS = {"intra_link_gbps", "nic_bandwidth", "shared_bus_latency_penalty", "shared_bus_contention"}
_REQUIRED = {"gpus_per_node", "intra_node_links", "intra_link_gbps", "nic_layout", "nics_per_node", "nic_bandwidth"}


@dataclass(frozen=True)
class Topology:
    name: str
    gpus_per_node: int
    intra_node_links: int
    intra_link_gbps: float
    nic_layout: str
    nics_per_node: int
    nic_bandwidth: float
    processes_per_gpu: int = 1
    shared_bus_latency_penalty: float = 2e-6
    shared_bus_contention: float = 1.5

    @property
    def intra_aggregate_gbps(self) -> float:
        return self.intra_node_links * self.intra_link_gbps


def load_topology(path) -> Topology:
    """key=value file, '#' comments; the reference's fields and errors (commsim.py:124-156)."""
    fields: dict = {}
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, 1):
            line = raw.split("#", 1)[0].strip()
            if not line:
                continue
            if "=" not in line:
                raise ValueError(f"{path}:{lineno}: expected key=value, got {line!r}")
            key, _, value = line.partition("=")
            key, value = key.strip(), value.strip()
            if key in _INTS:
                fields[key] = int(value)
            elif key in _FLOATS:
                fields[key] = float(value)
            elif key in ("name", "nic_layout"):
                fields[key] = value
            else:
                raise ValueError(f"{path}:{lineno}: unknown topology field {key!r}")
    missing = _REQUIRED - fields.keys()
    if missing:
        raise ValueError(f"{path}: missing topology fields: {', '.join(sorted(missing))}")
    fields.setdefault("name", str(path))
    return Topology(**fields)


def b200_node() -> Topology:
    return load_topology(TOPOLOGIES / "b200_nvswitch.txt")


def alltoall_bytes(shape: GridShape, world: int) -> float:
    """Bytes each rank sends per transpose: S/G * (G-1)/G (commsim.alltoall_volume, n1 = G)."""
    return shape.state_bytes / world * (world - 1) / world


def step_comm_seconds(shape: GridShape, world: int, topo: Topology | None = None) -> dict:
    """Predicted seconds of the collectives of one dist.py step on one node: two
    all-to-all transposes (home -> velocity layout and back) and the phi
    all-gather ((G-1)/G of the field per rank)."""
    topo = topo or b200_node()
    if world < 1 or world > topo.gpus_per_node * topo.processes_per_gpu:
        raise ValueError(f"{world} ranks do not fit one {topo.name} node")
    if world == 1:
        return {"alltoall_bytes": 0.0, "alltoall_s": 0.0, "allgather_s": 0.0, "step_s": 0.0}
    # the rank's share of the intra fabric, capped at its own link
    bw = min(topo.intra_aggregate_gbps / world, topo.intra_link_gbps) * GB
    a2a = alltoall_bytes(shape, world)
    ag = shape.field_bytes * (world - 1) / world
    return {"alltoall_bytes": a2a, "alltoall_s": a2a / bw, "allgather_s": ag / bw,
            "step_s": 2 * a2a / bw + ag / bw}
