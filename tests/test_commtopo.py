"""B200 NVSwitch communication model: the topology file parses in
the reference's format and the predicted transposes match the volumes of
SURVEY.md §8 (e) (commsim.alltoall_volume with n1 = G) at 900 GB/s per GPU."""
import pytest

from paper_2305_10553_b200.commtopo import alltoall_bytes, b200_node, load_topology, step_comm_seconds
from paper_2305_10553_b200.grid import make_case


def test_b200_topology_file():
    t = b200_node()
    assert (t.gpus_per_node, t.intra_node_links, t.intra_link_gbps, t.nic_layout) == (8, 8, 900.0, "per_gpu")


@pytest.mark.parametrize("world, gb, ms", [(2, 1.70, 1.89), (4, 1.27, 1.42), (8, 0.743, 0.83)])
def test_sh03b_transposes(world, gb, ms):
    shape = make_case("sh03b")
    assert alltoall_bytes(shape, world) / 1e9 == pytest.approx(gb, rel=5e-3)
    r = step_comm_seconds(shape, world)
    assert r["alltoall_s"] * 1e3 == pytest.approx(ms, rel=1e-2)
    assert r["step_s"] == pytest.approx(2 * r["alltoall_s"] + r["allgather_s"])


def test_single_rank_and_bad_world():
    assert step_comm_seconds(make_case("sh03b"), 1)["step_s"] == 0.0
    with pytest.raises(ValueError):
        step_comm_seconds(make_case("sh03b"), 16)


def test_topology_errors(tmp_path):
    p = tmp_path / "t.txt"
    p.write_text("gpus_per_node = 8\n")
    with pytest.raises(ValueError, match="missing topology fields"):
        load_topology(p)
    p.write_text("bogus = 1\n")
    with pytest.raises(ValueError, match="unknown topology field"):
        load_topology(p)
