"""The NCCL branch of the sharded-allocation collective (dist.gather_records,
SURVEY §8(e)) on the one GPU a test box has: a world-1 NCCL process group
runs the same all_gather_into_tensor of the device records (rank-to-rank
exchange needs more GPUs: the multi-rank logic is covered with gloo,
tests/test_dist_gloo.py, and with virtual ranks, tests/test_gpu_parity.py)."""
import socket

import pytest
import torch

import workloads as W
from oracle import coracle as co
from oracle import mapa_oracle as mo

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.fixture
def nccl_world1():
    import torch.distributed as tdist
    store = tdist.TCPStore("127.0.0.1", _free_port(), 1, True)
    tdist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        yield tdist.group.WORLD
    finally:
        tdist.destroy_process_group()


def test_nccl_gather_records_narrow_and_deep(nccl_world1):
    import paper_2110_03214_b200 as mp
    from paper_2110_03214_b200 import dist as md
    t = mp.Topology(text=W.het32_text())
    busy = 0xF0F00000
    for shape, k in (("ring", 5), ("full", 4)):
        p = mp.Pattern.make(shape, k)
        for sel, sens in ((0, False), (1, True), (1, False)):
            rec, _q = md.run_query(t, p, sel, sens, busy, raw=True)
            out = md.gather_records(rec, 4, nccl_world1)
            torch.cuda.synchronize()
            assert out.shape == (1, 4) and out.device.type == "cuda"
            assert torch.equal(out[0], rec)
            r = md.reduce_records(md.records_from_tensor(out))
            d = md.decode(t, p, busy, sel, sens, r, raw=True)
            kk, ee = mo.make_pattern(shape, k)
            o = co.allocate(mo.parse_topology(W.het32_text()), busy, kk, ee, sel, sens)
            for f in ("devices", "mapping", "used_edges", "raw"):
                assert d[f] == o[f], (shape, k, sel, sens, f)
            assert d["leaves"] == o["raw"]
    p = mp.Pattern.make("ring", 9)
    t16 = mp.Topology("cubemesh16")
    rec, _q = md.run_query_wide(t16, p, 0, False, 0x00F0, raw=True)
    out = md.gather_records(rec, 8, nccl_world1)
    torch.cuda.synchronize()
    assert out.shape == (1, 8) and torch.equal(out[0], rec)
