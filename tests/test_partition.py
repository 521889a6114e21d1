"""Host logic of the multi-GPU chain decomposition (no GPU): the parts tile the windows, interfaces match,
right-open parts are aligned to 256-segment blocks; and the same checks across a real gloo world of 2."""
import os

import numpy as np
import pytest

from mabd_scenes import generators as G


@pytest.fixture(scope="module")
def lib():
    from paper_2603_08079_b200 import build
    build.build()
    from paper_2603_08079_b200 import binding
    return binding


def _check_parts(infos):
    W = len(infos)
    assert all(i["parts"] == W for i in infos)
    nw = infos[0]["windows"]
    assert infos[0]["win_lo"] == 0 and infos[-1]["win_hi"] == nw
    for a, b in zip(infos[:-1], infos[1:]):
        assert a["win_hi"] == b["win_lo"] and a["long_hi"] == b["long_lo"]
        assert a["right_open"] == b["left_open"]
    for i in infos:
        n1 = i["long_hi"] - i["long_lo"]
        if i["right_open"]:
            assert n1 <= 256 or n1 % 256 == 0
        assert i["seq_unknowns"] <= 256


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_partition_long_chain(lib, world):
    sc = G.cfg3_long_chain(col_len=2000, n_cols=35, tail=7)
    infos = [lib.partition_info(sc, world, r) for r in range(world)]
    _check_parts(infos)
    assert sum(i["right_open"] for i in infos) == world - 1     # one chain: every boundary splits it


def test_partition_full_cfg3_balanced(lib):
    sc = G.cfg3_long_chain()
    for world in (2, 4, 8):
        infos = [lib.partition_info(sc, world, r) for r in range(world)]
        _check_parts(infos)
        sizes = [i["long_hi"] - i["long_lo"] for i in infos]
        assert max(sizes) - min(sizes) <= 256 + 1


def test_partition_independent_chains_no_interfaces(lib):
    sc = G.cfg2_batched_chains(64, 256)
    infos = [lib.partition_info(sc, 4, r) for r in range(4)]
    _check_parts(infos)
    assert not any(i["left_open"] or i["right_open"] for i in infos)
    assert [i["win_hi"] - i["win_lo"] for i in infos] == [16, 16, 16, 16]


def _gloo_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from paper_2603_08079_b200 import binding
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = G.cfg3_long_chain(col_len=3000, n_cols=40, tail=5)
    mine = binding.partition_info(sc, world, rank)
    got = [None] * world
    dist.all_gather_object(got, mine)
    ok = True
    try:
        _check_parts(got)
    except AssertionError:
        ok = False
    # the rank-0 NCCL unique id travels through the process group the way bench.py ships it
    blob = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        blob = torch.frombuffer(bytearray(os.urandom(128)), dtype=torch.uint8).clone()
    dist.broadcast(blob, src=0)
    blobs = [None] * world
    dist.all_gather_object(blobs, bytes(blob.tolist()))
    ok = ok and all(b == blobs[0] for b in blobs)
    out.put((rank, ok))
    dist.destroy_process_group()


def test_gloo_world2_partition_consistency(lib):
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


# ----------------------------------------------------------------------------- tree split

def _check_tree_parts(infos):
    W = len(infos)
    assert all(i["solver"] == 2 and i["tree_parts"] == W for i in infos)
    ng = infos[0]["groups"]
    assert infos[0]["group_lo"] == 0 and infos[-1]["group_hi"] == ng
    for a, b in zip(infos[:-1], infos[1:]):
        assert a["group_hi"] == b["group_lo"] and a["body_hi"] == b["body_lo"]
    for i in infos:
        assert i["group_hi"] - i["group_lo"] <= i["groups_per_part"]
        assert i["slots_per_part"] * W >= i["root_joints"]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_partition_tree_cfg4(lib, world):
    """Config 4 at full size: 128 CTA-local subtrees of 511 bodies (the larger group size: 65,535 bodies give every
    SM a group) below a 127-body top, split evenly."""
    sc = G.cfg4_binary_tree(16)
    infos = [lib.partition_info(sc, world, r) for r in range(world)]
    _check_tree_parts(infos)
    assert infos[0]["groups"] == 128 and infos[0]["root_joints"] == 128
    assert all(i["body_hi"] - i["body_lo"] == 511 * 128 // world for i in infos)
    assert infos[0]["slots_per_part"] == 128 // world


def _gloo_tree_worker(rank, world, port, out):
    import torch.distributed as dist
    from paper_2603_08079_b200 import binding
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sc = G.cfg4_binary_tree(12)
    got = [None] * world
    dist.all_gather_object(got, binding.partition_info(sc, world, rank))
    ok = True
    try:
        _check_tree_parts(got)
    except AssertionError:
        ok = False
    out.put((rank, ok))
    dist.destroy_process_group()


def test_gloo_world2_tree_partition_consistency(lib):
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_gloo_tree_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}
