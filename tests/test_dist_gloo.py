"""N>1 host-side logic on CPU (gloo, world_size 2): the handle exchange the
NVLink communicator uses, and the 3D-parallel group plan the hybrid policy
builds its per-dimension communicators from."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_2409_02423_b200 import ParallelLayout
    from paper_2409_02423_b200.dist import exchange_handles
    from paper_2409_02423_b200.hybrid import plan_groups

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # opaque per-rank blobs (HCCX_HANDLE_BYTES = 256) gathered in rank order
        blob = bytes([rank]) * 256
        got = exchange_handles(blob)
        assert [b[0] for b in got] == list(range(world)) and all(len(b) == 256 for b in got)
        # group plan for dp=2 (pp=tp=1) and the subgroups built from it
        lay = ParallelLayout(dp=world, pp=1, tp=1)
        plan = plan_groups(lay)
        assert plan["dp"] == [tuple(range(world))]
        assert plan["tp"] == [(r,) for r in range(world)]
        groups = {}
        for kind, gs in plan.items():
            for ranks in gs:
                pg = dist.new_group(list(ranks)) if len(ranks) > 1 else None
                if rank in ranks:
                    groups[kind] = (ranks, pg)
        t = torch.tensor([rank + 1.0])
        dist.all_reduce(t, group=groups["dp"][1])
        assert t.item() == sum(range(1, world + 1))
        # group-scoped exchange (what NvlinkComm does for a sub-communicator)
        got = exchange_handles(bytes([10 + rank]) * 8, groups["dp"][1])
        assert [b[0] for b in got] == [10 + r for r in range(world)]
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange_and_groups():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_plan_groups_3d():
    from paper_2409_02423_b200 import ParallelLayout
    from paper_2409_02423_b200.hybrid import plan_groups

    lay = ParallelLayout(dp=2, pp=3, tp=4)
    plan = plan_groups(lay)
    assert len(plan["dp"]) == 12 and len(plan["tp"]) == 6 and len(plan["pp"]) == 8
    for kind in plan:
        covered = sorted(r for g in plan[kind] for r in g)
        assert covered == list(range(24)), kind  # each dimension partitions the world
    assert (4, 5, 6, 7) in plan["tp"] and (5, 17) in plan["dp"] and (1, 5, 9) in plan["pp"]
