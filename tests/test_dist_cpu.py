"""World-size-2 gloo tests on CPU for the multi-process host logic: the
rendezvous that orders ranks by cluster id, and duplicate-id rejection."""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cids, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2401_01728_b200.dist import rendezvous
    from paper_2401_01728_b200.errors import ConfigError

    try:
        everyone, order, pos = rendezvous({"cid": cids[rank], "src": (b"h%d" % rank, 16 * rank)})
        q.put((rank, [e["cid"] for e in everyone], order, pos, everyone[order[0]]["src"]))
    except ConfigError as e:
        q.put((rank, "ConfigError", str(e)))
    dist.destroy_process_group()


def _run(world, cids):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cids, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    return sorted(out, key=lambda t: t[0])


def test_rendezvous_orders_by_cluster_id():
    out = _run(2, [7, 3])
    for rank, cids, order, pos, first_src in out:
        assert cids == [7, 3]
        assert order == [1, 0]          # position 0 = cluster 3 = rank 1
        assert pos == (1 if rank == 0 else 0)
        assert first_src == (b"h1", 16)


def test_rendezvous_rejects_duplicate_ids():
    out = _run(2, [5, 5])
    assert all(o[1] == "ConfigError" for o in out)


def _vote_worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2401_01728_b200.dist import agree_bind_live, agree_layouts
    from paper_2401_01728_b200.errors import ConfigError, LayoutError

    try:
        if case == "layout-same":
            agree_layouts((16384, 435328, 102, 166))
        elif case == "layout-differ":  # e.g. a rank with another SM count
            agree_layouts((16384, 435328, 102, 166 if rank == 0 else 83))
        elif case == "live-all":
            agree_bind_live(None, True)
        elif case == "live-some":
            agree_bind_live(None, rank == 0)
        elif case == "live-bad":
            agree_bind_live("live must match the parameter buffer's dtype and device" if rank == 1 else None, True)
        q.put((rank, "ok"))
    except ConfigError as e:
        q.put((rank, "ConfigError", str(e)))
    except LayoutError as e:
        q.put((rank, "LayoutError", str(e)))
    dist.destroy_process_group()


def _vote(case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_vote_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    return sorted(out, key=lambda t: t[0])


@pytest.mark.parametrize("case,want", [("layout-same", "ok"), ("layout-differ", "ConfigError"),
                                       ("live-all", "ok"), ("live-some", "ConfigError"),
                                       ("live-bad", "LayoutError")])
def test_collective_agreement_raises_on_every_rank(case, want):
    """DistRingGroup's layout check and the bind_live vote: every rank ends
    with the same verdict (no rank left waiting in a collective)."""
    out = _vote(case)
    assert [o[1] for o in out] == [want, want], out
    if want == "LayoutError":
        assert all("rank 1" in o[2] for o in out)


def test_auto_protocol_thresholds():
    """'auto' transport choice (dist.choose_protocol): a function of the
    bytes per cluster, dtype and rank count only, so every rank agrees."""
    from paper_2401_01728_b200.dist import choose_protocol

    mib = 1 << 20
    assert choose_protocol("auto", 4 * mib) == "ll"
    assert choose_protocol("auto", 4 * mib, fp32=False) == "pull"
    assert choose_protocol("auto", 16 * mib, n_ranks=4) == "pull"
    assert choose_protocol("auto", 32 * mib, n_ranks=4) == "push"
    assert choose_protocol("auto", 102 * mib, n_ranks=2) == "pull"   # ResNet-50 at 2 GPUs
    assert choose_protocol("auto", 438 * mib, n_ranks=2) == "push"   # BERT-base at 2 GPUs
    assert choose_protocol("auto", 102 * mib, n_ranks=8) == "push"
    assert choose_protocol("pull", 1 << 30) == "pull"
    with pytest.raises(Exception):
        choose_protocol("nvls", 1)
