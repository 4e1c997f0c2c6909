"""Host logic of the split verifier / speculator run on CPU:
role assignment, branch sharding, counter merging, and the mailbox-handle
exchange over a real 2-process gloo group (127.0.0.1)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2603_03251_b200 import split
from paper_2603_03251_b200 import _native as N
from paper_2603_03251_b200.api import ConfigError


def test_roles():
    assert [split.role_of(r, 5, tp=2) for r in range(5)] == [N.ROLE_VERIFIER] * 2 + [N.ROLE_SPECULATOR] * 3
    with pytest.raises(ConfigError):
        split.role_of(0, 2, tp=2)
    assert split.role_of(0, 2) == N.ROLE_VERIFIER
    assert [split.role_of(r, 4) for r in range(1, 4)] == [N.ROLE_SPECULATOR] * 3
    with pytest.raises(ConfigError):
        split.role_of(0, 1)
    with pytest.raises(ConfigError):
        split.role_of(3, 3)


@pytest.mark.parametrize("B", [0, 1, 5, 20, 33, 80])
@pytest.mark.parametrize("G", [1, 2, 3, 7])
def test_branch_blocks_partition_every_branch_once(B, G):
    seen = []
    sizes = []
    for g in range(G):
        lo, n = split.branch_block(B, g, G)
        sizes.append(n)
        seen.extend(range(lo, lo + n))
    assert seen == list(range(B))
    assert max(sizes) - min(sizes) <= 1
    for b in range(B):
        lo, n = split.branch_block(B, split.branch_owner(b, B, G), G)
        assert lo <= b < lo + n


def _stats(**kw):
    d = {k: 0 for k in split.COUNTERS}
    d.update(device_ms=1.0, kernel_launches=10)
    d.update(kw)
    return d


def test_merge_stats():
    v = _stats(tokens=30, accepted_sum=20.0, rounds=10, device_ms=5.0)
    s = _stats(tokens=30, accepted_sum=20.0, rounds=10, primary_origin_lookups=9, primary_origin_hits=7, device_ms=6.0)
    m = split.merge_stats([v, s, dict(s)])
    assert m["primary_origin_hits"] == 7 and m["tokens"] == 30
    assert m["device_ms"] == 6.0 and m["kernel_launches"] == 30
    with pytest.raises(ConfigError):
        split.merge_stats([v, s, _stats(tokens=30, accepted_sum=20.0, rounds=10, primary_origin_hits=6)])
    with pytest.raises(ConfigError):
        split.merge_stats([_stats(tokens=31, accepted_sum=20.0, rounds=10), s])
    # tensor-parallel verifier ranks must agree
    assert split.merge_stats([v, dict(v), s], tp=2)["primary_origin_hits"] == 7
    with pytest.raises(ConfigError):
        split.merge_stats([v, _stats(tokens=29, accepted_sum=20.0, rounds=10), s], tp=2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _exchange_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        h = bytes([rank]) * N.MAILBOX_HANDLE_BYTES
        got = split.exchange_handles(h)
        q.put((rank, [g[0] for g in got], [len(g) for g in got], split.role_of(rank, world)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_handle_exchange_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, order, lens, role in res:
        assert order == list(range(world)) and lens == [N.MAILBOX_HANDLE_BYTES] * world
        assert role == (N.ROLE_VERIFIER if rank == 0 else N.ROLE_SPECULATOR)
