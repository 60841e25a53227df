"""Host logic of the multi-GPU batched mode, on CPU with gloo,
world size 2 (and 3 for uneven blocks): scenario shards partition the scenario list in
order, the timing reduction is the max over ranks, the final gather reassembles the
per-scenario fields in scenario order."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1707_03581_b200 import dist as D
from paper_1707_03581_b200 import inputs as I


def test_shard_range_partitions():
    for n in (0, 1, 5, 63, 64, 65):
        for world in (1, 2, 3, 8):
            blocks = [D.shard_range(n, r, world) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            for (lo, hi), (lo2, _) in zip(blocks, blocks[1:]):
                assert hi == lo2
            sizes = [hi - lo for lo, hi in blocks]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        D.shard_range(4, 2, 2)


def test_shard_config_keeps_meshes():
    cfg = I.make_config("cfg4", n_scen=5)
    parts = [D.shard_config(cfg, r, 2) for r in range(2)]
    assert [p.n_scen for p in parts] == [3, 2]
    assert parts[0].fixed is cfg.fixed and parts[1].moving is cfg.moving
    assert parts[0].scenarios + parts[1].scenarios == cfg.scenarios
    with pytest.raises(ValueError):
        D.shard_config(I.make_config("cfg4", n_scen=1), 1, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_scen, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = D.shard_range(n_scen, rank, world)
        # per-scenario "field": row s is s * 10 + arange(4) (only this rank's block)
        local = np.stack([s * 10.0 + np.arange(4.0) for s in range(lo, hi)])
        full = D.gather_scenarios(local, n_scen)
        tmax = D.max_over_ranks(1.5 + rank)
        tsum = D.sum_over_ranks(float(hi - lo))
        q.put((rank, full.tolist(), tmax, tsum))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_scen", [(2, 64), (2, 5), (3, 7)])
def test_gloo_shard_gather_max(world, n_scen):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_scen, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = np.stack([s * 10.0 + np.arange(4.0) for s in range(n_scen)])
    for rank, full, tmax, tsum in res:
        np.testing.assert_array_equal(np.array(full), expect)
        assert tmax == 1.5 + (world - 1)
        assert tsum == n_scen
