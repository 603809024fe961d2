"""Multi-GPU host logic on CPU: world_size-2 gloo process groups run the
(window, restart) sharding of the sweep with the CPU oracle as the per-unit
worker and must reproduce the single-process result exactly.
"""
import os
import socket

import numpy as np
import pytest

from paper_2204_12346_b200 import sharding


def test_partition_is_balanced_and_exact():
    for n in (0, 1, 7, 139, 1000):
        for world in (1, 2, 3, 8):
            parts = [sharding.partition(n, world, r) for r in range(world)]
            assert sum(len(p) for p in parts) == n
            assert [i for p in parts for i in p] == list(range(n))
            sizes = [len(p) for p in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        sharding.partition(5, 2, 2)


def test_merge_by_index_rejects_gaps():
    assert sharding.merge_by_index([[(1, "b")], [(0, "a"), (2, "c")]]) == ["a", "b", "c"]
    with pytest.raises(ValueError):
        sharding.merge_by_index([[(0, "a")], [(2, "c")]])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _unit_result(w, restart, series):
    from oracle import oracle_py
    from paper_2204_12346_b200.sirdfit import mix_seed
    ora = oracle_py.load("port")
    I, R, D = series
    a = 3 * w
    sl = slice(a, a + 21)
    N = 38e6
    init = [N - I[a] - R[a] - D[a], I[a], R[a], D[a]]
    rc, best, cost, hist = ora.fit_swarm("ird-mxse", I[sl], R[sl], D[sl], init, N, [0] * 6,
                                         [2, 2, 13, 13, 1, 0.1], 24, 4,
                                         seed=mix_seed(sharding.restart_seed(2204, restart), w))
    return (rc, best.tobytes(), cost, hist.tobytes())


def _worker(rank, world, port, series, out_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    units = sharding.units(6, 2)
    # the library's runner: each rank computes its contiguous share in one call
    merged = sharding.run_sharded(len(units), lambda idx: [_unit_result(*units[i], series) for i in idx])
    # max-over-ranks timing reduction, as bench.py does over NCCL
    import torch
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        out_q.put((merged, float(t.item())))
    dist.destroy_process_group()


def test_two_rank_gloo_sweep_matches_single_process(poland):
    import torch.multiprocessing as mp
    series = (poland["I"], poland["R"], poland["D"])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, series, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged, tmax = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0
    want = [_unit_result(w, r, series) for (w, r) in sharding.units(6, 2)]
    assert merged == want
