"""world_size-2 gloo tests of the data-parallel host logic (CPU only): the
unique-id bootstrap broadcast, contiguous sharding, max-over-ranks timing, and
that per-rank shard gradients scaled by 1/B_global sum to the full-batch
gradient (the decomposition the NCCL path relies on; oracle arithmetic)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        from paper_1404_1521_b200 import dp
        out = {}
        uid = bytes(range(128)) if rank == 0 else b"\x00" * 128
        out["uid"] = dp.broadcast_bytes(uid, rank, 128)
        out["max"] = dp.max_over_ranks(float(rank + 1) * 1.5)
        V, d, n, h, B = 300, 8, 5, 16, 64
        p = oracle.Params.init(V, d, n, h, 7)
        idx, corr = synth.batch(V, n, B, seed=3)
        si, sc = dp.shard(idx, corr, rank, world)
        g = oracle.backward(p, si, sc, inv_batch=1.0 / B)
        dC = np.zeros_like(p.C)
        np.add.at(dC, g["rows"], g["Y"])
        flat = np.concatenate([dC.ravel(), g["dW1"].ravel(), g["db1"], g["dw2"], [g["db2"]]])
        out["grad"] = dp.sum_over_ranks(flat)
        full = oracle.backward(p, idx, corr)
        dCf = np.zeros_like(p.C)
        np.add.at(dCf, full["rows"], full["Y"])
        out["full"] = np.concatenate([dCf.ravel(), full["dW1"].ravel(), full["db1"], full["dw2"], [full["db2"]]])
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_dp_host_logic():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert res[r]["uid"] == bytes(range(128))
        assert res[r]["max"] == 3.0
        np.testing.assert_allclose(res[r]["grad"], res[r]["full"], rtol=1e-12, atol=1e-15)
    np.testing.assert_array_equal(res[0]["grad"], res[1]["grad"])


def test_shard_rejects_uneven():
    from paper_1404_1521_b200 import dp
    idx = np.zeros((10, 5), np.int32); corr = np.zeros(10, np.int32)
    with pytest.raises(ValueError):
        dp.shard(idx, corr, 0, 3)
    a, b = dp.shard(idx, corr, 1, 2)
    assert a.shape == (5, 5) and b.shape == (5,)
