"""Multi-process (world size 2, gloo, CPU) tests of the slot-sharding host
logic used by bench.py under torchrun (static contiguous
partition, no data-path collective, results gathered to rank 0, timings
reduced with MAX)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2206_05998_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, out_dir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        seeds = shard.slot_seeds(total, world, rank)
        # stand-in per-slot device results: (seed, K=3 bit-error counters)
        local = np.stack([seeds.astype(np.int64), seeds.astype(np.int64) % 7,
                          seeds.astype(np.int64) % 5, seeds.astype(np.int64) % 3], axis=1)
        got = shard.gather_to_rank0(local)
        t = shard.max_over_ranks(1.5 + rank)
        if rank == 0:
            np.save(os.path.join(out_dir, "gathered.npy"), got)
            np.save(os.path.join(out_dir, "tmax.npy"), np.array([t]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total", [37, 2, 296])
def test_two_rank_partition_gather_and_max(tmp_path, total):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), total, str(tmp_path)), nprocs=world, join=True)
    got = np.load(tmp_path / "gathered.npy")
    assert got.shape == (total, 4)
    assert np.array_equal(got[:, 0], np.arange(1000, 1000 + total))  # every slot once, in order
    assert np.array_equal(got[:, 1], got[:, 0] % 7)
    assert float(np.load(tmp_path / "tmax.npy")[0]) == 2.5


def test_partition_covers_every_slot_once():
    for total in (0, 1, 7, 148, 32768):
        for world in (1, 2, 3, 4, 8):
            spans = [shard.slot_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.slot_range(10, 2, 2)
