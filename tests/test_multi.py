"""The N>1 plumbing of the DM-sharded driver on CPU with gloo, world size 2.

The shard layout, the input broadcast (C1) and the row gather (C2) are the
product's own functions (paper_1601_05052_b200.multi); the per-shard compute,
which needs a GPU, is stood in for by the test oracle, and the assembled
result must equal the single-process oracle output bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1601_05052_b200.multi import gather_rows, shard_range, broadcast_input


def test_shard_range_partitions_evenly():
    for d, n, a in [(4096, 8, 64), (4096, 3, 8), (12, 4, 3), (7, 7, 1), (64, 2, 1)]:
        ranges = [shard_range(d, n, r, a) for r in range(n)]
        assert ranges[0][0] == 0
        for (o1, c1), (o2, _) in zip(ranges, ranges[1:]):
            assert o1 + c1 == o2
        assert sum(c for _, c in ranges) == d
        assert all(c % a == 0 for _, c in ranges)
        assert max(c for _, c in ranges) - min(c for _, c in ranges) <= a
    with pytest.raises(ValueError):
        shard_range(100, 2, 0, 64)
    with pytest.raises(ValueError):
        shard_range(64, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    setup, d, align = O.Setup("mini", 64, 8, 100.0, 25.0, 0.0, 0.5), 24, 4
    t, _, _ = O.instance_sizing(setup, d)
    block = torch.from_numpy(O.noise(setup.channels, t, 1.0, 3)) if rank == 0 else \
        torch.zeros((setup.channels, t), dtype=torch.float32)
    broadcast_input(block, src=0)
    off, cnt = shard_range(d, world, rank, align)
    full_sh, _ = O.delay_table(setup, d)
    local = torch.from_numpy(O.dedisperse_reference(block.numpy(), full_sh[off:off + cnt], 64))
    out = gather_rows(local, d, align)
    if rank == 0:
        ref = O.dedisperse_reference(block.numpy(), full_sh, 64)
        np.save(result_path, np.stack([out.numpy(), ref]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_broadcast_shard_gather(tmp_path, world):
    path = str(tmp_path / "r.npy")
    mp.start_processes(_worker, args=(world, _free_port(), path), nprocs=world,
                       start_method="spawn")
    got, ref = np.load(path)
    assert got.tobytes() == ref.tobytes()
