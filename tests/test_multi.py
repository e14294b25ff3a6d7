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

from paper_1601_05052_b200.multi import (allgather_channels, broadcast_input, channel_groups,
                                         gather_rows, rank_part, shard_range)


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


def test_channel_groups_split_evenly_over_ranks():
    assert channel_groups(1024, 8, 2) == [(0, 512), (512, 1024)]
    assert channel_groups(32, 8, 4) == [(0, 8), (8, 16), (16, 24), (24, 32)]
    assert channel_groups(32, 8, 8) == [(0, 8), (8, 16), (16, 24), (24, 32)]  # 1 row/rank min
    assert channel_groups(12, 3, 4) == [(0, 3), (3, 6), (6, 9), (9, 12)]
    assert channel_groups(10, 4, 2) == []  # not divisible: the caller broadcasts
    for c, n, g in [(1024, 8, 4), (32, 2, 3), (24, 3, 5)]:
        groups = channel_groups(c, n, g)
        assert groups[0][0] == 0 and groups[-1][1] == c
        for c0, c1 in groups:
            parts = [rank_part(c0, c1, n, r) for r in range(n)]
            assert parts[0][0] == c0 and parts[-1][1] == c1
            assert all(p1 - p0 == (c1 - c0) // n for p0, p1 in parts)


def _allgather_worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    setup, d, align = O.Setup("mini", 64, 12, 100.0, 25.0, 0.0, 0.5), 24, 4
    t, _, _ = O.instance_sizing(setup, d)
    host = torch.from_numpy(O.noise(setup.channels, t, 1.0, 3))  # every rank's copy
    block = torch.full((setup.channels, t + 3), float("nan"))  # pitched rows
    for c0, c1 in channel_groups(setup.channels, world, 2):
        p0, p1 = rank_part(c0, c1, world, rank)
        block[p0:p1, :t] = host[p0:p1]  # only this rank's share is "uploaded"
        allgather_channels(block, c0, c1)
    off, cnt = shard_range(d, world, rank, align)
    full_sh, _ = O.delay_table(setup, d)
    local = torch.from_numpy(O.dedisperse_reference(np.ascontiguousarray(block[:, :t].numpy()),
                                                    full_sh[off:off + cnt], 64))
    out = gather_rows(local, d, align)
    if rank == 0:
        assert torch.equal(block[:, :t], host)
        ref = O.dedisperse_reference(host.numpy(), full_sh, 64)
        np.save(result_path, np.stack([out.numpy(), ref]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_upload_allgather(tmp_path, world):
    """C1 as the e2e path runs it at N>1: each rank holds only its share of
    every channel group, the in-place all-gather assembles the block, and
    the gathered rows equal the one-process output bit for bit."""
    path = str(tmp_path / "r.npy")
    mp.start_processes(_allgather_worker, args=(world, _free_port(), path), nprocs=world,
                       start_method="spawn")
    got, ref = np.load(path)
    assert got.tobytes() == ref.tobytes()


def test_bench_launcher_spawns_ranks():
    """bench.py --gpus 2 outside torchrun re-launches itself with 2 ranks
    (torch.distributed.run, 127.0.0.1); --plumbing-check runs the rank
    setup, sharded upload + all-gather and row gather on gloo."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--plumbing-check"],
                       cwd=root, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line == {"plumbing": "ok", "n_gpus": 2, "world_size": 2,
                    "channel_groups": [[0, 4], [4, 8], [8, 12], [12, 16]],
                    "block_assembled": True, "rows_gathered": 48}
    # inside a torchrun environment the world size must match --gpus
    env = dict(os.environ, WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2"], cwd=root, env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 2 and "WORLD_SIZE=3" in r.stderr
