"""DM-sharded multi-GPU driver (BASELINE config 4).

One process per GPU (torchrun), torch.distributed/NCCL for the plumbing.
Every DM row is independent and costs s*c additions, so rank r of N owns the
contiguous DM range shard_range(d, N, r): its shift-table slice is built on
its own device by K1 (dm_offset = first row, no table traffic at all), the
full input block arrives once per pass, and the rank writes its output rows
in place.  The block's one exchange (C1) is an all-gather of channel slices:
every rank uploads only its 1/N share of each channel group over its own
PCIe link and NCCL assembles the group on every GPU over NVLink, so the
per-rank H2D shrinks with N and the kernels of a group start as soon as it
has landed (accumulating through the output across groups: bit-exact, see
dd_plan_execute_channels).  A rank-0 H2D + broadcast remains for callers
that hold the block on one rank only.  Outputs stay resident (the paper's
pipeline assumption), go back to each rank's host over its own
link, or are gathered to rank 0 (C2).  Because shards are disjoint rows, the
N-rank output equals the 1-rank output bit for bit.

The plumbing functions (shard_range, channel_groups, allgather_channels,
broadcast_input, gather_rows) take plain torch tensors so they are exercised
on CPU with the gloo backend (tests/test_multi.py); the compute goes only
through the CUDA library.
"""
from __future__ import annotations

import os
from typing import List, Optional, Tuple

import numpy as np
import torch
import torch.distributed as dist

from . import api


def world() -> Tuple[int, int]:
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def shard_range(num_dms: int, world_size: int, rank: int, align: int = 1) -> Tuple[int, int]:
    """Contiguous DM range (offset, count) of `rank`.  Units of `align` rows
    (the config's tile_dm) are dealt out as evenly as possible, earlier ranks
    taking the remainder, so every shard stays tileable."""
    if world_size < 1 or not 0 <= rank < world_size:
        raise ValueError("bad rank/world size")
    if align < 1 or num_dms % align != 0:
        raise ValueError(f"tile_dm {align} does not divide the trial count {num_dms}")
    units = num_dms // align
    base, extra = divmod(units, world_size)
    start = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return start * align, count * align


def channel_groups(channels: int, world_size: int, groups: int) -> List[Tuple[int, int]]:
    """Channel groups [c0, c1) for the sharded upload: at most `groups`
    equal groups whose width splits evenly over the ranks (rank r uploads
    the r-th 1/N of every group).  Empty when the channels do not split
    over the ranks (the caller then falls back to a broadcast)."""
    if channels % world_size != 0:
        return []
    g = max(1, min(groups, channels // world_size))
    while channels % (g * world_size) != 0:
        g -= 1
    w = channels // g
    return [(i * w, (i + 1) * w) for i in range(g)]


def rank_part(c0: int, c1: int, world_size: int, rank: int) -> Tuple[int, int]:
    """Rank `rank`'s rows of channel group [c0, c1)."""
    per = (c1 - c0) // world_size
    return c0 + rank * per, c0 + (rank + 1) * per


def allgather_channels(block: torch.Tensor, c0: int, c1: int, group=None) -> None:
    """C1, sharded: rows [c0, c1) of the channel-major block (rows contiguous)
    assembled in place on every rank from each rank's equal part (NCCL over
    NVLink on the GPU box, gloo on CPU in tests)."""
    rank, n = world()
    if n == 1:
        return
    rows = block[c0:c1]
    p0, p1 = rank_part(c0, c1, n, rank)
    dist.all_gather_into_tensor(rows.reshape(-1), block[p0:p1].reshape(-1), group=group)


def broadcast_input(block: torch.Tensor, src: int = 0, group=None) -> torch.Tensor:
    """C1: the filterbank block from `src` to every rank (NCCL over NVLink on
    the GPU box, gloo on CPU in tests)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(block, src=src, group=group)
    return block


def gather_rows(local: torch.Tensor, num_dms: int, align: int = 1, dst: int = 0,
                group=None) -> Optional[torch.Tensor]:
    """C2: assemble the DM-major output on `dst` from every rank's rows.
    Shards may differ in size, so ranks send padded blocks and `dst` trims."""
    rank, n = world()
    if n == 1:
        return local
    counts = [shard_range(num_dms, n, r, align)[1] for r in range(n)]
    width = local.shape[1]
    pad = torch.zeros((max(counts), width), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(n)] if rank == dst else None
    dist.gather(pad, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)


class ShardedDedisperser:
    """This rank's share of one dedispersion instance on its GPU."""

    def __init__(self, setup: api.ObservationSetup, num_dms: int, cfg: api.KernelConfig,
                 dm_tile_depth: int = 1, staging: str = "auto", device: Optional[int] = None,
                 gpu_tiling: bool = False, stage_channels: int = 0, flags: int = 0):
        """flags: raw DD_CONFIG_* bits (as in tuning records), OR-ed with the
        gpu_tiling / stage_channels arguments."""
        self.rank, self.world = world()
        self.setup, self.num_dms, self.cfg = setup, num_dms, cfg
        self.device = torch.cuda.current_device() if device is None else device
        torch.cuda.set_device(self.device)
        self.offset, self.count = shard_range(num_dms, self.world, self.rank, cfg.tile_dm())
        inst = api.instance_sizing(setup, num_dms)
        self.num_samples = inst.num_samples
        self.pitch = (self.num_samples + 3) // 4 * 4
        c, s = setup.channels, setup.samples_per_second
        # a context of its own (not the per-device api.context() singleton):
        # the library launches on the context's stream, so two drivers sharing
        # one context would move each other's kernels off their own streams
        self.ctx = api.Context(self.device)
        # one dedicated stream shared by the library, torch copies and NCCL;
        # callers run under `with torch.cuda.stream(dd.stream)`
        self.stream = torch.cuda.Stream(self.device)
        self.ctx.set_stream(self.stream.cuda_stream)
        self.shifts = torch.empty((self.count, c), dtype=torch.int32, device=self.device)
        self.max_delay = self.ctx.delay_table(setup, self.count, self.shifts.data_ptr(),
                                              dm_offset=self.offset)
        self.block = torch.empty((c, self.pitch), dtype=torch.float32, device=self.device)
        self.out = torch.empty((self.count, s), dtype=torch.float32, device=self.device)
        self._depth, self._staging, self._gpu_tiling, self._cps, self._flags = (
            dm_tile_depth, staging, gpu_tiling, stage_channels, flags)
        self.plan = self.ctx.plan(self.shifts.data_ptr(), c, self.count, s, self.num_samples,
                                  self.pitch, cfg, dm_tile_depth, staging,
                                  gpu_tiling=gpu_tiling, stage_channels=stage_channels,
                                  flags=flags)
        self._bufs = None

    @property
    def flop(self) -> int:
        """Additions this rank performs per pass."""
        return self.count * self.setup.samples_per_second * self.setup.channels

    def load(self, host_block: Optional[torch.Tensor]) -> None:
        """Put a pinned host block [c][t] on every rank's device.  Every rank
        holding the block: each uploads its channel share and one all-gather
        assembles it (C1, sharded); only rank 0 holding it: H2D on rank 0 and
        one broadcast."""
        t = self.num_samples
        with torch.cuda.stream(self.stream):
            have = torch.tensor([0 if host_block is None else 1], device=self.device)
            if self.world > 1:
                dist.all_reduce(have, op=dist.ReduceOp.MIN)
            parts = channel_groups(self.setup.channels, self.world, 1)
            if self.world > 1 and int(have.item()) == 1 and parts:
                p0, p1 = rank_part(0, self.setup.channels, self.world, self.rank)
                self.block[p0:p1, :t].copy_(host_block[p0:p1], non_blocking=True)
                allgather_channels(self.block, 0, self.setup.channels)
            else:
                if self.rank == 0:
                    assert host_block is not None
                    self.block[:, :t].copy_(host_block, non_blocking=True)
                broadcast_input(self.block, src=0)

    def run(self) -> torch.Tensor:
        """One pass of this rank's DM range, enqueued on self.stream."""
        self.plan.execute(self.block.data_ptr(), self.out.data_ptr())
        return self.out

    def pipeline(self, chunks: int, channel_groups_: int = 4, h2d: str = "auto") -> None:
        """Prepare run_host()/stream_host(): the shard's DM range cut into
        `chunks` plans (tile-aligned), each over its slice of the shift table,
        so the D2H of chunk i overlaps the kernel of chunk i+1.  The block
        arrives by one of three routes:
          "time"     (single rank) in time order: chunk i starts once the
                     samples its delays reach have landed -- the low-DM chunks
                     need little more than the first second -- so output leaves
                     the device while the block's tail is still arriving;
          "channels" (single rank, staged families) in channel groups, the
                     kernels of group g accumulating through the output
                     (bit-exact) under the H2D of group g+1;
          "sharded"  (N ranks) each rank uploads its 1/N of every channel
                     group and an all-gather assembles the group (C1), the
                     group's kernels starting as soon as it is complete;
          "broadcast" (N ranks, channels not divisible by N) rank 0 uploads
                     the block and broadcasts it.
        "auto": time order on one rank, sharded on several."""
        c, s, td = self.setup.channels, self.setup.samples_per_second, self.cfg.tile_dm()
        units = self.count // td
        chunks = max(1, min(chunks, units))
        self.chunks = []
        for i in range(chunks):
            lo = (units * i // chunks) * td
            hi = (units * (i + 1) // chunks) * td
            plan = self.ctx.plan(self.shifts.data_ptr() + lo * c * 4, c, hi - lo, s,
                                 self.num_samples, self.pitch, self.cfg, self._depth,
                                 self._staging, gpu_tiling=self._gpu_tiling,
                                 stage_channels=self._cps, flags=self._flags)
            self.chunks.append((lo, hi, plan, torch.cuda.Event()))
        staged = self.chunks[0][2].info()["family"] in ("smem", "regwin", "tmem")
        if h2d == "auto":
            h2d = "time" if self.world == 1 else "sharded"
        if self.world > 1 and h2d in ("time", "channels"):
            h2d = "sharded"
        if self.world == 1 and h2d == "broadcast":
            h2d = "time"
        # (h2d="sharded" on one rank runs the N-rank route with N = 1 -- the
        # channel-group uploads, per-group events and accumulating kernels,
        # with the all-gather a no-op: how tests exercise it on one GPU)
        groups = []
        if h2d == "sharded":
            groups = channel_groups(c, self.world, channel_groups_ if staged else 1)
            if not groups:
                h2d = "broadcast"
        if h2d == "broadcast":
            groups = [(0, c)]
        self.h2d_mode = h2d
        self.uploads = []
        if h2d == "time":
            # samples chunk i may read: its largest shift + s, plus one tile of
            # slack for a predicated last tile and the 16-byte copy rounding
            # (chunks are cut in DM order; the running maximum keeps the
            # uploads in time order for any table)
            tt = self.cfg.tile_time()
            upto = 0
            for lo, hi, _, _ in self.chunks:
                md = int(self.shifts[lo:hi].max().item())
                upto = max(upto, min(self.num_samples, s + md + tt + 8))
                self.uploads.append((upto, torch.cuda.Event()))
            groups = [(0, c)]
        elif h2d == "channels":
            g = max(1, min(channel_groups_, c)) if staged else 1
            groups = [(c * i // g, c * (i + 1) // g) for i in range(g)]
        # per group: H2D landed, group complete on this device (after C1)
        self.groups = [(c0, c1, torch.cuda.Event(), torch.cuda.Event()) for c0, c1 in groups]
        self.h2d_stream = torch.cuda.Stream(self.device)
        self.copy_stream = torch.cuda.Stream(self.device)
        self.comm_stream = torch.cuda.Stream(self.device)
        # per device buffer: kernels done reading the block, D2H done per chunk
        self._read_done = [torch.cuda.Event(), torch.cuda.Event()]
        self._d2h_done = [[torch.cuda.Event() for _ in self.chunks] for _ in range(2)]
        self._used = [False, False]

    def h2d_bytes(self) -> int:
        """Bytes this rank copies host -> device per block on the pipeline's
        route (samples no DM reads are not shipped in time order)."""
        c, t = self.setup.channels, self.num_samples
        if self.h2d_mode == "time":
            return c * self.uploads[-1][0] * 4
        if self.h2d_mode == "sharded":
            return sum(rank_part(c0, c1, self.world, self.rank)[1] -
                       rank_part(c0, c1, self.world, self.rank)[0]
                       for c0, c1, _, _ in self.groups) * t * 4
        if self.h2d_mode == "broadcast":
            return c * t * 4 if self.rank == 0 else 0
        return c * t * 4

    def d2h_bytes(self) -> int:
        return self.count * self.setup.samples_per_second * 4

    def _enqueue(self, b: int, host_block: torch.Tensor, host_out: torch.Tensor) -> None:
        """One block through the pipeline on device buffer pair b: input
        (H2D, plus C1 on several ranks), kernels, D2H of each chunk's rows as
        soon as they are final.  Waits only on the previous use of the same
        buffers (double buffering)."""
        block, out = self._bufs[b]
        reuse = self._used[b]
        t, c = self.num_samples, self.setup.channels
        if self.h2d_mode == "time":
            with torch.cuda.stream(self.h2d_stream):
                if reuse:  # block b is free once its previous kernels are done
                    self.h2d_stream.wait_event(self._read_done[b])
                done_t = 0
                for upto, ev in self.uploads:
                    if upto > done_t:
                        self.ctx.upload_block_range(host_block.data_ptr(), t, block.data_ptr(),
                                                    self.pitch, c, done_t, upto,
                                                    self.h2d_stream.cuda_stream)
                        done_t = upto
                    ev.record(self.h2d_stream)
            for j, ((lo, hi, plan, done), (_, ev)) in enumerate(zip(self.chunks, self.uploads)):
                self.stream.wait_event(ev)  # the samples this chunk reads have landed
                if reuse:  # rows lo:hi of out b have left for the host
                    self.stream.wait_event(self._d2h_done[b][j])
                plan.execute(block.data_ptr(), out[lo].data_ptr())
                self._emit(j, b, out, host_out)
            self._read_done[b].record(self.stream)
            self._used[b] = True
            return
        # channel groups: H2D (this rank's part, or all of it), then C1
        with torch.cuda.stream(self.h2d_stream):
            if reuse:
                self.h2d_stream.wait_event(self._read_done[b])
            for c0, c1, landed, _ in self.groups:
                if self.h2d_mode == "sharded":
                    p0, p1 = rank_part(c0, c1, self.world, self.rank)
                elif self.h2d_mode == "broadcast":
                    p0, p1 = (c0, c1) if self.rank == 0 else (c0, c0)
                else:
                    p0, p1 = c0, c1
                if p1 > p0:
                    block[p0:p1, :t].copy_(host_block[p0:p1], non_blocking=True)
                landed.record(self.h2d_stream)
        comm = self.h2d_mode in ("sharded", "broadcast")
        if comm:
            with torch.cuda.stream(self.comm_stream):
                for c0, c1, landed, ready in self.groups:
                    self.comm_stream.wait_event(landed)
                    if self.h2d_mode == "sharded":
                        allgather_channels(block, c0, c1)
                    else:
                        broadcast_input(block, src=0)
                    ready.record(self.comm_stream)
        ng = len(self.groups)
        waited = set()
        for gi, ci in self.launch_order():
            c0, c1, landed, ready = self.groups[gi]
            lo, hi, plan, done = self.chunks[ci]
            self.stream.wait_event(ready if comm else landed)  # group gi is on this device
            if reuse and ci not in waited:
                self.stream.wait_event(self._d2h_done[b][ci])
                waited.add(ci)
            if ng == 1:
                plan.execute(block.data_ptr(), out[lo].data_ptr())
            else:
                plan.execute_channels(block.data_ptr(), out[lo].data_ptr(), c0, c1,
                                      accumulate=gi > 0)
            if gi == ng - 1:
                self._emit(ci, b, out, host_out)
        self._read_done[b].record(self.stream)
        self._used[b] = True

    def _emit(self, j: int, b: int, out: torch.Tensor, host_out: torch.Tensor) -> None:
        """Chunk j's rows are final: D2H on the copy stream."""
        lo, hi, _, done = self.chunks[j]
        done.record(self.stream)
        with torch.cuda.stream(self.copy_stream):
            self.copy_stream.wait_event(done)
            host_out[lo:hi].copy_(out[lo:hi], non_blocking=True)
            self._d2h_done[b][j].record(self.copy_stream)

    def _buffers(self) -> None:
        if self._bufs is None:
            c, s = self.setup.channels, self.setup.samples_per_second
            blk2 = torch.empty((c, self.pitch), dtype=torch.float32, device=self.device)
            out2 = torch.empty((self.count, s), dtype=torch.float32, device=self.device)
            self._bufs = [(self.block, self.out), (blk2, out2)]

    def run_host(self, host_block: Optional[torch.Tensor], host_out: torch.Tensor) -> None:
        """End to end from host memory, one block (pipeline() first): input
        by the pipeline's route, each chunk's kernels as soon as their input
        landed, each chunk's rows D2H as soon as they are final.  host_block:
        pinned [c][t] (sharded: every rank's copy; broadcast: rank 0's);
        host_out: pinned [count][s]."""
        self._buffers()
        self._enqueue(0, host_block, host_out)
        self.copy_stream.synchronize()

    def stream_host(self, host_blocks, host_outs, steps: int) -> None:
        """A survey's steady state: `steps` consecutive blocks, double-buffered
        on the device so block i+1's input route (H2D, C1) and kernels overlap
        block i's D2H (PCIe is full duplex; the D2H of the output is the larger
        transfer).  Block i comes from host_blocks[i % len(host_blocks)] and
        its rows land in host_outs[i % 2] (pinned [count][s]); every sample a
        kernel reads is copied in and every output row is read back."""
        if len(host_outs) != 2:
            raise ValueError("stream_host needs two host output buffers")
        self._buffers()
        for i in range(steps):
            self._enqueue(i % 2, host_blocks[i % len(host_blocks)], host_outs[i % 2])
        self.copy_stream.synchronize()

    def launch_order(self):
        """(channel group, DM chunk) kernel order for the grouped routes.  No
        chunk can go D2H before the whole block is on the device, so the first
        `lead` chunks run their leading channel groups while the later
        groups are still in flight; after that each chunk is finished and
        handed to the copy stream in turn, so the D2H of the output (the
        larger transfer) starts as soon as the H2D ends.  Per output the
        groups still run in ascending channel order (bit-exact)."""
        n, g = len(self.chunks), len(self.groups)
        lead = n if g == 1 else max(1, (n + 1) // 2)
        order, done = [], set()
        for gi in range(g - 1):
            for ci in range(lead):
                order.append((gi, ci))
                done.add((gi, ci))
        for ci in range(n):
            for gi in range(g):
                if (gi, ci) not in done:
                    order.append((gi, ci))
        return order

    def gather(self) -> Optional[torch.Tensor]:
        with torch.cuda.stream(self.stream):
            return gather_rows(self.out, self.num_dms, self.cfg.tile_dm())
