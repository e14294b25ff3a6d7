"""DM-sharded multi-GPU driver (BASELINE config 4).

One process per GPU (torchrun), torch.distributed/NCCL for the plumbing.
Every DM row is independent and costs s*c additions, so rank r of N owns the
contiguous DM range shard_range(d, N, r): its shift-table slice is built on
its own device by K1 (dm_offset = first row, no table traffic at all), the
full input block arrives once (H2D on rank 0, then ONE broadcast -- the
path's only exchange, C1), and the rank writes its output rows in place.
Outputs stay resident (the paper's pipeline assumption) or are
gathered to rank 0 (C2) on request.  Because shards are disjoint rows, the
N-rank output equals the 1-rank output bit for bit.

The plumbing functions (shard_range, broadcast_input, gather_rows) take
plain torch tensors so they are exercised on CPU with the gloo backend
(tests/test_multi.py); the compute goes only through the CUDA library.
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
        self.ctx = api.context(self.device)
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

    @property
    def flop(self) -> int:
        """Additions this rank performs per pass."""
        return self.count * self.setup.samples_per_second * self.setup.channels

    def load(self, host_block: Optional[torch.Tensor]) -> None:
        """H2D on rank 0 (pinned host tensor [c][t]), then broadcast (C1)."""
        with torch.cuda.stream(self.stream):
            if self.rank == 0:
                assert host_block is not None
                self.block[:, : self.num_samples].copy_(host_block, non_blocking=True)
            broadcast_input(self.block, src=0)

    def run(self) -> torch.Tensor:
        """One pass of this rank's DM range, enqueued on self.stream."""
        self.plan.execute(self.block.data_ptr(), self.out.data_ptr())
        return self.out

    def pipeline(self, chunks: int, channel_groups: int = 4, h2d: str = "auto") -> None:
        """Prepare run_host(): the shard's DM range cut into `chunks` plans
        (tile-aligned), each over its slice of the shift table, so the D2H of
        chunk i overlaps the kernel of chunk i+1.  The block goes H2D either
        in time order (h2d="time"; single rank): chunk i starts once the
        samples its delays reach have landed -- the low-DM chunks need little
        more than the first second -- so output leaves the device while the
        block's tail is still arriving; or (h2d="channels"; staged families)
        in `channel_groups` channel ranges, the kernels of group g
        accumulating through the output (bit-exact) under the H2D of group
        g+1.  "auto": time order on a single rank."""
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
        self.h2d_mode = h2d if h2d != "auto" else ("time" if self.world == 1 else "channels")
        if self.world > 1:
            self.h2d_mode = "channels"
        if self.h2d_mode == "time":
            # samples chunk i may read: its largest shift + s, plus one tile of
            # slack for a predicated last tile and the 16-byte copy rounding
            # (chunks are cut in DM order; the running maximum keeps the
            # uploads in time order for any table)
            tt = self.cfg.tile_time()
            self.uploads, upto = [], 0
            for lo, hi, _, _ in self.chunks:
                md = int(self.shifts[lo:hi].max().item())
                upto = max(upto, min(self.num_samples, s + md + tt + 8))
                self.uploads.append((upto, torch.cuda.Event()))
            g = 1
        else:
            g = max(1, min(channel_groups, c)) if (staged and self.world == 1) else 1
        self.groups = [(c * i // g, c * (i + 1) // g, torch.cuda.Event()) for i in range(g)]
        self.h2d_stream = torch.cuda.Stream(self.device)
        self.copy_stream = torch.cuda.Stream(self.device)
        self._d2h_done = [[]]  # stream_host's per-chunk events follow the new cut

    def run_host(self, host_block: Optional[torch.Tensor], host_out: torch.Tensor) -> None:
        """End to end from host memory: the block's channel groups go H2D on
        their own stream (or, with several ranks, H2D + broadcast); the
        kernels of channel group g start as soon as its rows landed; each DM
        chunk's output rows go D2H as soon as its last kernel is done.
        host_out: pinned [count][s]."""
        t = self.num_samples
        if self.h2d_mode == "time":
            with torch.cuda.stream(self.h2d_stream):
                done_t = 0
                for upto, ev in self.uploads:
                    if upto > done_t:
                        self.ctx.upload_block_range(host_block.data_ptr(), t,
                                                    self.block.data_ptr(), self.pitch,
                                                    self.setup.channels, done_t, upto,
                                                    self.h2d_stream.cuda_stream)
                        done_t = upto
                    ev.record(self.h2d_stream)
            for (lo, hi, plan, done), (_, ev) in zip(self.chunks, self.uploads):
                self.stream.wait_event(ev)  # the samples this chunk reads have landed
                plan.execute(self.block.data_ptr(), self.out[lo].data_ptr())
                done.record(self.stream)
                with torch.cuda.stream(self.copy_stream):
                    self.copy_stream.wait_event(done)
                    host_out[lo:hi].copy_(self.out[lo:hi], non_blocking=True)
            self.copy_stream.synchronize()
            return
        if len(self.groups) == 1:
            self.load(host_block)
        else:
            with torch.cuda.stream(self.h2d_stream):
                for c0, c1, ev in self.groups:
                    self.block[c0:c1, :t].copy_(host_block[c0:c1], non_blocking=True)
                    ev.record(self.h2d_stream)
        for gi, ci in self.launch_order():
            c0, c1, ev = self.groups[gi]
            lo, hi, plan, done = self.chunks[ci]
            if len(self.groups) == 1:
                plan.execute(self.block.data_ptr(), self.out[lo].data_ptr())
            else:
                self.stream.wait_event(ev)  # group gi's rows have landed
                plan.execute_channels(self.block.data_ptr(), self.out[lo].data_ptr(), c0, c1,
                                      accumulate=gi > 0)
            if gi == len(self.groups) - 1:
                done.record(self.stream)
                with torch.cuda.stream(self.copy_stream):
                    self.copy_stream.wait_event(done)
                    host_out[lo:hi].copy_(self.out[lo:hi], non_blocking=True)
        self.copy_stream.synchronize()

    def stream_host(self, host_blocks, host_outs, steps: int) -> None:
        """A survey's steady state: `steps` consecutive blocks, each through
        the run_host(time) path, double-buffered on the device so block i+1's
        H2D and kernels overlap block i's D2H (PCIe is full duplex; the D2H
        of the output is the larger transfer).  Block i comes from
        host_blocks[i % len(host_blocks)] and its rows land in
        host_outs[i % 2] (pinned [count][s]); every block is copied in and
        read back in full.  Single rank, h2d="time" (pipeline() first)."""
        if self.world != 1 or self.h2d_mode != "time":
            raise ValueError("stream_host needs a single rank and pipeline(h2d='time')")
        if len(host_outs) != 2:
            raise ValueError("stream_host needs two host output buffers")
        n = len(self.chunks)
        if getattr(self, "_bufs", None) is None:
            c, s = self.setup.channels, self.setup.samples_per_second
            blk2 = torch.empty((c, self.pitch), dtype=torch.float32, device=self.device)
            out2 = torch.empty((self.count, s), dtype=torch.float32, device=self.device)
            self._bufs = [(self.block, self.out), (blk2, out2)]
        if len(getattr(self, "_d2h_done", [[]])[0]) != n:  # pipeline() re-cut the chunks
            # per buffer: kernels done reading the block, D2H done per chunk
            self._read_done = [torch.cuda.Event(), torch.cuda.Event()]
            self._d2h_done = [[torch.cuda.Event() for _ in range(n)] for _ in range(2)]
        t = self.num_samples
        for i in range(steps):
            b = i % 2
            block, out = self._bufs[b]
            hb, ho = host_blocks[i % len(host_blocks)], host_outs[b]
            with torch.cuda.stream(self.h2d_stream):
                if i >= 2:  # block b is free once step i-2's kernels are done
                    self.h2d_stream.wait_event(self._read_done[b])
                done_t = 0
                for upto, ev in self.uploads:
                    if upto > done_t:
                        self.ctx.upload_block_range(hb.data_ptr(), t, block.data_ptr(),
                                                    self.pitch, self.setup.channels, done_t,
                                                    upto, self.h2d_stream.cuda_stream)
                        done_t = upto
                    ev.record(self.h2d_stream)
            for j, ((lo, hi, plan, done), (_, ev)) in enumerate(zip(self.chunks, self.uploads)):
                self.stream.wait_event(ev)
                if i >= 2:  # rows lo:hi of out b have left for the host
                    self.stream.wait_event(self._d2h_done[b][j])
                plan.execute(block.data_ptr(), out[lo].data_ptr())
                done.record(self.stream)
                with torch.cuda.stream(self.copy_stream):
                    self.copy_stream.wait_event(done)
                    ho[lo:hi].copy_(out[lo:hi], non_blocking=True)
                    self._d2h_done[b][j].record(self.copy_stream)
            self._read_done[b].record(self.stream)
        self.copy_stream.synchronize()

    def launch_order(self):
        """(channel group, DM chunk) kernel order for run_host.  No chunk can
        go D2H before the whole block is on the device, so the first
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
