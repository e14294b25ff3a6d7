"""Streaming block ingest.

The reference dedisperses one padded 1-s block (setup.cpp:130-133).  A live
pipeline receives consecutive seconds of data; output second n needs input
samples [n*s, (n+1)*s + max_delay).  BlockStream keeps, per channel, a ring
row of t + R*s samples (t = instance_sizing's num_samples, R = ceil(t/s)):
each push appends one second behind the current window, the window start
advances by s (the plan runs on the window through an offset pointer, no
copy), and only when the row is used up is the window's tail moved to the
front -- once every R pushes, between non-overlapping ranges.  Once the
window holds t samples every push yields the dedispersed output of its
first second -- identical, bit for bit, to a one-shot pass over the same
samples (same kernel, same data, same order).
"""
from __future__ import annotations

from typing import Optional

import torch

from . import api


class BlockStream:
    def __init__(self, setup: api.ObservationSetup, num_dms: int, cfg: api.KernelConfig,
                 dm_tile_depth: int = 1, staging: str = "auto", device: int = 0,
                 gpu_tiling: bool = False, stage_channels: int = 0):
        self.setup, self.num_dms = setup, num_dms
        c, s = setup.channels, setup.samples_per_second
        self.s, self.c = s, c
        self.t = api.instance_sizing(setup, num_dms).num_samples
        # ring rows of t + R*s samples; the window start advances by s, so the
        # staged kernels' 16-byte alignment needs s % 4 == 0 (else compact on
        # every push, through a temporary)
        self.ring = s % 4 == 0
        self.rounds = -(-self.t // s) if self.ring else 0
        self.pitch = (self.t + self.rounds * s + 3) // 4 * 4
        self.ctx = api.Context(device)  # own context: its stream is this stream's
        self.stream = torch.cuda.Stream(device)
        self.ctx.set_stream(self.stream.cuda_stream)
        self.shifts = torch.empty((num_dms, c), dtype=torch.int32, device=device)
        self.ctx.delay_table(setup, num_dms, self.shifts.data_ptr())
        self.window = torch.zeros((c, self.pitch), dtype=torch.float32, device=device)
        self.out = torch.empty((num_dms, s), dtype=torch.float32, device=device)
        self.plan = self.ctx.plan(self.shifts.data_ptr(), c, num_dms, s, self.t, self.pitch, cfg,
                                  dm_tile_depth, staging, gpu_tiling=gpu_tiling,
                                  stage_channels=stage_channels)
        self.start = 0        # window start within the ring row
        self.filled = 0       # samples per channel currently in the window
        self.emitted = 0      # output seconds produced so far
        self.compactions = 0  # tail moves to the row front (once per R pushes)

    def push(self, second: torch.Tensor) -> Optional[torch.Tensor]:
        """Append one second ([channels][s], host or device).  Returns the
        [num_dms][s] output of the window's first second once the window is
        full (a view into a buffer reused by the next push), else None."""
        if tuple(second.shape) != (self.c, self.s):
            raise ValueError(f"expected a [{self.c}][{self.s}] block")
        with torch.cuda.stream(self.stream):
            if self.filled == self.t:  # slide: drop the oldest second
                self.start += self.s
                self.filled -= self.s
                if not self.ring:
                    tail = self.window[:, self.start: self.start + self.filled].clone()
                    self.window[:, : self.filled].copy_(tail)
                    self.start = 0
                    self.compactions += 1
            if self.start + self.filled + self.s > self.pitch:
                # row used up: move the window's tail to the front (the ranges
                # do not overlap: start >= R*s >= t - s = filled)
                assert self.start >= self.filled
                self.window[:, : self.filled].copy_(
                    self.window[:, self.start: self.start + self.filled])
                self.start = 0
                self.compactions += 1
            end = self.start + self.filled
            self.window[:, end: end + self.s].copy_(second, non_blocking=True)
            self.filled += self.s
            if self.filled < self.t:
                return None
            self.plan.execute(self.window.data_ptr() + 4 * self.start, self.out.data_ptr())
        self.emitted += 1
        return self.out
