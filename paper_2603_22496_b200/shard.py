"""Multi-GPU partitioning of the KK hot path.

One process per GPU (torchrun), ``torch.distributed`` for the plumbing:

* **Frame sharding** (config 4, ensembles): rank r owns the contiguous frame
  range ``frame_range(F, r, G)``; frames are independent, so there is no
  data-path collective — each rank runs ``KKEngine`` on its frames.
* **Row-block sharding** (config 5, one large frame): rank r owns the
  contiguous lateral block ``row_block_range(X, r, G)`` of the (X, Z) image.
  Stage 1 (decomposition, ~0.1 ms) is replicated on every rank; each rank
  gathers only its block's pixels with the K5 kernel over the block's rows of
  the delay tables; the complex64 blocks are then all-gathered (NCCL over
  NVLink on GPUs, gloo in the CPU tests).  The per-pixel pair order does not
  depend on the partition, so the gathered image is bit-identical to the
  single-GPU image for any world size.
"""

from __future__ import annotations

import numpy as np


def balanced_range(count: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [begin, end) share of `count` items for `rank` of `world`
    (sizes differ by at most one, larger shares first)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(count, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def frame_range(n_frames: int, rank: int, world: int) -> tuple[int, int]:
    """Frames [begin, end) processed by `rank` (ensemble sharding)."""
    return balanced_range(n_frames, rank, world)


def row_block_range(nx: int, rank: int, world: int) -> tuple[int, int]:
    """Lateral rows ix in [begin, end) of the (X, Z) image owned by `rank`."""
    return balanced_range(nx, rank, world)


def gather_row_blocks(block, nx: int, nz: int, group=None):
    """All-gather the per-rank (rows, nz) complex64 blocks into the full
    (nx, nz) image on every rank.  `block` is a torch tensor on the process
    group's device (CUDA for NCCL, CPU for gloo)."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rows_max = max(e - b for b, e in (row_block_range(nx, r, world) for r in range(world)))
    send = torch.zeros((rows_max, nz), dtype=block.dtype, device=block.device)
    send[: block.shape[0]].copy_(block)
    recv = torch.empty((world * rows_max, nz), dtype=block.dtype, device=block.device)
    # complex payloads travel as float pairs (NCCL has no complex type)
    dist.all_gather_into_tensor(torch.view_as_real(recv).reshape(-1),
                                torch.view_as_real(send).reshape(-1), group=group)
    parts = []
    for r in range(world):
        b, e = row_block_range(nx, r, world)
        parts.append(recv[r * rows_max: r * rows_max + (e - b)])
    return torch.cat(parts, dim=0)


class RowBlockKK:
    """Config-5 style single-frame KK beamforming split by image row-block.

    Every rank decomposes the whole frame (stage 1 replicated), beamforms the
    rows ``row_block_range(X, rank, world)`` with the K5 kernel and the
    matching rows of the delay tables, then ``gather()`` assembles the image."""

    def __init__(self, array, params, receive, grid, rank: int, world: int, *,
                 interpolation: str = "linear", pulse_delay: float = 0.0):
        import ctypes

        from . import _device as dev
        from . import _lib
        from .beamform import build_kk_luts_device
        from .engine import KKEngine

        self.rank, self.world = rank, world
        self.grid = grid
        self.ix0, self.ix1 = row_block_range(grid.nx, rank, world)
        self.engine = KKEngine(array, params, receive, grid, frames=1, want_db=False,
                               interpolation=interpolation, pulse_delay=pulse_delay)
        t = dev.require_cuda()
        N, M, T = params.num_transmits, receive.num_angles, params.num_samples
        luts = build_kk_luts_device(grid, params.transmit_angles, receive.angles, params.sound_speed)
        rows = self.ix1 - self.ix0
        self.rows = rows
        self.block = t.empty((max(rows, 1), grid.nz), dtype=t.complex64, device="cuda")
        self._plan = None
        if rows > 0:
            ltx = luts["lut_tx_x"][self.ix0:self.ix1].contiguous()
            lrx = luts["lut_rx_x"][self.ix0:self.ix1].contiguous()
            kp = ctypes.c_void_p()
            _lib.call("kkb_kk_plan_create", dev.ptr(ltx), dev.ptr(luts["lut_tx_z"]), dev.ptr(lrx),
                      dev.ptr(luts["lut_rx_z"]), N, M, T, rows, grid.nz, None,
                      float(self.engine.fs), float(self.engine.shift),
                      int(interpolation == "linear"), dev.stream_handle(), ctypes.byref(kp))
            self._plan = kp
        self._keep = (luts,)

    def beamform_block(self, rf, stream=None):
        """Stage 1 on the whole frame, K5 on this rank's rows; asynchronous."""
        from . import _device as dev
        from . import _lib

        self.engine.decompose(rf[None] if rf.dim() == 3 else rf, n_frames=1, stream=stream)
        if self._plan is not None:
            _lib.call("kkb_kk_plan_run", self._plan, dev.ptr(self.engine.traces), 1, 0,
                      dev.ptr(self.block), _lib.KKB_OUT_C64, 0, None, None,
                      dev.stream_handle(stream))
        return self.block[: self.rows]

    def gather(self, group=None):
        return gather_row_blocks(self.block[: self.rows], self.grid.nx, self.grid.nz, group)

    def close(self):
        from . import _lib

        if self._plan is not None:
            _lib.load().kkb_kk_plan_destroy(self._plan)
            self._plan = None
        self.engine.close()
