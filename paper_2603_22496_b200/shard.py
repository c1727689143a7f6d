"""Multi-GPU partitioning of the KK hot path.

One process per GPU (torchrun), ``torch.distributed`` for the plumbing:

* **Frame sharding** (config 4, ensembles): rank r owns the contiguous frame
  range ``frame_range(F, r, G)``; frames are independent, so there is no
  data-path collective — each rank runs ``KKEngine`` on its frames.
* **Row-block sharding** (config 5, one large frame): rank r owns the
  contiguous lateral block ``row_block_range(X, r, G)`` of the (X, Z) image.
  Stage 1 (decomposition, ~0.1 ms) is replicated on every rank; each rank
  gathers only its block's pixels with the K5 kernel over the block's rows of
  the delay tables.  Assembling the image is fused into that kernel
  (transport "p2p", the default): every rank maps the full-image buffers of
  all ranks with CUDA IPC and the gather epilogue stores each IQ pixel into
  all of them over NVLink (``kkb_kk_plan_run_scatter``), so the "all-gather"
  is the kernel's own stores plus one barrier.  Transport "nccl" all-gathers
  the complex64 blocks instead (and is the fallback when peer mapping is not
  available, or in the gloo CPU tests).  The per-pixel pair order does not
  depend on the partition, so the image is bit-identical to the single-GPU
  image for any world size and either transport.
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


def exchange_handles(local: bytes, group=None) -> list:
    """All ranks' 64-byte CUDA IPC handles, in rank order (host-side
    plumbing of the P2P transport; any process-group backend)."""
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized():
        return [local]
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, local, group=group)
    return out


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

    Every rank decomposes the whole frame (stage 1 replicated) and beamforms
    the rows ``row_block_range(X, rank, world)`` with the K5 kernel and the
    matching rows of the delay tables.  With transport "p2p" the kernel writes
    the rows straight into every rank's full-image buffer (CUDA IPC over
    NVLink); ``gather()`` then only waits (stream sync + barrier) and returns
    the local image, valid until the next ``beamform_block``.  With "nccl" the
    blocks are all-gathered after the kernel."""

    def __init__(self, array, params, receive, grid, rank: int, world: int, *,
                 interpolation: str = "linear", pulse_delay: float = 0.0,
                 transport: str = "auto", group=None):
        import ctypes

        from . import _device as dev
        from . import _lib
        from .beamform import build_kk_luts_device
        from .engine import KKEngine

        if transport not in ("auto", "p2p", "nccl"):
            raise ValueError(f"unknown transport {transport!r}")
        self.rank, self.world = rank, world
        self.grid = grid
        self.group = group
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
        self._img = None
        self._peers = []
        self.transport = "nccl"
        import torch.distributed as dist

        multi = dist.is_available() and dist.is_initialized()
        if transport in ("auto", "p2p") and world <= _lib.KKB_MAX_DST and (world == 1 or multi):
            try:
                self._setup_p2p()
                self.transport = "p2p"
            except Exception:
                if transport == "p2p":
                    raise
                self._release_p2p()

    def _setup_p2p(self):
        """Full-image buffer per rank, IPC handles exchanged, peers mapped."""
        import ctypes

        import torch

        from . import _lib

        nbytes = self.grid.nx * self.grid.nz * 8
        p = ctypes.c_void_p()
        _lib.call("kkb_ipc_alloc", nbytes, ctypes.byref(p))
        self._img = p
        h = ctypes.create_string_buffer(64)
        _lib.call("kkb_ipc_get_handle", p, h)
        handles = exchange_handles(h.raw, self.group)
        if len(handles) != self.world:
            raise RuntimeError("p2p transport needs one process per rank")
        dsts = [p.value]
        for r, hr in enumerate(handles):
            if r == self.rank:
                continue
            q = ctypes.c_void_p()
            _lib.call("kkb_ipc_open_handle", ctypes.create_string_buffer(hr, 64), ctypes.byref(q))
            self._peers.append(q)
            dsts.append(q.value)
        self._dsts = (ctypes.c_void_p * len(dsts))(*dsts)

        class _View:  # CUDA array interface over the raw allocation
            __cuda_array_interface__ = {"shape": (self.grid.nx, self.grid.nz), "typestr": "<c8",
                                        "data": (p.value, False), "version": 3, "strides": None}

        self.image = torch.as_tensor(_View(), device="cuda")

    def _release_p2p(self):
        from . import _lib

        lib = _lib.load()
        for q in self._peers:
            lib.kkb_ipc_close_handle(q)
        self._peers = []
        if self._img is not None:
            lib.kkb_ipc_free(self._img)
            self._img = None

    def beamform_block(self, rf, stream=None):
        """Stage 1 on the whole frame, K5 on this rank's rows; asynchronous.
        p2p: the rows land in every rank's image buffer."""
        from . import _device as dev
        from . import _lib

        self.engine.decompose(rf[None] if rf.dim() == 3 else rf, n_frames=1, stream=stream)
        if self._plan is None:
            return self.block[:0]
        if self.transport == "p2p":
            _lib.call("kkb_kk_plan_run_scatter", self._plan, dev.ptr(self.engine.traces), 1, 0,
                      self._dsts, len(self._dsts), self.ix0 * self.grid.nz, _lib.KKB_OUT_C64, 0,
                      dev.stream_handle(stream))
            return self.image[self.ix0:self.ix1]
        _lib.call("kkb_kk_plan_run", self._plan, dev.ptr(self.engine.traces), 1, 0,
                  dev.ptr(self.block), _lib.KKB_OUT_C64, 0, None, None,
                  dev.stream_handle(stream))
        return self.block[: self.rows]

    def gather(self, stream=None):
        """The full (X, Z) complex64 image on this rank."""
        import torch
        import torch.distributed as dist

        if self.transport == "p2p":
            (stream or torch.cuda.current_stream()).synchronize()
            if self.world > 1:
                dist.barrier(group=self.group)
            return self.image
        if self.world == 1:
            return self.block[: self.rows]
        return gather_row_blocks(self.block[: self.rows], self.grid.nx, self.grid.nz, self.group)

    def close(self):
        from . import _lib

        if self._plan is not None:
            _lib.load().kkb_kk_plan_destroy(self._plan)
            self._plan = None
        self._release_p2p()
        self.engine.close()
