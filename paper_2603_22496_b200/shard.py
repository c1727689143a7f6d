"""Multi-GPU partitioning of the KK hot path.

One process per GPU (torchrun), ``torch.distributed`` for the plumbing:

* **Frame sharding** (config 4, ensembles): rank r owns the contiguous frame
  range ``frame_range(F, r, G)``; frames are independent, so there is no
  data-path collective — each rank runs ``KKEngine`` on its frames.
* **Row-block sharding** (config 5, one large frame): rank r owns the
  contiguous lateral block ``row_block_range(X, r, G)`` of the (X, Z) image.
  Stage 1 (decomposition, ~0.13 ms) is replicated on every rank (default), or
  split by transmit with the trace all-gather fused into the inverse FFT's
  epilogue (``stage1="sharded"``, P2P stores into every rank's trace buffer);
  each rank gathers only its block's pixels with the K5 kernel over the block's rows of
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


def _gather_dim0(block, count: int, group=None):
    """All-gather per-rank blocks of a dim-0 array split by balanced_range."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rows_max = max(e - b for b, e in (balanced_range(count, r, world) for r in range(world)))
    rest = tuple(block.shape[1:])
    send = torch.zeros((rows_max,) + rest, dtype=block.dtype, device=block.device)
    send[: block.shape[0]].copy_(block)
    recv = torch.empty((world * rows_max,) + rest, dtype=block.dtype, device=block.device)
    # complex payloads travel as float pairs (NCCL has no complex type)
    real = (lambda x: torch.view_as_real(x)) if block.is_complex() else (lambda x: x)
    dist.all_gather_into_tensor(real(recv).reshape(-1), real(send).reshape(-1), group=group)
    parts = []
    for r in range(world):
        b, e = balanced_range(count, r, world)
        parts.append(recv[r * rows_max: r * rows_max + (e - b)])
    return torch.cat(parts, dim=0)


def gather_row_blocks(block, nx: int, nz: int, group=None):
    """All-gather the per-rank (rows, nz) complex64 blocks into the full
    (nx, nz) image on every rank.  `block` is a torch tensor on the process
    group's device (CUDA for NCCL, CPU for gloo)."""
    if tuple(block.shape[1:]) != (nz,):
        raise ValueError("block must be (rows, nz)")
    return _gather_dim0(block, nx, group)


def gather_transmit_blocks(block, n_tx: int, group=None):
    """All-gather per-rank (n_tx_r, M, T) complex64 trace blocks (transmit
    ranges ``balanced_range(n_tx, r, G)``) into the full (N, M, T) traces."""
    return _gather_dim0(block, n_tx, group)


class _IpcBuffer:
    """One rank's device buffer allocated for CUDA IPC, the peers' buffers
    mapped into this process (rank order), and a torch view of the local one."""

    def __init__(self, nbytes: int, shape, dtype, rank: int, world: int, group=None):
        import ctypes

        import torch

        from . import _lib

        self._own = None
        self._peers = []
        p = ctypes.c_void_p()
        _lib.call("kkb_ipc_alloc", nbytes, ctypes.byref(p))
        self._own = p
        try:
            h = ctypes.create_string_buffer(64)
            _lib.call("kkb_ipc_get_handle", p, h)
            handles = exchange_handles(h.raw, group)
            if len(handles) != world:
                raise RuntimeError("p2p transport needs one process per rank")
            ptrs = []
            for r, hr in enumerate(handles):
                if r == rank:
                    ptrs.append(p.value)
                    continue
                q = ctypes.c_void_p()
                _lib.call("kkb_ipc_open_handle", ctypes.create_string_buffer(hr, 64), ctypes.byref(q))
                self._peers.append(q)
                ptrs.append(q.value)
        except Exception:
            self.close()
            raise
        # own buffer first, then the peers (store order of the scatter kernels)
        order = [ptrs[rank]] + [v for r, v in enumerate(ptrs) if r != rank]
        self.dsts = (ctypes.c_void_p * len(order))(*order)
        typestr = {torch.complex64: "<c8", torch.float32: "<f4"}[dtype]

        class _View:  # CUDA array interface over the raw allocation
            __cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                        "data": (p.value, False), "version": 3, "strides": None}

        self.tensor = torch.as_tensor(_View(), device="cuda")

    def close(self):
        from . import _lib

        lib = _lib.load()
        for q in self._peers:
            lib.kkb_ipc_close_handle(q)
        self._peers = []
        if self._own is not None:
            lib.kkb_ipc_free(self._own)
            self._own = None


class RowBlockKK:
    """Config-5 style single-frame KK beamforming split by image row-block.

    Each rank beamforms the rows ``row_block_range(X, rank, world)`` with the
    K5 kernel and the matching rows of the delay tables.

    Stage 1 (``stage1``):
    * "replicated" (the north star's default): every rank decomposes the
      whole frame.
    * "sharded" (SURVEY §8(e) alternative): rank r decomposes only transmits
      ``balanced_range(N, r, G)`` (of a full (N, L, T) frame, or of its own
      (n_r, L, T) block) and the traces are all-gathered before K5.  With the
      p2p transport the all-gather is fused into the inverse FFT: its epilogue
      stores every trace row into all ranks' IPC-mapped trace buffers
      (``kkb_decomposer_run_scatter``), followed by one barrier.

    Image assembly (``transport``): "p2p" — the K5 epilogue writes the rows
    straight into every rank's full-image buffer (CUDA IPC over NVLink);
    ``gather()`` then only waits (stream sync + barrier) and returns the local
    image.  The IPC image is double-buffered: call i writes half i % 2, so a
    fast rank's call i + 1 never overwrites the image a slow rank is still
    reading after gather() i; a rank can only reach call i + 2 (the same half
    again) after every rank has passed gather() i + 1, i.e. has finished with
    image i.  The returned image is valid until the next gather().  "nccl" — the blocks (and,
    sharded, the traces) are all-gathered with NCCL after the kernels.  Per-row
    and per-pixel arithmetic does not depend on the split, so the image is
    bit-identical to the single-GPU image for any world size, stage-1 mode
    and transport."""

    def __init__(self, array, params, receive, grid, rank: int, world: int, *,
                 interpolation: str = "linear", pulse_delay: float = 0.0,
                 transport: str = "auto", stage1: str = "replicated", group=None):
        import ctypes

        from . import _device as dev
        from . import _lib
        from .beamform import build_kk_luts_device
        from .engine import KKEngine

        if transport not in ("auto", "p2p", "nccl"):
            raise ValueError(f"unknown transport {transport!r}")
        if stage1 not in ("replicated", "sharded"):
            raise ValueError(f"unknown stage-1 mode {stage1!r}")
        t = dev.require_cuda()
        self.t = t
        self.rank, self.world = rank, world
        self.grid = grid
        self.group = group
        self.stage1 = stage1
        self.ix0, self.ix1 = row_block_range(grid.nx, rank, world)
        N, M, T = params.num_transmits, receive.num_angles, params.num_samples
        self.N, self.M, self.T, self.L = N, M, T, array.num_elements
        self.n0, self.n1 = balanced_range(N, rank, world)
        fs = array.sampling_frequency
        shift = (pulse_delay - params.start_time) * fs
        self.engine = None
        self._sdec = None
        self._img = self._tr = None
        self.traces = None
        if stage1 == "replicated":
            self.engine = KKEngine(array, params, receive, grid, frames=1, want_db=False,
                                   interpolation=interpolation, pulse_delay=pulse_delay)
        elif self.n1 > self.n0:
            pos = np.ascontiguousarray(array.positions, dtype=np.float64)
            ang = np.ascontiguousarray(receive.angles, dtype=np.float64)
            h = ctypes.c_void_p()
            _lib.call("kkb_decomposer_create", self.n1 - self.n0, self.L, T, pos.ctypes.data,
                      ang.ctypes.data, M, float(fs), float(params.sound_speed), 1, ctypes.byref(h))
            self._sdec = h
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
                      dev.ptr(luts["lut_rx_z"]), N, M, T, rows, grid.nz, None, float(fs),
                      float(shift), int(interpolation == "linear"), dev.stream_handle(),
                      ctypes.byref(kp))
            self._plan = kp
        self._keep = (luts,)
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
        if stage1 == "sharded" and self._tr is None:
            self.traces = t.empty((N, M, T), dtype=t.complex64, device="cuda")
            self._own_tr = t.empty((max(self.n1 - self.n0, 1), M, T), dtype=t.complex64,
                                   device="cuda")

    def _setup_p2p(self):
        """Full-image (and, sharded, full-trace) buffer per rank; IPC handles
        exchanged, peers mapped."""
        t = self.t
        self._img = _IpcBuffer(2 * self.grid.nx * self.grid.nz * 8, (2, self.grid.nx, self.grid.nz),
                               t.complex64, self.rank, self.world, self.group)
        self._half = 1  # half written by the latest beamform_block (0 after the first call)
        self.image = self._img.tensor[self._half]
        if self.stage1 == "sharded":
            self._tr = _IpcBuffer(self.N * self.M * self.T * 8, (self.N, self.M, self.T),
                                  t.complex64, self.rank, self.world, self.group)
            self.traces = self._tr.tensor

    def _release_p2p(self):
        for b in (self._img, self._tr):
            if b is not None:
                b.close()
        self._img = self._tr = None
        self.traces = None

    def _barrier(self, stream):
        import torch.distributed as dist

        (stream or self.t.cuda.current_stream()).synchronize()
        if self.world > 1:
            dist.barrier(group=self.group)

    def _stage1_sharded(self, rf, stream):
        from . import _device as dev
        from . import _lib

        nr = self.n1 - self.n0
        if rf.dim() == 4:
            rf = rf[0]
        if rf.shape[0] == self.N and nr != self.N:
            rf = rf[self.n0:self.n1]
        if (tuple(rf.shape) != (nr, self.L, self.T) or rf.dtype not in (self.t.float32, self.t.int16)
                or not rf.is_cuda or not rf.is_contiguous()):
            raise ValueError(f"expected contiguous CUDA float32/int16 RF of shape ({self.N} or {nr}, "
                             f"{self.L}, {self.T})")
        s = dev.stream_handle(stream)
        i16 = int(rf.dtype == self.t.int16)
        if self.transport == "p2p":
            if self.world > 1:
                self._barrier(stream)  # no rank still reads the previous traces
            if nr > 0:
                _lib.call("kkb_decomposer_run_scatter", self._sdec, dev.ptr(rf), i16, 1,
                          self._tr.dsts, len(self._tr.dsts), self.n0 * self.M * self.T,
                          self.N * self.M * self.T, s)
            if self.world > 1:
                self._barrier(stream)  # every rank's rows have landed
            return
        if nr > 0:
            name = "kkb_decomposer_run_i16" if i16 else "kkb_decomposer_run"
            _lib.call(name, self._sdec, dev.ptr(rf), 1, dev.ptr(self._own_tr), s)
        if self.world == 1:
            self.traces.copy_(self._own_tr)
        else:
            (stream or self.t.cuda.current_stream()).synchronize()
            self.traces.copy_(gather_transmit_blocks(self._own_tr[:nr], self.N, self.group))

    def beamform_block(self, rf, stream=None):
        """Stage 1, then K5 on this rank's rows; asynchronous (the sharded
        stage 1 synchronises with the peers).  p2p: the rows land in every
        rank's image buffer."""
        from . import _device as dev
        from . import _lib

        if self.stage1 == "sharded":
            self._stage1_sharded(rf, stream)
            traces = self.traces
        else:
            self.engine.decompose(rf[None] if rf.dim() == 3 else rf, n_frames=1, stream=stream)
            traces = self.engine.traces
        if self._plan is None:
            return self.block[:0]
        if self.transport == "p2p":
            # alternate halves: peers may still read the other one (class doc)
            self._half ^= 1
            self.image = self._img.tensor[self._half]
            _lib.call("kkb_kk_plan_run_scatter", self._plan, dev.ptr(traces), 1, 0,
                      self._img.dsts, len(self._img.dsts),
                      (self._half * self.grid.nx + self.ix0) * self.grid.nz,
                      _lib.KKB_OUT_C64, 0, dev.stream_handle(stream))
            return self.image[self.ix0:self.ix1]
        _lib.call("kkb_kk_plan_run", self._plan, dev.ptr(traces), 1, 0,
                  dev.ptr(self.block), _lib.KKB_OUT_C64, 0, None, None,
                  dev.stream_handle(stream))
        return self.block[: self.rows]

    def gather(self, stream=None):
        """The full (X, Z) complex64 image on this rank."""
        if self.transport == "p2p":
            self._barrier(stream)
            return self.image
        if self.world == 1:
            return self.block[: self.rows]
        return gather_row_blocks(self.block[: self.rows], self.grid.nx, self.grid.nz, self.group)

    def close(self):
        from . import _lib

        lib = _lib.load()
        if self._plan is not None:
            lib.kkb_kk_plan_destroy(self._plan)
            self._plan = None
        if self._sdec is not None:
            lib.kkb_decomposer_destroy(self._sdec)
            self._sdec = None
        self._release_p2p()
        if self.engine is not None:
            self.engine.close()
