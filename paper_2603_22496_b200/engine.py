"""Device-resident, batched KK pipeline (the throughput path).

One ``KKEngine`` owns the plans for a fixed geometry — the decomposition
ramps, the four delay tables and the gather window — plus the per-batch
buffers, and runs the whole hot path for F frames with every array in HBM:

    RF (F, N, L, T) float32
      -> K1  real-pair FFT of every element trace            (spectral.py:90)
      -> K2  per-bin contraction over elements x ramps        (compress.py:78-81)
      -> K3  inverse FFT over the non-negative bins           (compress.py:81)
         traces (F, N, M, T) complex64
      -> K5  pixel gather over the N x M coarray pairs        (beamform.py:212-236)
         IQ (F, X, Z) complex64 + fused |IQ|^2 + per-frame max
      -> K6  10 log10(I / max I) display map (new; not in the reference)

This is the reference's own staged data flow (bench.py:113-153 for stage 1,
kk for stage 2) for a batch of frames; the reference times it per frame on
the CPU.  ``run_host`` is the end-to-end form: pinned host RF in, IQ out,
with host<->device copies overlapped with compute on two streams.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _device as dev
from . import _lib
from .beamform import build_kk_luts_device
from .core import AcquisitionParams, ImageGrid, TransducerArray
from .errors import ConfigError
from .sampling import ReceiveAngleSet


class KKEngine:
    def __init__(self, array: TransducerArray, params: AcquisitionParams,
                 receive: ReceiveAngleSet, grid: ImageGrid, frames: int, *,
                 chunk_frames: int | None = None, pipeline: tuple | None = None,
                 interpolation: str = "linear",
                 pulse_delay: float = 0.0, channel_weights=None, floor_db: float = -60.0,
                 want_db: bool = True, groups: int = 1, fuse_tc: bool = False,
                 fused_stage1: bool = False):
        t = dev.require_cuda()
        self.t = t
        self.array, self.params, self.receive, self.grid = array, params, receive, grid
        self.F = int(frames)
        if self.F < 1:
            raise ConfigError("frames must be >= 1")
        self.N = params.num_transmits
        self.L = array.num_elements
        self.M = receive.num_angles
        self.T = params.num_samples
        self.fs = array.sampling_frequency
        self.c = params.sound_speed
        self.shift = (pulse_delay - params.start_time) * self.fs
        self.linear = interpolation == "linear"
        self.floor_db = float(floor_db)
        self.want_db = want_db
        self.chunk = int(chunk_frames or self.F)
        self.groups = int(groups)   # >1: overlap decomposition and gather across frame groups
        # fused_stage1: K1 + K2 as one kernel (opt-in, kkb_decomposer_set_fused;
        # uniform arrays, T = 1536, <= 6 angle classes; ConfigError otherwise)
        self.fused_stage1 = bool(fused_stage1)
        self._side = None
        lib = _lib.load()

        self._dec = self._new_decomposer(self.chunk)
        if pipeline is not None:
            # (frames per pass, streams): overlapped, L2-resident decomposition passes
            _lib.call("kkb_decomposer_set_pipeline", self._dec, int(pipeline[0]), int(pipeline[1]))
        self._stream_decs = []  # one per stream of run_host (scratch is per plan)

        self.luts = build_kk_luts_device(grid, params.transmit_angles, receive.angles, self.c)
        w = None
        if channel_weights is not None:
            w = np.asarray(channel_weights, dtype=np.float64)
            if w.shape != (self.M,):
                raise ConfigError(f"channel_weights must have shape ({self.M},)")
        self._w = dev.to_device(w) if w is not None else None
        kp = ctypes.c_void_p()
        _lib.call("kkb_kk_plan_create", dev.ptr(self.luts["lut_tx_x"]), dev.ptr(self.luts["lut_tx_z"]),
                  dev.ptr(self.luts["lut_rx_x"]), dev.ptr(self.luts["lut_rx_z"]), self.N, self.M,
                  self.T, grid.nx, grid.nz, dev.ptr(self._w), float(self.fs), float(self.shift),
                  int(self.linear), dev.stream_handle(), ctypes.byref(kp))
        self._kk = kp
        self.window = int(lib.kkb_kk_plan_window(kp))

        F, N, M, T, X, Z = self.F, self.N, self.M, self.T, grid.nx, grid.nz
        self.traces = t.empty((F, N, M, T), dtype=t.complex64, device="cuda")
        self.iq = t.empty((F, X, Z), dtype=t.complex64, device="cuda")
        self.inten = t.empty((F, X, Z), dtype=t.float32, device="cuda")
        self.fmax = t.zeros((F,), dtype=t.int32, device="cuda")
        self.db = t.empty((F, X, Z), dtype=t.float32, device="cuda") if want_db else None
        # fused stage 1 -> tensor-core gather (fuse_tc): K3 writes the gather's
        # split fp16 planes (kkb_decomposer_run_planes) instead of complex64
        # traces, so the gather skips its own frame-max and split passes.  Used
        # for whole float32 batches the tensor-core gather takes; self.traces
        # then holds traces only for a batch with a NaN / Inf bin.
        self.fused = False
        self._planes_frames = 0
        min_f = 48 if self.linear else 128   # kk.cuh KKB_KK_TC_MIN_FRAMES(_NEAREST)
        if (fuse_tc and self.T in (1024, 1536, 2048) and pipeline is None and self.chunk == F and F >= min_f
                and int(lib.kkb_kk_plan_tc_ksteps(kp)) > 0):
            nb = int(lib.kkb_tc_planes_bytes(F, N * M, T))
            self._planes = t.empty((nb,), dtype=t.uint8, device="cuda")
            self._fbound = t.zeros((F,), dtype=t.int32, device="cuda")
            self._nonfinite = t.zeros((1,), dtype=t.int32, device="cuda")
            self.fused = True
        self._closed = False

    def _new_decomposer(self, chunk: int):
        pos = np.ascontiguousarray(self.array.positions, dtype=np.float64)
        ang = np.ascontiguousarray(self.receive.angles, dtype=np.float64)
        h = ctypes.c_void_p()
        _lib.call("kkb_decomposer_create", self.N, self.L, self.T, pos.ctypes.data, ang.ctypes.data,
                  self.M, float(self.fs), float(self.c), int(chunk), ctypes.byref(h))
        if self.fused_stage1:
            if _lib.load().kkb_decomposer_set_fused(h, 1) != 0:
                _lib.load().kkb_decomposer_destroy(h)
                raise ConfigError("fused_stage1 needs a uniform symmetric array, T = 1536, L a multiple of 8 "
                                  "up to 256 and at most 6 receive-angle classes")
        return h

    # ------------------------------------------------------------------ info
    @property
    def pixel_pairs_per_frame(self) -> int:
        return self.grid.nx * self.grid.nz * self.N * self.M

    def workspace_bytes(self) -> int:
        lib = _lib.load()
        own = sum(x.numel() * x.element_size() for x in
                  (self.traces, self.iq, self.inten, self.fmax) + ((self.db,) if self.db is not None else ()))
        return int(lib.kkb_decomposer_workspace_bytes(self._dec)) + own

    # ------------------------------------------------------------------ device path
    def _run_decomposer(self, handle, rf, n_frames, traces, stream_handle):
        # float32 RF, or int16-quantised RF converted exactly inside the FFT load
        name = "kkb_decomposer_run_i16" if rf.dtype == self.t.int16 else "kkb_decomposer_run"
        _lib.call(name, handle, dev.ptr(rf), n_frames, dev.ptr(traces), stream_handle)

    def _check_rf(self, rf, n_frames: int):
        t = self.t
        if not (0 <= n_frames <= self.F):
            raise ConfigError(f"n_frames must be in [0, {self.F}]")
        if (rf.dtype not in (t.float32, t.int16) or rf.dim() != 4 or rf.shape[0] < n_frames
                or tuple(rf.shape[1:]) != (self.N, self.L, self.T)):
            raise ConfigError(f"expected float32 or int16 RF of shape (>= {n_frames}, {self.N}, "
                              f"{self.L}, {self.T}), got {rf.dtype} {tuple(rf.shape)}")
        if not rf.is_cuda or not rf.is_contiguous():
            raise ConfigError("RF must be a contiguous CUDA tensor")

    def decompose(self, rf, n_frames: int | None = None, stream=None):
        F = self.F if n_frames is None else n_frames
        self._check_rf(rf, F)
        if self.fused and F == self.F and rf.dtype == self.t.float32:
            _lib.call("kkb_decomposer_run_planes", self._dec, dev.ptr(rf), F, dev.ptr(self._planes),
                      dev.ptr(self._fbound), dev.ptr(self._nonfinite), dev.ptr(self.traces),
                      dev.stream_handle(stream))
            self._planes_frames = F
            return self.traces[:F]
        self._planes_frames = 0
        self._run_decomposer(self._dec, rf, F, self.traces, dev.stream_handle(stream))
        return self.traces[:F]

    def _run_planes(self, F, iq, inten, fmax, accumulate, s):
        P = self.grid.nx * self.grid.nz
        _lib.call("kkb_kk_plan_run_planes", self._kk, dev.ptr(self._planes), dev.ptr(self._fbound),
                  dev.ptr(self._nonfinite), dev.ptr(self.traces), F, dev.ptr(iq), _lib.KKB_OUT_C64, P,
                  dev.ptr(inten), dev.ptr(fmax), _lib.KKB_RUN_ACCUMULATE_INTENSITY if accumulate else 0, s)

    def beamform(self, traces=None, n_frames: int | None = None, stream=None, out_offset: int = 0,
                 inten=None, fmax=None, accumulate: bool = False, want_db: bool | None = None):
        """K5 (+ fused detection) and K6 on decomposed traces.  `inten` / `fmax`
        redirect the detection to caller buffers; `accumulate` adds |IQ|^2 to
        `inten` (incoherent compounding, see MultiSetEngine)."""
        F = self.F if n_frames is None else n_frames
        traces = self.traces if traces is None else traces
        P = self.grid.nx * self.grid.nz
        s = dev.stream_handle(stream)
        iq = self.iq[out_offset:out_offset + F]
        inten = (self.inten if inten is None else inten)[out_offset:out_offset + F]
        fmax = None if fmax is False else (self.fmax if fmax is None else fmax)[out_offset:out_offset + F]
        if traces is self.traces and out_offset == 0 and F == self._planes_frames:
            self._run_planes(F, iq, inten, fmax, accumulate, s)
        else:
            _lib.call("kkb_kk_plan_run_ex", self._kk, dev.ptr(traces), F, self.N * self.M * self.T,
                      dev.ptr(iq), _lib.KKB_OUT_C64, P, dev.ptr(inten), dev.ptr(fmax),
                      _lib.KKB_RUN_ACCUMULATE_INTENSITY if accumulate else 0, s)
        if self.want_db if want_db is None else want_db:
            db = self.db[out_offset:out_offset + F]
            _lib.call("kkb_log_compress", dev.ptr(inten), dev.ptr(fmax), F, P, self.floor_db,
                      dev.ptr(db), s)
        return iq

    def gather(self, n_frames: int | None = None, stream=None):
        """K5 alone on self.traces (bench instrumentation)."""
        F = self.F if n_frames is None else n_frames
        P = self.grid.nx * self.grid.nz
        fmax = self.fmax[:F]
        if F == self._planes_frames:
            self._run_planes(F, self.iq, self.inten, fmax, False, dev.stream_handle(stream))
            return self.iq[:F]
        _lib.call("kkb_kk_plan_run", self._kk, dev.ptr(self.traces), F, self.N * self.M * self.T,
                  dev.ptr(self.iq), _lib.KKB_OUT_C64, P, dev.ptr(self.inten), dev.ptr(fmax),
                  dev.stream_handle(stream))
        return self.iq[:F]

    def detect(self, n_frames: int | None = None, stream=None):
        """K6 dB map alone (bench instrumentation)."""
        F = self.F if n_frames is None else n_frames
        P = self.grid.nx * self.grid.nz
        _lib.call("kkb_log_compress", dev.ptr(self.inten), dev.ptr(self.fmax), F, P, self.floor_db,
                  dev.ptr(self.db), dev.stream_handle(stream))
        return self.db[:F]

    def run(self, rf, stream=None, groups=None, gather_events=None):
        """Whole hot path for a (F, N, L, T) float32 CUDA tensor; asynchronous.
        Returns the complex64 IQ images (F, X, Z) (``self.inten`` / ``self.db``
        hold the detected and log-compressed images)."""
        if tuple(rf.shape[:1]) != (self.F,):
            raise ConfigError(f"expected float32 or int16 RF of shape {(self.F, self.N, self.L, self.T)}")
        self._check_rf(rf, self.F)
        groups = self.groups if groups is None else int(groups)
        if groups <= 1 or self.F < 2:
            self.decompose(rf, stream=stream)
            return self.beamform(stream=stream)
        return self._run_overlapped(rf, groups, stream, gather_events)

    def _run_overlapped(self, rf, groups, stream, gather_events=None):
        """Frame groups: decomposition of group g+1 (FFT/FMA/latency-bound) runs
        on the caller's stream while the gather of group g (shared-memory
        bound) runs on a side stream, so the two bottlenecks share the SMs."""
        t = self.t
        from .shard import balanced_range

        main = stream if stream is not None else t.cuda.current_stream()
        if self._side is None:
            self._side = t.cuda.Stream()
        side = self._side
        side.wait_stream(main)  # outputs may still be read by earlier work on main
        self._planes_frames = 0
        NMT = self.N * self.M * self.T
        for g in range(groups):
            f0, f1 = balanced_range(self.F, g, groups)
            n = f1 - f0
            if n == 0:
                continue
            tr = self.traces[f0:f1]
            self._run_decomposer(self._dec, rf[f0:f1], n, tr, main.cuda_stream)
            ev = t.cuda.Event()
            ev.record(main)
            side.wait_event(ev)
            if gather_events is not None:
                gather_events[g][0].record(side)
            self.beamform(traces=tr, n_frames=n, stream=side, out_offset=f0)
            if gather_events is not None:
                gather_events[g][1].record(side)
        main.wait_stream(side)
        return self.iq

    def capture(self, rf, groups: int = 1):
        """CUDA graph of the whole hot path (``run``) on the static RF buffer
        ``rf``: returns a ``KKGraph`` whose ``replay()`` reruns every launch
        with no host work, for low-latency frame-by-frame imaging (refill
        ``rf`` in place between replays; outputs land in ``iq`` / ``inten`` /
        ``db`` as for ``run``)."""
        t = self.t
        self._check_rf(rf, self.F)
        s = t.cuda.Stream()
        s.wait_stream(t.cuda.current_stream())
        with t.cuda.stream(s):  # warm-up: attributes, allocator pools
            self.run(rf, stream=s, groups=groups)
        s.synchronize()
        g = t.cuda.CUDAGraph()
        with t.cuda.graph(g, stream=s):
            self.run(rf, stream=s, groups=groups)
        t.cuda.current_stream().wait_stream(s)
        return KKGraph(g, self, rf)

    # ------------------------------------------------------------------ end-to-end path
    def run_host(self, rf_host, iq_host, chunk_frames: int = 16, streams=None, staging=None):
        """Pinned host RF (F, N, L, T) float32 -> pinned host IQ (F, X, Z) complex64.

        Chunks of frames are copied in, processed and copied out on alternating
        streams so that H2D, kernels and D2H overlap."""
        t = self.t
        F = self.F
        if rf_host.is_cuda or tuple(rf_host.shape) != (F, self.N, self.L, self.T) or \
                rf_host.dtype not in (t.float32, t.int16):
            raise ConfigError(f"expected host float32 or int16 RF of shape {(F, self.N, self.L, self.T)}")
        if iq_host.is_cuda or tuple(iq_host.shape) != (F, self.grid.nx, self.grid.nz) or \
                iq_host.dtype != t.complex64:
            raise ConfigError(f"expected a host complex64 IQ buffer of shape {(F, self.grid.nx, self.grid.nz)}")
        C = max(1, min(chunk_frames, self.chunk, F))
        self._planes_frames = 0
        if streams is None:
            streams = [t.cuda.Stream(), t.cuda.Stream()]
        cur = t.cuda.current_stream()
        for s in streams:  # earlier work on the caller's stream may still use the buffers
            s.wait_stream(cur)
        while len(self._stream_decs) < len(streams):
            self._stream_decs.append(self._new_decomposer(C))
        if staging is None:
            staging = [t.empty((C, self.N, self.L, self.T), dtype=rf_host.dtype, device="cuda")
                       for _ in streams]
        for i, f0 in enumerate(range(0, F, C)):
            n = min(C, F - f0)
            s = streams[i % len(streams)]
            buf = staging[i % len(staging)]
            with t.cuda.stream(s):
                buf[:n].copy_(rf_host[f0:f0 + n], non_blocking=True)
                tr = self.traces[f0:f0 + n]
                self._run_decomposer(self._stream_decs[i % len(streams)], buf[:n], n, tr,
                                     s.cuda_stream)
                self.beamform(traces=tr, n_frames=n, stream=s, out_offset=f0)
                iq_host[f0:f0 + n].copy_(self.iq[f0:f0 + n], non_blocking=True)
        for s in streams:
            s.synchronize()
        return iq_host

    def close(self):
        if not self._closed:
            lib = _lib.load()
            lib.kkb_decomposer_destroy(self._dec)
            for h in self._stream_decs:
                lib.kkb_decomposer_destroy(h)
            lib.kkb_kk_plan_destroy(self._kk)
            self._closed = True

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class KKGraph:
    """A captured ``KKEngine.run`` (see ``KKEngine.capture``)."""

    def __init__(self, graph, engine, rf):
        self.graph, self.engine, self.rf = graph, engine, rf

    def replay(self):
        """Rerun the captured hot path on the current contents of ``rf``;
        asynchronous on the current stream.  Returns the IQ images."""
        self.graph.replay()
        return self.engine.iq


class MultiSetEngine:
    """Several receive-angle sets over one RF batch, compounded on the device
    (the reference's hybrid / multi-j acquisitions: cli.py:93-107, 250-266;
    compound_coherent / compound_incoherent, beamform.py:396-411).

    The RF is decomposed ONCE over the concatenated angle list (the sets laid
    out one after another along the receive axis), so the element FFTs are
    shared by all sets.
    mode "incoherent": ONE gather launch over the shared traces
      (``kkb_kk_plan_run_sets``): each CTA stages the tables once and sums the
      sets one after another, storing B_j in ``iq[j]`` and sum_j |B_j|^2 (and
      its per-frame max) in ``inten``.
    mode "coherent": |sum_j B_j|^2 is the kk image over the whole list (kk sums
      over every receive angle): one gather over all rows.
    """

    def __init__(self, array: TransducerArray, params: AcquisitionParams, receive_sets,
                 grid: ImageGrid, frames: int, mode: str = "incoherent", want_db: bool = True,
                 floor_db: float = -60.0, **kw):
        from .sampling import explicit_angles

        sets = [rs[1] if isinstance(rs, tuple) else rs for rs in receive_sets]
        if not sets:
            raise ConfigError("need at least one receive set")
        if mode not in ("incoherent", "coherent"):
            raise ConfigError(f"unknown compounding mode {mode!r}")
        if mode == "incoherent" and len(sets) > _lib.KKB_MAX_SETS:
            raise ConfigError(f"at most {_lib.KKB_MAX_SETS} receive sets per launch")
        self.mode, self.want_db, self.floor_db = mode, want_db, float(floor_db)
        self.sets = sets
        union = explicit_angles(np.concatenate([s.angles for s in sets]), sets[0].delta_theta_i)
        # the union engine: shared decomposition and the plan over all angles
        self.engine = KKEngine(array, params, union, grid, frames,
                               want_db=want_db and mode == "coherent", floor_db=floor_db, **kw)
        self.engines = [self.engine]
        e = self.engine
        if mode == "coherent":
            self.inten, self.fmax, self.db = e.inten, e.fmax, e.db
            return
        t = e.t
        self.inten, self.fmax = e.inten, e.fmax
        self.db = t.empty_like(e.inten) if want_db else None
        bounds = np.concatenate([[0], np.cumsum([s.num_angles for s in sets])]).astype(np.int32)
        self._m_off = bounds[:-1].astype(int)
        self._bounds = (ctypes.c_int * len(bounds))(*[int(b) for b in bounds])
        # per-set IQ, (S, F, X, Z): iq[j] is set j's images
        self.iq = t.empty((len(sets), e.F, grid.nx, grid.nz), dtype=t.complex64, device="cuda")

    @property
    def pixel_pairs_per_frame(self) -> int:
        return self.engine.pixel_pairs_per_frame

    def run(self, rf, stream=None):
        """Compounded intensity (F, X, Z) float32 for a (F, N, L, T) RF batch;
        asynchronous."""
        e = self.engine
        if tuple(rf.shape[:1]) != (e.F,):
            raise ConfigError(f"expected RF of shape {(e.F, e.N, e.L, e.T)}")
        if self.mode == "coherent":
            e.run(rf, stream=stream, groups=1)
            return self.inten
        e.decompose(rf, stream=stream)
        s = dev.stream_handle(stream)
        P = e.grid.nx * e.grid.nz
        _lib.call("kkb_kk_plan_run_sets", e._kk, dev.ptr(e.traces), e.F, e.N * e.M * e.T,
                  len(self.sets), self._bounds, dev.ptr(self.iq), _lib.KKB_OUT_C64, P, e.F * P,
                  dev.ptr(self.inten), dev.ptr(self.fmax), 0, s)
        if self.want_db:
            _lib.call("kkb_log_compress", dev.ptr(self.inten), dev.ptr(self.fmax), e.F, P,
                      self.floor_db, dev.ptr(self.db), s)
        return self.inten

    def close(self):
        self.engine.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
