"""Benchmark of the KK hot path (BASELINE.json metric: KK frames/s and
pixel-pair samples/s, with the roofline fraction).

Default workload: config 4 (functional-ultrasound ensemble, BASELINE.json
configs[3]) — the configuration the metric is quoted on at 1/2/4/8 GPUs.
A step = the whole hot path over one 400-frame ensemble per rank:
real FFT -> per-bin element contraction -> inverse FFT -> kk pixel gather
(+ fused |IQ|^2, per-frame max) -> dB map, every array in HBM.  The RF
batch is 3.46 GB per rank (> 126 MB L2), so no L2 flush is needed between
steps.  Multi-GPU: one process per GPU (torchrun), frames sharded by rank
with no data-path collective (weak scaling: 400 frames per rank); the
step time is the max over ranks of CUDA-event time.

--impl reference: the CPU restatement of the reference path (oracle/:
numpy/scipy stage 1 in the reference benchmark's complex64 form, C/OpenMP
kk loop) on the host cores, bounded samples of the same workload.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "KK frames/s (pixel-pair samples/s alongside), whole hot path"
UNIT = "frames/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _gather_traffic(frames: int):
    """dram read+write bytes of one k_kk_gather launch from the newest committed
    ncu --set full capture (profiles/r*_gather_traffic.json), scaled to `frames`."""
    import glob

    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_gather_traffic.json")))
    if not paths:
        return None
    with open(paths[-1]) as f:
        d = json.load(f)
    return d["dram_bytes_per_launch"] * frames / d["frames_per_launch"]


def _workload(cfg: int, frames: int):
    from paper_2603_22496_b200 import configs

    if cfg == 4:
        return configs.config4(frames=frames)
    w = configs.CONFIGS[cfg]()
    return w


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- CPU arms
def cpu_model() -> str:
    """Host CPU model name (/proc/cpuinfo), for the CPU-baseline record."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_pipeline_rate(w, seconds: float = 12.0, min_frames: int = 2, threads: int = 0):
    """Oracle port of the reference path on the host: frames/s over a bounded
    sample (>= min_frames, ~`seconds` of work).  The kk loop uses every host
    core (threads=0), explicitly: torchrun exports OMP_NUM_THREADS=1."""
    threads = threads or (os.cpu_count() or 1)
    from oracle import kkbeam_oracle as O
    from paper_2603_22496_b200 import configs

    O.build()
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    fs, c = arr.sampling_frequency, p.sound_speed
    luts = O.kk_luts(g.x, g.z, p.transmit_angles, rx.angles, c)
    rf = configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples, seed=0)
    ones = np.ones(rx.num_angles)
    shift = (0.0 - p.start_time) * fs

    def frame():
        tr = O.decompose_c64_staged(rf, fs, arr.positions, rx.angles, c)
        img = O.kk_kernel(tr, *luts, ones, fs, shift, threads=threads)
        return O.log_compress_db(O.intensity(img))

    frame()  # warm-up (OpenMP pool, scipy planning)
    n, t0 = 0, time.perf_counter()
    while n < min_frames or time.perf_counter() - t0 < seconds:
        frame()
        n += 1
    dt = time.perf_counter() - t0
    return n / dt, n, dt


def _config(w, frames, world):
    """The `config` object of both arms (identical keys and values)."""
    g, p = w.grid, w.params
    return {"workload": w.name, "frames_per_rank": frames, "N_tx": p.num_transmits,
            "M_rx": w.receive.num_angles, "L_el": w.array.num_elements, "T": p.num_samples,
            "grid": [g.nx, g.nz], "pixel_pairs_per_frame": g.nx * g.nz * w.pairs,
            "l2": "inputs larger than L2 (3.46 GB RF per rank), no flush",
            "parallelism": f"frame-sharded x{world}"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    w = _workload(args.config, args.frames)
    cores = os.cpu_count() or 1
    # each step: a bounded sample of 2 frames of the same workload
    per_step = []
    for _ in range(args.warmup):
        cpu_pipeline_rate(w, seconds=0.0, min_frames=1)
    for _ in range(args.steps):
        r, n, dt = cpu_pipeline_rate(w, seconds=0.0, min_frames=2)
        per_step.append(dt)
    t = sum(per_step)
    value = 2 * args.steps / t
    pp = w.grid.nx * w.grid.nz * w.pairs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32",
        "dtype_detail": "complex64 stage 1 and traces, float64 delay-index math, complex128 image accumulation",
        "data": "synthetic (seeded noise RF, reference bench.noise_volume)",
        "config": _config(w, args.frames, int(os.environ.get("WORLD_SIZE", "1"))),
        "pixel_pair_samples_per_s": value * pp,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "cpu": cpu_model(),
                         "sample": f"2 frames per step of the {args.frames}-frame workload: numpy/scipy "
                                   "complex64 stage 1 (bench.py:113-138 form) + C/OpenMP kk loop "
                                   "(all cores)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ----------------------------------------------------------------- GPU arm
def _init_dist(torch, dist, world, local):
    """One process per GPU over NCCL.  KKB_DIST_BACKEND=gloo (a functional
    check of the multi-rank code path on a one-GPU box: ranks share cuda:0,
    their timings are not measurements) also wraps the device index."""
    backend = os.environ.get("KKB_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return local


def _onchip_peaks():
    """Measured shared-memory (LDS.128) and FP32 FMA peaks of this B200
    (scripts/ubench/peaks.cu, profiles/r02_onchip_peaks.json); the driver's
    MEASURED_PEAKS.json has only HBM and bf16 tensor figures."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_onchip_peaks.json")) as f:
            d = json.load(f)
        return float(d["smem_lds128_GBps"]), float(d["fp32_fma_TFLOPs"]), "measured"
    except (OSError, KeyError, ValueError):
        return None, None, "missing"


def _l2_roofline(achieved_taps):
    """SURVEY 8(d)'s gather roofline: 16 B of taps per pixel-pair over the
    measured L2 read bandwidth (profiles/r01g_l2_bw.json, scripts/ubench/
    l2_bw.cu; the driver's MEASURED_PEAKS.json has no L2 figure)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01g_l2_bw.json")) as f:
            peak = float(json.load(f)["peak_L2_read_GBps"])
    except (OSError, KeyError, ValueError):
        return None
    return {"kernel": "k_kk_gather", "bound": "l2", "achieved": achieved_taps, "peak": peak,
            "unit": "GB/s", "frac": achieved_taps / peak,
            "peak_kind": "measured (scripts/ubench/l2_bw.cu, 48 MB L2-resident set)",
            "note": "frac > 1: the taps come from shared memory, each staged trace sample "
                    "serving every pixel of the tile that reads it"}


def _tensor_peak():
    """Dense bf16/f16 tensor peak (MEASURED_PEAKS.json, driver-written): the
    sustained figure, the gather being timed inside a multi-kernel step."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p.get("bf16_tflops_sustained") or p["bf16_tflops"]), "measured (sustained bf16 matmul)"
    except Exception:
        return 2250.0, "fallback (nominal dense bf16)"


def run_gpu(args):
    import torch
    import torch.distributed as dist

    import paper_2603_22496_b200 as kb
    from paper_2603_22496_b200 import _lib, configs

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = _init_dist(torch, dist, world, local)
    host_cpus = None
    if world > 1:  # pinned host buffers on the GPU's own NUMA node (first touch)
        from paper_2603_22496_b200._numa import bind_to_device

        host_cpus = bind_to_device(local)

    w = _workload(args.config, args.frames)
    F = w.frames if args.config == 4 else args.frames
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    N, L, T, M = p.num_transmits, arr.num_elements, p.num_samples, rx.num_angles
    P = g.nx * g.nz
    pp_frame = P * N * M

    # per-rank input: seeded noise frames (tiled from a few distinct frames to keep
    # host generation short); each rank gets different seeds
    distinct = min(F, 8)
    base = np.stack([configs.noise_rf(N, L, T, seed=1000 * rank + s) for s in range(distinct)])
    rf_dev = torch.empty((F, N, L, T), dtype=torch.float32, device="cuda")
    src = torch.from_numpy(base).cuda()
    for f0 in range(0, F, distinct):
        n = min(distinct, F - f0)
        rf_dev[f0:f0 + n].copy_(src[:n])
    del src

    pipeline = (args.pipe_chunk, args.pipe_slots) if args.pipe_slots > 1 else None
    eng = kb.KKEngine(arr, p, rx, g, frames=F, chunk_frames=args.chunk, pipeline=pipeline,
                      fuse_tc=not args.no_fuse)
    stream = torch.cuda.current_stream()

    G = max(1, args.groups)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def step(marks):
        """One pass of the hot path over the 400-frame batch.  G > 1: frame groups,
        decomposition of group g+1 overlapped with the gather of group g
        (KKEngine._run_overlapped); marks = per-group (start, end) events of
        the gather launches on their stream."""
        if G > 1:
            eng.run(rf_dev, groups=G, gather_events=marks)
        else:
            eng.decompose(rf_dev)
            marks[0][0].record(stream)
            eng.gather()
            marks[0][1].record(stream)
            eng.detect()

    for _ in range(args.warmup):
        step([(ev(), ev()) for _ in range(G)])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    marks = [[(ev(), ev()) for _ in range(G)] for _ in range(args.steps)]
    launches0 = _lib.launch_count()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_start, t_end = ev(), ev()
    t_start.record(stream)
    for i in range(args.steps):
        step(marks[i])
    t_end.record(stream)
    torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    total_ms = t_start.elapsed_time(t_end)
    if world > 1:
        tt = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())
    ms_step = total_ms / args.steps
    value = world * F / (total_ms / 1e3 / args.steps)
    # K5 launch durations inside the timed region (G launches of F/G frames per step;
    # with G > 1 they include the K6 dB map and share the SMs with the decomposition)
    kk_launch_ms = statistics.median(a.elapsed_time(b) for m in marks for a, b in m)
    frames_per_launch = F / G

    # stage split from sequential instrumented passes after the timed region
    seq = []
    for _ in range(3):
        e = [ev() for _ in range(4)]
        e[0].record(stream)
        eng.decompose(rf_dev)
        e[1].record(stream)
        eng.gather()
        e[2].record(stream)
        eng.detect()
        e[3].record(stream)
        seq.append(e)
    torch.cuda.synchronize()
    dec_ms = statistics.median(e[0].elapsed_time(e[1]) for e in seq)
    kk_ms = statistics.median(e[1].elapsed_time(e[2]) for e in seq)
    det_ms = statistics.median(e[2].elapsed_time(e[3]) for e in seq)

    # device-resident int16 ingest (BASELINE config 2's sample format; the FFT
    # load converts exactly): same step on int16-quantised copies of the frames
    scale = float(np.abs(base).max()) / 32767.0
    rf_q = torch.empty((F, N, L, T), dtype=torch.int16, device="cuda")
    qb = torch.from_numpy(np.clip(np.round(base / scale), -32767, 32767).astype(np.int16)).cuda()
    for f0 in range(0, F, distinct):
        n = min(distinct, F - f0)
        rf_q[f0:f0 + n].copy_(qb[:n])
    del qb

    def step_q():
        eng.decompose(rf_q)
        eng.gather()
        eng.detect()

    for _ in range(2):
        step_q()
    torch.cuda.synchronize()
    q0, q1 = ev(), ev()
    q0.record(stream)
    for _ in range(args.steps):
        step_q()
    q1.record(stream)
    torch.cuda.synchronize()
    q_ms = q0.elapsed_time(q1) / args.steps
    if world > 1:
        tt = torch.tensor([q_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        q_ms = float(tt.item())
    del rf_q

    # ---- roofline of the dominant kernel (K5 gather), per launch in the timed region ----
    hbm_peak, peak_kind = _peaks()
    sm_count = torch.cuda.get_device_properties(local).multi_processor_count
    fl = frames_per_launch
    gather_bytes_alg = 16.0 * pp_frame * fl                    # 16 B x pp
    compulsory = fl * (N * M * T * 8 + P * (8 + 4)) + 8 * (g.nx + g.nz) * (N + M)
    achieved_hbm = compulsory / (kk_launch_ms / 1e3) / 1e9
    sm_mhz = clk.get("sm_mhz") or 1965.0
    smem_meas, fp32_meas, onchip_kind = _onchip_peaks()
    smem_derived = sm_count * 128 * sm_mhz * 1e6 / 1e9          # GB/s, 128 B/clk/SM crossbar
    smem_peak = smem_meas or smem_derived
    achieved_taps = gather_bytes_alg / (kk_launch_ms / 1e3) / 1e9
    # which K5 ran (the sequential passes above): the tensor-core gather's work
    # is its split-fp16 MMAs, 3 per K = 16 step of 128 pixels x 16 columns
    # (re | im of 8 frames) x 16 samples, ksteps per group of 8 frames
    k5_inst = _lib.KKB_KK_INST_NAMES.get(_lib.last_instance() & 15, "?")
    tc_ksteps = int(_lib.load().kkb_kk_plan_tc_ksteps(eng._kk)) if k5_inst == "tc" else -1
    tc_flops = tc_ksteps * math.ceil(fl / 8) * 3 * 2.0 * 128 * 16 * 16 if tc_ksteps > 0 else None
    tensor_peak, tensor_kind = _tensor_peak()
    # stage 1 (K1-K3) is HBM-bound: bytes its three kernels must move per batch
    # (RF in, spectra written then read, contracted bins written then read,
    # traces out) and the two-array compulsory minimum (RF in + traces out)
    ldk = (T // 2 + 1 + 1) & ~1
    s1_bytes = F * (4.0 * N * L * T + 2 * 8.0 * N * L * ldk + 2 * 8.0 * N * M * ldk + 8.0 * N * M * T)
    s1_min = F * (4.0 * N * L * T + 8.0 * N * M * T)
    s1_achieved = s1_bytes / (dec_ms / 1e3) / 1e9
    # SURVEY 8(d) flop units: contraction 8*N*L*M*K, FFTs 2.5*N*L*T*log2 T + 5*N*M*T*log2 T
    K = T // 2 + 1
    s1_flops = F * (8.0 * N * L * M * K + 2.5 * N * L * T * math.log2(T) + 5.0 * N * M * T * math.log2(T))
    fp32_peak = fp32_meas or sm_count * 128 * 2 * sm_mhz * 1e6 / 1e12  # TFLOP/s
    frame_bytes = 4.0 * N * L * T + 2 * 8.0 * N * M * T + 8.0 * P + 8.0 * (g.nx + g.nz) * (N + M)

    # ---- end to end through the public API: pinned host RF in, host IQ out ----
    e2e = e2e_i16 = None
    if not args.no_e2e:
        host_rf = torch.empty((F, N, L, T), dtype=torch.float32).pin_memory()
        for f0 in range(0, F, distinct):
            n = min(distinct, F - f0)
            host_rf[f0:f0 + n].copy_(torch.from_numpy(base[:n]))
        host_iq = torch.empty((F, g.nx, g.nz), dtype=torch.complex64).pin_memory()
        streams = [torch.cuda.Stream(), torch.cuda.Stream()]
        e2e_steps = max(1, min(args.steps, 5))

        def e2e_rate(host_in):
            for _ in range(max(1, min(args.warmup, 2))):
                eng.run_host(host_in, host_iq, chunk_frames=args.e2e_chunk, streams=streams)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                eng.run_host(host_in, host_iq, chunk_frames=args.e2e_chunk, streams=streams)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if world > 1:
                tt = torch.tensor([dt], device="cuda")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                dt = float(tt.item())
            return world * F * e2e_steps / dt

        e2e = {"value": e2e_rate(host_rf), "unit": UNIT,
               "h2d_bytes_per_step": int(host_rf.numel() * 4),
               "d2h_bytes_per_step": int(host_iq.numel() * 8),
               "path": "KKEngine.run_host: pinned H2D float32 RF, decompose+kk on 2 streams, D2H IQ"}
        # the leg's bound: host->device bytes per second it sustains (PCIe)
        e2e["h2d_GBps_per_gpu"] = e2e["h2d_bytes_per_step"] / (world * F / e2e["value"]) / 1e9
        # same path fed int16-quantised RF (BASELINE config 2 sample format; exact)
        del host_rf
        scale = float(np.abs(base).max()) / 32767.0
        q = np.clip(np.round(base / scale), -32767, 32767).astype(np.int16)
        host_q = torch.empty((F, N, L, T), dtype=torch.int16).pin_memory()
        for f0 in range(0, F, distinct):
            n = min(distinct, F - f0)
            host_q[f0:f0 + n].copy_(torch.from_numpy(q[:n]))
        e2e_i16 = {"value": e2e_rate(host_q), "unit": UNIT,
                   "h2d_bytes_per_step": int(host_q.numel() * 2),
                   "d2h_bytes_per_step": int(host_iq.numel() * 8),
                   "path": "KKEngine.run_host with int16 RF (converted exactly on device)"}
        del host_q

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        r, n, dt = cpu_pipeline_rate(w, seconds=args.cpu_seconds)
        cpu = {"value": r, "unit": UNIT, "cores": os.cpu_count(), "kind": "port", "cpu": cpu_model(),
               "sample": f"{n} frames of {w.name} in {dt:.1f} s: numpy/scipy complex64 stage 1 "
                         "(reference bench.py:113-138 form) + C/OpenMP kk loop on all cores"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f32",
            "dtype_detail": "complex64 spectra/traces/IQ, float32 taps and sums, float64 delay-index math",
            "data": "synthetic (seeded noise RF, shapes of BASELINE config 4)",
            "config": _config(w, F, world),
            "pixel_pair_samples_per_s": value * pp_frame,
            "stage_ms_sequential": {"decompose(K1-K3)": dec_ms, "kk_gather(K5)": kk_ms,
                                    "db_map(K6)": det_ms},
            "overlap_groups": G,
            "stage1_to_k5": ("fused: K3 writes the tensor-core gather's split fp16 planes "
                             "(kkb_decomposer_run_planes -> kkb_kk_plan_run_planes)") if eng.fused else
                            "complex64 traces (K5 splits them itself when it runs on the tensor cores)",
            "value_int16_ingest": {"value": world * F / (q_ms / 1e3), "unit": UNIT, "ms_per_step": q_ms,
                                   "note": "same device-resident step on int16-quantised RF "
                                           "(converted exactly in the FFT load)"},
            # the dominant kernel's roofline.  The tensor-core gather (the bench
            # dispatch): its split-fp16 MMA work against the measured tensor
            # peak.  The FMA gather: its taps against the measured LDS.128 peak
            # (both kept: "taps_roofline" is the algorithmic on-chip figure)
            "roofline": ({"kernel": "k_kk_gather_tc", "bound": "tensor",
                          "achieved": tc_flops / (kk_launch_ms / 1e3) / 1e12, "peak": tensor_peak,
                          "unit": "TFLOP/s", "frac": tc_flops / (kk_launch_ms / 1e3) / 1e12 / tensor_peak,
                          "traffic": _gather_traffic(fl), "launch_ms": kk_launch_ms,
                          "frames_per_launch": fl, "flops_per_launch": tc_flops,
                          "k_steps_per_frame_group": tc_ksteps,
                          "flops": "issued split-fp16 MMA work of the gather's GEMM form: 3 products "
                                   "(hi*hi, hi*lo, lo*hi) x 2*128*16*16 per K = 16 step, one or two "
                                   "steps per (tile, pair) from the plan's exact windows "
                                   "(kkb_kk_plan_tc_ksteps), per group of 8 frames; the direct form's "
                                   "algorithmic work is the taps below",
                          "peak_kind": tensor_kind,
                          "launch_note": "launch_ms spans the K5 call: the per-frame max and plane "
                                         "split passes plus the gather (profiles/r02b_launches_"
                                         "bench_default.csv has each kernel's share)"}
                         if tc_flops else {"kernel": "k_kk_gather_tc" if tc_flops else "k_kk_gather", "bound": "smem",
                         "achieved": achieved_taps, "peak": smem_peak, "unit": "GB/s",
                         "frac": achieved_taps / smem_peak, "traffic": _gather_traffic(fl),
                         "launch_ms": kk_launch_ms, "frames_per_launch": fl,
                         "algorithmic_bytes_per_launch": gather_bytes_alg,
                         "algorithmic_bytes": "16 B of taps (two complex64 samples) per pixel-pair "
                                              "(SURVEY 8d) x pixel-pairs per launch",
                         "peak_kind": (f"{onchip_kind} (scripts/ubench/peaks.cu: conflict-free LDS.128 "
                                       "on every SM, profiles/r02_onchip_peaks.json)") if smem_meas else
                                      "derived (148 SMs x 128 B/clk x sampled SM clock)",
                         "peak_derived_at_sampled_clock": smem_derived,
                         "pixel_pairs_per_s": pp_frame * fl / (kk_launch_ms / 1e3),
                         "pixel_pairs_per_s_isolated": pp_frame * F / (kk_ms / 1e3),
                         "traffic_note": "ncu dram read+write per launch of the gather kernel (newest "
                                         "profiles/r*_gather_traffic.json); below the compulsory HBM "
                                         "bytes because the gather reads only the trace samples the "
                                         "image's delays reach"}),
            "taps_roofline": {"kernel": "k_kk_gather_tc" if tc_flops else "k_kk_gather", "bound": "smem",
                         "achieved": achieved_taps, "peak": smem_peak, "unit": "GB/s",
                         "frac": achieved_taps / smem_peak, "traffic": _gather_traffic(fl),
                         "launch_ms": kk_launch_ms, "frames_per_launch": fl,
                         "algorithmic_bytes_per_launch": gather_bytes_alg,
                         "algorithmic_bytes": "16 B of taps (two complex64 samples) per pixel-pair "
                                              "(SURVEY 8d) x pixel-pairs per launch",
                         "peak_kind": (f"{onchip_kind} (scripts/ubench/peaks.cu: conflict-free LDS.128 "
                                       "on every SM, profiles/r02_onchip_peaks.json)") if smem_meas else
                                      "derived (148 SMs x 128 B/clk x sampled SM clock)",
                         "peak_derived_at_sampled_clock": smem_derived,
                         "pixel_pairs_per_s": pp_frame * fl / (kk_launch_ms / 1e3),
                         "pixel_pairs_per_s_isolated": pp_frame * F / (kk_ms / 1e3),
                         "traffic_note": "ncu dram read+write per launch of the gather kernel (newest "
                                         "profiles/r*_gather_traffic.json); below the compulsory HBM "
                                         "bytes because the gather reads only the trace samples the "
                                         "image's delays reach"},
            "hbm_roofline": {"kernel": "k_kk_gather_tc" if tc_flops else "k_kk_gather", "bound": "hbm",
                             "achieved": achieved_hbm, "peak": hbm_peak, "unit": "GB/s",
                             "frac": achieved_hbm / hbm_peak, "peak_kind": peak_kind,
                             "algorithmic_bytes_per_launch": compulsory,
                             "algorithmic_bytes": "compulsory HBM per launch: traces read + IQ/intensity "
                                                  "write + tables (SURVEY 8d); not the binding bound"},
            "l2_roofline": _l2_roofline(achieved_taps),
            "frame_roofline": {"bound": "hbm", "bytes_per_frame": frame_bytes,
                               "achieved": value / world * frame_bytes / 1e9, "peak": hbm_peak,
                               "unit": "GB/s", "frac": value / world * frame_bytes / 1e9 / hbm_peak,
                               "algorithmic_bytes": "SURVEY 8(d) compulsory HBM per frame: RF in "
                                                    "+ traces write/read + IQ out + tables"},
            "stage1_roofline": {"kernels": "k_r2c + k_contract_sym + k_c2c", "bound": "hbm",
                                "achieved": s1_min / (dec_ms / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                                "frac": s1_min / (dec_ms / 1e3) / 1e9 / hbm_peak, "ms": dec_ms,
                                "algorithmic_bytes_per_step": s1_min,
                                "algorithmic_bytes": "compulsory: RF in (float32) + decomposed traces out "
                                                     "(complex64)",
                                "structure_bytes_per_step": s1_bytes,
                                "structure_frac": s1_achieved / hbm_peak,
                                "structure_note": "bytes the three-kernel structure moves (RF in, spectra "
                                                  "written and read back, contracted bins written and read "
                                                  "back, traces out) over the same time",
                                "tflops": s1_flops / (dec_ms / 1e3) / 1e12,
                                "fp32_peak_tflops": fp32_peak,
                                "fp32_peak_kind": onchip_kind if fp32_meas else "derived",
                                "flop_frac": s1_flops / (dec_ms / 1e3) / 1e12 / fp32_peak},
            "gpu_launches": int(launches),
            "clocks": clk,
            "host_binding": (f"{len(host_cpus)} CPUs local to the GPU" if host_cpus else "unbound"),
        }
        if e2e:
            line["e2e"] = e2e
            line["e2e_int16_ingest"] = e2e_i16
        if cpu:
            line["cpu_baseline"] = cpu
        print(json.dumps(line))
    eng.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_gpu_rowblock(args):
    """Config 5: one large frame per step, image row-blocks sharded over ranks,
    stage 1 replicated (or, --stage1 sharded, split by transmit with the
    trace all-gather fused into the inverse FFT's P2P stores); the gather kernel stores its rows into every rank's
    image over NVLink (P2P, CUDA IPC), NCCL all-gather as the fallback
    (strong scaling)."""
    import torch
    import torch.distributed as dist

    from paper_2603_22496_b200 import _lib, configs, shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = _init_dist(torch, dist, world, local)
    w = configs.config5()
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    rf = torch.from_numpy(configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples,
                                           seed=5)).cuda()
    rb = shard.RowBlockKK(arr, p, rx, g, rank, world, stage1=args.stage1)
    if args.stage1 == "sharded":  # each rank holds only its transmits' RF
        n0, n1 = shard.balanced_range(p.num_transmits, rank, world)
        rf = rf[n0:n1].contiguous()
    stream = torch.cuda.current_stream()

    def step():
        rb.beamform_block(rf)
        if world > 1:
            rb.gather()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    launches0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    if world > 1:
        tt = torch.tensor([ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_step = ms / args.steps
    pp = g.nx * g.nz * w.pairs
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": 1e3 / ms_step, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32",
            "dtype_detail": "complex64 spectra/traces/IQ, float32 taps and sums, float64 delay-index math",
            "data": "synthetic (seeded noise RF, shapes of BASELINE config 5)",
            "config": {"workload": w.name, "frames_per_step": 1, "pixel_pairs_per_frame": pp,
                       "parallelism": f"row-block x{world}, stage 1 {args.stage1}"
                                      + (" (trace all-gather fused into the inverse FFT)"
                                         if args.stage1 == "sharded" and rb.transport == "p2p" else "")
                                      + ", "
                                      + ("P2P stores from the gather epilogue (CUDA IPC over NVLink)"
                                         if rb.transport == "p2p" else "NCCL all-gather")},
            "pixel_pair_samples_per_s": pp * 1e3 / ms_step, "gpu_launches": int(launches),
            "clocks": clk}))
    rb.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kkb", choices=["kkb", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--frames", type=int, default=400)
    ap.add_argument("--chunk", type=int, default=None, help="frames per decomposition pass")
    ap.add_argument("--pipe-chunk", type=int, default=8, help="frames per pipelined pass")
    ap.add_argument("--pipe-slots", type=int, default=1, help="decomposition streams (1 = off)")
    ap.add_argument("--no-fuse", action="store_true",
                    help="K3 writes complex64 traces and the gather splits them (no fused planes)")
    ap.add_argument("--groups", type=int, default=1,
                    help="frame groups: decomposition of group g+1 overlaps the gather of group g")
    ap.add_argument("--e2e-chunk", type=int, default=16)
    ap.add_argument("--stage1", default="replicated", choices=["replicated", "sharded"],
                    help="config 5: decompose the whole frame on every rank, or only the "
                         "rank's transmits with a fused trace all-gather")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "kkb":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.config == 5:
        return run_gpu_rowblock(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
