"""Per-rank work of the multi-GPU partitions, timed on ONE B200 (VERDICT r1
item 6): the sandbox grants one GPU, so 2/4/8-GPU runs cannot be measured;
this times each rank's share of the work and states the communication terms
it cannot time as explicit assumptions.

* Config 5 (strong scaling, one 1024 x 2048 frame, 961 pairs):
  - stage 1 replicated: the whole decomposition on every rank;
  - stage 1 sharded: the decomposition of the largest transmit share
    (ceil(31 / G) transmits);
  - K5 on the largest row block (ceil(1024 / G) rows x 2048), default dispatch;
  - assumed: P2P stores at 700 GB/s per GPU over NVLink 5 (the image
    block scatter overlaps the gather epilogue, so only the trace scatter of
    the sharded stage 1 is added), 15 us per host barrier.
* Config 4 (weak scaling, 400 frames per rank): frames are independent and
  no collective runs, so each rank's device-resident step equals the 1-GPU
  step; the e2e leg is bound by each GPU's own PCIe link.

CUDA-event medians of 10 runs after 3 warm-ups.  Prints one JSON object.
usage: python scripts/scaling_predict.py [out.json]
"""

from __future__ import annotations

import ctypes
import json
import math
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NVLINK_GBPS = 700.0
BARRIER_MS = 0.015


def med_ms(fn, reps=10, warm=3):
    import torch

    for _ in range(warm):
        fn()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)


def main():
    import torch

    import paper_2603_22496_b200 as kb
    from paper_2603_22496_b200 import _device as dev
    from paper_2603_22496_b200 import _lib, configs, shard
    from paper_2603_22496_b200.beamform import build_kk_luts_device

    w = configs.config5()
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    N, M, T, L = p.num_transmits, rx.num_angles, p.num_samples, arr.num_elements
    fs = arr.sampling_frequency
    shift = (0.0 - p.start_time) * fs
    rf = torch.from_numpy(configs.noise_rf(N, L, T, seed=5)).cuda()
    eng = kb.KKEngine(arr, p, rx, g, frames=1, want_db=False)
    s1_full = med_ms(lambda: eng.decompose(rf[None], n_frames=1))
    eng.decompose(rf[None], n_frames=1)
    traces = eng.traces
    luts = build_kk_luts_device(g, p.transmit_angles, rx.angles, p.sound_speed)
    out = {"tool": "scripts/scaling_predict.py", "assumptions": {
        "nvlink_GBps_per_gpu": NVLINK_GBPS, "host_barrier_ms": BARRIER_MS,
        "note": "per-rank compute measured on one B200; communication terms assumed, not measured"},
        "config5": {"stage1_replicated_ms": s1_full, "ranks": {}}}
    t1 = None
    for G in (1, 2, 4, 8):
        n_share = math.ceil(N / G)
        pos = np.ascontiguousarray(arr.positions)
        ang = np.ascontiguousarray(rx.angles)
        h = ctypes.c_void_p()
        _lib.call("kkb_decomposer_create", n_share, L, T, pos.ctypes.data, ang.ctypes.data, M, float(fs),
                  float(p.sound_speed), 1, ctypes.byref(h))
        own = torch.empty((n_share, M, T), dtype=torch.complex64, device="cuda")
        sub = rf[:n_share].contiguous()
        s1_shard = med_ms(lambda: _lib.call("kkb_decomposer_run", h, dev.ptr(sub), 1, dev.ptr(own),
                                            dev.stream_handle()))
        _lib.load().kkb_decomposer_destroy(h)
        r0, r1 = shard.row_block_range(g.nx, 0, G)
        ltx = luts["lut_tx_x"][r0:r1].contiguous()
        lrx = luts["lut_rx_x"][r0:r1].contiguous()
        kp = ctypes.c_void_p()
        _lib.call("kkb_kk_plan_create", dev.ptr(ltx), dev.ptr(luts["lut_tx_z"]), dev.ptr(lrx),
                  dev.ptr(luts["lut_rx_z"]), N, M, T, r1 - r0, g.nz, None, float(fs), float(shift), 1,
                  dev.stream_handle(), ctypes.byref(kp))
        blk = torch.empty((r1 - r0, g.nz), dtype=torch.complex64, device="cuda")
        k5 = med_ms(lambda: _lib.call("kkb_kk_plan_run", kp, dev.ptr(traces), 1, 0, dev.ptr(blk),
                                      _lib.KKB_OUT_C64, 0, None, None, dev.stream_handle()))
        inst = _lib.KKB_KK_INST_NAMES[_lib.last_instance() & 15]
        _lib.load().kkb_kk_plan_destroy(kp)
        tr_bytes = N * M * T * 8
        scatter_tr = (tr_bytes * (G - 1) / G) / (NVLINK_GBPS * 1e9) * 1e3 if G > 1 else 0.0
        bar = BARRIER_MS if G > 1 else 0.0
        rep = s1_full + k5 + bar
        shd = s1_shard + scatter_tr + bar + k5 + bar
        if t1 is None:
            t1 = s1_full + k5
        out["config5"]["ranks"][G] = {
            "stage1_sharded_ms": s1_shard, "k5_block_ms": k5, "k5_instance": inst, "block_rows": r1 - r0,
            "trace_scatter_ms_assumed": scatter_tr,
            "frame_ms_replicated": rep, "frame_ms_sharded": shd,
            "speedup_replicated": t1 / rep, "speedup_sharded": t1 / shd,
            "efficiency_replicated": t1 / rep / G, "efficiency_sharded": t1 / shd / G}
        print(G, json.dumps(out["config5"]["ranks"][G]), flush=True)
    eng.close()
    # config 4: per-rank step = the 1-GPU step (no collective); e2e per GPU PCIe link
    out["config4"] = {"per_rank_step": "identical to the 1-GPU step (400 frames per rank, no collective)",
                      "predicted_efficiency_device_resident": 1.0,
                      "e2e_bound": "each GPU's own PCIe link (~55 GB/s pinned H2D measured, "
                                   "profiles/r01g_pcie_bw.json); host memory must serve G x 55 GB/s "
                                   "(NUMA-local pinned buffers: paper_2603_22496_b200/_numa.py)"}
    text = json.dumps(out, indent=1)
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            f.write(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
