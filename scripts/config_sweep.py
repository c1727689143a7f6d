"""Per-configuration throughput of the whole KK path
on one B200, next to the oracle port on the host cores.

For each workload: device-resident batched rate (F frames per launch
sequence, CUDA events), single-frame latency (F = 1), pixel-pair samples/s,
and the CPU port's per-frame time (numpy/scipy stage 1 + C/OpenMP kk, all
host cores, bounded sample).  Config 3 reports its four sampling schemes."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_22496_b200 as kb  # noqa: E402
from paper_2603_22496_b200 import configs  # noqa: E402


def device_rate(w, params, rx, frames, reps=5, fuse_tc=False):
    import torch

    eng = kb.KKEngine(w.array, params, rx, w.grid, frames=frames, fuse_tc=fuse_tc)
    N, L, T = params.num_transmits, w.array.num_elements, params.num_samples
    base = configs.noise_rf(N, L, T, seed=0)
    rf = torch.from_numpy(np.broadcast_to(base, (frames,) + base.shape).copy()).cuda()
    for _ in range(3):
        eng.run(rf)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        eng.run(rf)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    pp = eng.pixel_pairs_per_frame
    if fuse_tc:
        from paper_2603_22496_b200 import _lib
        pp = (pp, eng.fused, _lib.KKB_KK_INST_NAMES[_lib.last_instance() & 15])
    eng.close()
    return ms, pp


def multiset_rate(w, params, sets, frames, reps=5):
    """Incoherent compounding of several receive sets (MultiSetEngine: one
    decomposition over the union, one gather launch for all sets)."""
    import torch

    eng = kb.MultiSetEngine(w.array, params, sets, w.grid, frames, mode="incoherent")
    N, L, T = params.num_transmits, w.array.num_elements, params.num_samples
    base = configs.noise_rf(N, L, T, seed=0)
    rf = torch.from_numpy(np.broadcast_to(base, (frames,) + base.shape).copy()).cuda()
    for _ in range(3):
        eng.run(rf)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        eng.run(rf)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    pp = eng.pixel_pairs_per_frame
    eng.close()
    return ms, pp


def cpu_frame_ms(w, params, rx, seconds=4.0):
    from oracle import kkbeam_oracle as O

    O.build()
    arr, g = w.array, w.grid
    fs, c = arr.sampling_frequency, params.sound_speed
    luts = O.kk_luts(g.x, g.z, params.transmit_angles, rx.angles, c)
    rf = configs.noise_rf(params.num_transmits, arr.num_elements, params.num_samples, seed=0)
    ones = np.ones(rx.num_angles)
    shift = -params.start_time * fs

    def frame():
        tr = O.decompose_c64_staged(rf, fs, arr.positions, rx.angles, c)
        O.kk_kernel(tr, *luts, ones, fs, shift)

    frame()
    n, t0 = 0, time.perf_counter()
    while n < 1 or time.perf_counter() - t0 < seconds:
        frame()
        n += 1
    return (time.perf_counter() - t0) / n * 1e3


def main():
    cases = []
    for cfg in (1, 2, 4, 5):
        w = configs.CONFIGS[cfg]()
        cases.append((w.name, w, w.params, w.receive))
    w3 = configs.config3()
    for name, (p, rx) in w3.extra_receive.items():
        cases.append((f"config3_{name}", w3, p, rx))
    out = []
    for name, w, p, rx in cases:
        big = name.startswith("config5")
        F = 1 if big else 16
        ms_b, pp = device_rate(w, p, rx, F, reps=3 if big else 5)
        ms_1, _ = device_rate(w, p, rx, 1, reps=3 if big else 10)
        cpu = None if big else cpu_frame_ms(w, p, rx)
        row = {"workload": name, "pairs": p.num_transmits * rx.num_angles,
               "grid": [w.grid.nx, w.grid.nz], "T": p.num_samples,
               "gpu_ms_per_frame_batched": ms_b / F, "batch": F,
               "gpu_ms_single_frame": ms_1, "pixel_pairs_per_s": pp / (ms_b / F / 1e3),
               "cpu_port_ms_per_frame": cpu, "cpu_threads": os.cpu_count()}
        if not big:  # large batches: the tensor-core gather (fused from stage 1 where eligible)
            ms_l, (_, fused, inst) = device_rate(w, p, rx, 128, reps=3, fuse_tc=True)
            row.update({"gpu_ms_per_frame_batch128": ms_l / 128, "batch128_gather": inst,
                        "batch128_fused_stage1": fused, "pixel_pairs_per_s_batch128": pp / (ms_l / 128 / 1e3)})
        out.append(row)
        print(json.dumps(row), flush=True)
    # config 3 hybrid compounded incoherently (cli.py:257-266): confocal(25, 3)
    # and vernier(25, 2) images, sum of |B_j|^2, one gather launch
    hp = w3.extra_receive["hybrid"][0]
    d = hp.transmit_angles[1] - hp.transmit_angles[0]
    sets = [kb.confocal_angles(25, 3, 12 * d), kb.uniform_vernier_angles(25, 2, 12 * d, 0)]
    ms_b, pp = multiset_rate(w3, hp, sets, 16)
    ms_1, _ = multiset_rate(w3, hp, sets, 1, reps=10)
    row = {"workload": "config3_hybrid_incoherent", "pairs": pp // (w3.grid.nx * w3.grid.nz),
           "grid": [w3.grid.nx, w3.grid.nz], "T": hp.num_samples,
           "gpu_ms_per_frame_batched": ms_b / 16, "batch": 16, "gpu_ms_single_frame": ms_1,
           "pixel_pairs_per_s": pp / (ms_b / 16 / 1e3), "cpu_port_ms_per_frame": None,
           "cpu_threads": os.cpu_count()}
    print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
