"""K5 launch time per instance (forced with KKB_KK_INST) against the default
dispatch, on the shapes the dispatch has to choose between:

* config-5 row blocks at G = 1/2/4/8 ranks (RowBlockKK's table slice of
  rank 0: the per-rank gather of strong scaling, one frame);
* config-4 batches of F = 1 ... 400 frames (frame sharding, and the bench);
* single frames of configs 1-3.

CUDA-event time of the gather alone, median of 7 launches after 3 warm-ups.
Prints one JSON line per (shape, instance).  Predicts per-rank K5 time of the
multi-GPU runs that the one-GPU sandbox cannot execute.
"""

from __future__ import annotations

import ctypes
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    from paper_2603_22496_b200 import _device as dev
    from paper_2603_22496_b200 import _lib, configs, shard
    from paper_2603_22496_b200.beamform import build_kk_luts_device

    out = open(sys.argv[1], "w") if len(sys.argv) > 1 else sys.stdout

    def time_plan(kp, traces, F, P, reps=7):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * reps)]
        s = dev.stream_handle()
        NMT = traces[0].numel()
        iq = torch.empty((F, P), dtype=torch.complex64, device="cuda")
        for _ in range(3):
            _lib.call("kkb_kk_plan_run", kp, dev.ptr(traces), F, NMT, dev.ptr(iq), _lib.KKB_OUT_C64, P,
                      None, None, s)
        for r in range(reps):
            ev[2 * r].record()
            _lib.call("kkb_kk_plan_run", kp, dev.ptr(traces), F, NMT, dev.ptr(iq), _lib.KKB_OUT_C64, P,
                      None, None, s)
            ev[2 * r + 1].record()
        torch.cuda.synchronize()
        return statistics.median(ev[2 * r].elapsed_time(ev[2 * r + 1]) for r in range(reps)), \
            _lib.KKB_KK_INST_NAMES[_lib.last_instance() & 15]

    def sweep(name, w, F, rows=None):
        p, rx, g = w.params, w.receive, w.grid
        N, M, T = p.num_transmits, rx.num_angles, p.num_samples
        fs = w.array.sampling_frequency
        shift = (0.0 - p.start_time) * fs
        luts = build_kk_luts_device(g, p.transmit_angles, rx.angles, p.sound_speed)
        ix0, ix1 = rows if rows else (0, g.nx)
        ltx = luts["lut_tx_x"][ix0:ix1].contiguous()
        lrx = luts["lut_rx_x"][ix0:ix1].contiguous()
        nx = ix1 - ix0
        kp = ctypes.c_void_p()
        _lib.call("kkb_kk_plan_create", dev.ptr(ltx), dev.ptr(luts["lut_tx_z"]), dev.ptr(lrx),
                  dev.ptr(luts["lut_rx_z"]), N, M, T, nx, g.nz, None, float(fs), float(shift), 1,
                  dev.stream_handle(), ctypes.byref(kp))
        gen = torch.Generator(device="cuda").manual_seed(0)
        tr = torch.randn((F, N, M, T, 2), generator=gen, device="cuda")
        traces = torch.view_as_complex(tr)
        pp = nx * g.nz * N * M * F
        for inst in ("default", "big_fr", "big", "mid", "small", "direct"):
            if inst == "direct" and pp > 5e9:
                continue
            if inst == "default":
                os.environ.pop("KKB_KK_INST", None)
            else:
                os.environ["KKB_KK_INST"] = inst
            ms, ran = time_plan(kp, traces, F, nx * g.nz)
            os.environ.pop("KKB_KK_INST", None)
            rec = {"shape": name, "frames": F, "rows": nx, "nz": g.nz, "pairs": N * M, "asked": inst,
                   "ran": ran, "ms": round(ms, 4), "pp_per_s": pp / (ms * 1e-3)}
            print(json.dumps(rec), file=out, flush=True)
        _lib.load().kkb_kk_plan_destroy(kp)
        del traces, tr

    w5 = configs.config5()
    for G in (1, 2, 4, 8):
        sweep(f"config5_rowblock_G{G}", w5, 1, rows=shard.row_block_range(w5.grid.nx, 0, G))
    for F in (1, 2, 4, 8, 12, 16, 20, 24, 32, 64, 400):
        sweep("config4", configs.config4(frames=F), F)
    for c in (1, 2, 3):
        sweep(f"config{c}", configs.CONFIGS[c](), 1)
        sweep(f"config{c}", configs.CONFIGS[c](), 16)


if __name__ == "__main__":
    main()
