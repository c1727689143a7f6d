"""K7 DAS comparison rate on the config-2 DAS workload (75
transmits x 128 elements x 256 x 400 pixels = 9.83e8 pixel·tx·element samples;
the reference takes 4.74 s on 8 threads).  Device-resident analytic data
(seeded noise), CUDA-event timing after warm-up."""
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_22496_b200 as kb  # noqa: E402
from paper_2603_22496_b200 import _device as dev, _lib, configs  # noqa: E402

w = configs.config2()
params, _ = w.extra_receive["das75"]
arr, g = w.array, w.grid
luts = kb.build_das_luts(g, arr, params)
t = dev.require_cuda()
rng = np.random.default_rng(0)
N, L, T = params.num_transmits, arr.num_elements, params.num_samples
data = t.complex(t.randn(N, L, T, device="cuda"), t.randn(N, L, T, device="cuda"))
out = t.empty((g.nx, g.nz), dtype=t.complex64, device="cuda")
xd, zd = dev.to_device(g.x), dev.to_device(g.z)
fs = arr.sampling_frequency
res = {}
for label, tan_max in (("ungated", math.inf), ("gated_0.3rad", math.tan(0.3))):
    def launch():
        _lib.call("kkb_das", dev.ptr(data), N, L, T, dev.ptr(luts.dev("lut_tx_x")),
                  dev.ptr(luts.dev("lut_tx_z")), dev.ptr(luts.dev("lut_rx_hypot")),
                  int(luts.lut_rx_hypot.shape[0]), dev.ptr(luts.dev("rx_base")),
                  dev.ptr(luts.dev("rx_frac")), dev.ptr(xd), dev.ptr(zd),
                  dev.ptr(luts.dev("element_positions")), float(tan_max), None, float(fs),
                  float(-params.start_time * fs), 1, g.nx, g.nz, dev.ptr(out), _lib.KKB_OUT_C64,
                  dev.stream_handle())
    for _ in range(3):
        launch()
    e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    t.cuda.synchronize()
    e0.record()
    reps = 10
    for _ in range(reps):
        launch()
    e1.record()
    t.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    samples = N * L * g.nx * g.nz
    res[label] = {"ms": ms, "samples_per_s": samples / (ms * 1e-3)}
print(json.dumps({"workload": "config2 DAS (75 tx x 128 el, 256x400 px, T=2048)",
                  "samples": N * L * g.nx * g.nz, **res}))
