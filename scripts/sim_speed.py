"""Time the K8 forward simulator on the config-5 speckle medium (SURVEY §8(d):
~3.3 M scatterers, 20 per resolution cell) against the C restatement of
_render_traces (oracle, all host cores) on a scatterer subset."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_22496_b200 as kb  # noqa: E402
from paper_2603_22496_b200 import configs  # noqa: E402
from paper_2603_22496_b200 import _device as dev  # noqa: E402

w = configs.config5()
a = w.array.aperture
ph = kb.speckle_phantom((-a / 2, a / 2, 2e-3, 52e-3), 1.3e9, seed=0)
pulse = kb.make_pulse(7.5e6, 0.6, 30e6)
t = dev.require_cuda()
kb.render_rf_device(w.array, w.params, kb.Phantom(ph.x[:1000], ph.z[:1000], ph.reflectivity[:1000]),
                    pulse)  # warm-up
t.cuda.synchronize()
t0 = time.perf_counter()
out = kb.render_rf_device(w.array, w.params, ph, pulse)
t.cuda.synchronize()
gpu_s = time.perf_counter() - t0
sub = 20000
from oracle import kkbeam_oracle as O  # noqa: E402

O.build()
t0 = time.perf_counter()
O.simulate_rf(w.array.positions, w.params.transmit_angles, w.params.sound_speed, 4096,
              w.params.start_time, 30e6, ph.x[:sub], ph.z[:sub], ph.reflectivity[:sub],
              pulse.waveform)
cpu_sub = time.perf_counter() - t0
updates = 31 * 256 * len(ph) * pulse.waveform.size
print(json.dumps({"scatterers": len(ph), "traces": 31 * 256, "pulse_len": int(pulse.waveform.size),
                  "gpu_s": gpu_s, "sample_updates_per_s": updates / gpu_s,
                  "cpu_threads": os.cpu_count(), "cpu_s_extrapolated": cpu_sub * len(ph) / sub,
                  "cpu_sample": f"{sub} scatterers in {cpu_sub:.2f} s"}))
