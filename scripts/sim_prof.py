"""One K8 launch on the config-5 geometry (300 k speckle scatterers) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_22496_b200 as kb  # noqa: E402
from paper_2603_22496_b200 import configs  # noqa: E402

w = configs.config5()
a = w.array.aperture
ph = kb.speckle_phantom((-a / 2, a / 2, 2e-3, 52e-3), 1.3e8, seed=0)
kb.render_rf_device(w.array, w.params, ph, kb.make_pulse(7.5e6, 0.6, 30e6))
print("ok", len(ph))
