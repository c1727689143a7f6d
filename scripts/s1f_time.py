"""Time the fused stage-1 kernel against K1 -> K2 at the bench shape
(config 4, 400 frames): CUDA events around kkb_decomposer_run with the
fused kernel on and off (the K3 inverse FFT runs in both)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2603_22496_b200 as kb
from paper_2603_22496_b200 import _device as dev, _lib, configs

F = int(os.environ.get("S1F_FRAMES", "400"))
w = configs.config4(frames=F)
arr, p, rx, g = w.array, w.params, w.receive, w.grid
rf = torch.randn(F, p.num_transmits, arr.num_elements, p.num_samples, device="cuda")
eng = kb.KKEngine(arr, p, rx, g, frames=F, want_db=False)
out = {}
for fused in (1, 0):
    _lib.call("kkb_decomposer_set_fused", eng._dec, fused)
    for _ in range(3):
        eng.decompose(rf)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.decompose(rf)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    out["fused" if fused else "k1_k2"] = float(np.median(ts))
print(json.dumps({"frames": F, "decompose_ms": out}))
