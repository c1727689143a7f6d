"""Stage 1 at the bench shape (config 4, 400 frames) in pipelined chunks
(kkb_decomposer_set_pipeline: K1 of chunk c+1 overlapping K2 of chunk c on
rotating streams, the chunk's spectra consumed while L2-resident) against
one pass: CUDA events around KKEngine.decompose."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2603_22496_b200 as kb
from paper_2603_22496_b200 import configs

F = 400
w = configs.config4(frames=F)
arr, p, rx, g = w.array, w.params, w.receive, w.grid
rf = torch.randn(F, p.num_transmits, arr.num_elements, p.num_samples, device="cuda")
res = []
for pipe in [None, (4, 2), (4, 3), (8, 2), (8, 3), (16, 2), (2, 3)]:
    eng = kb.KKEngine(arr, p, rx, g, frames=F, want_db=False, pipeline=pipe)
    for _ in range(3):
        eng.decompose(rf)
    torch.cuda.synchronize()
    ts = []
    for _ in range(8):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        eng.decompose(rf)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    res.append({"pipeline": pipe, "decompose_ms": float(np.median(ts))})
    eng.close()
    print(json.dumps(res[-1]), flush=True)
