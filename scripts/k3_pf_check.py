"""Bit-identity check of the two K3 forms (KKB_K3_PREFETCH=1, the default
persistent kernel with bulk-copy prefetch, vs =0, the one-shot kernel): run
in two processes, each saves the decomposed traces' planes-driven IQ of a
seeded config-4 batch (tensor-core bench path), then compare.
    KKB_K3_PREFETCH=0 python scripts/k3_pf_check.py out0.npy
    KKB_K3_PREFETCH=1 python scripts/k3_pf_check.py out1.npy
    python scripts/k3_pf_check.py --compare out0.npy out1.npy"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

if sys.argv[1] == "--compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    same = a.tobytes() == b.tobytes()
    print(f"k3 forms bit-identical: {same} (shape {a.shape}, max|diff| {np.abs(a - b).max():.3e})")
    sys.exit(0 if same else 1)

import torch

import paper_2603_22496_b200 as kb
from paper_2603_22496_b200 import configs

for F in (48, 61):  # full and ragged last frame group
    w = configs.config4(frames=F)
    eng = kb.KKEngine(w.array, w.params, w.receive, w.grid, frames=F, fuse_tc=True)
    assert eng.fused, F
    g = torch.Generator(device="cuda").manual_seed(11 + F)
    rf = torch.randn((F, w.params.num_transmits, w.array.num_elements, w.params.num_samples),
                     generator=g, device="cuda", dtype=torch.float32)
    iq = eng.run(rf)
    torch.cuda.synchronize()
    out = iq.cpu().numpy()
    eng.close()
    if F == 48:
        res = out
    else:
        res = np.concatenate([res.reshape(-1), out.reshape(-1)])
np.save(sys.argv[1], res)
print("saved", sys.argv[1], res.shape)
