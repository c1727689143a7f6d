"""Single-frame latency breakdown helper: run the engine once per config (for an
ncu launch list)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2603_22496_b200 as kb  # noqa: E402
from paper_2603_22496_b200 import configs  # noqa: E402

for cfg in [int(c) for c in (sys.argv[1:] or ["1", "2"])]:
    w = configs.CONFIGS[cfg]()
    eng = kb.KKEngine(w.array, w.params, w.receive, w.grid, frames=1)
    p = w.params
    rf = torch.from_numpy(configs.noise_rf(p.num_transmits, w.array.num_elements, p.num_samples)[None]).cuda()
    for _ in range(3):
        eng.run(rf)
    torch.cuda.synchronize()
    eng.close()
print("ok")
