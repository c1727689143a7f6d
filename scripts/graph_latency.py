"""Single-frame latency of the whole hot path: eager launches vs one CUDA
graph replay (KKEngine.capture), host wall clock per frame incl. sync."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2603_22496_b200 as kb  # noqa: E402
from paper_2603_22496_b200 import configs  # noqa: E402

res = {}
for cfg in (1, 2, 4, 5):
    w = configs.CONFIGS[cfg]()
    p = w.params
    eng = kb.KKEngine(w.array, p, w.receive, w.grid, frames=1)
    rf = torch.from_numpy(configs.noise_rf(p.num_transmits, w.array.num_elements,
                                           p.num_samples)[None]).cuda()
    for _ in range(3):
        eng.run(rf)
    torch.cuda.synchronize()
    ref = eng.iq.clone()
    g = eng.capture(rf)
    g.replay()
    torch.cuda.synchronize()
    same = bool(torch.equal(ref, eng.iq))

    def per_frame(fn, n):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
            torch.cuda.synchronize()
        return (time.perf_counter() - t0) / n * 1e3

    n = 20 if cfg == 5 else 300
    res[w.name] = {"eager_ms": per_frame(lambda: eng.run(rf), n),
                   "graph_ms": per_frame(g.replay, n), "bit_identical": same}
    eng.close()
print(json.dumps(res))
