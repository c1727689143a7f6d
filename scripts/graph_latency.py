import sys, os, time, json
sys.path.insert(0, '/root/repo' if os.path.exists('/root/repo') else '.')
import numpy as np, torch
import paper_2603_22496_b200 as kb
from paper_2603_22496_b200 import configs
res = {}
for cfg in (1, 2, 4):
    w = configs.CONFIGS[cfg]()
    eng = kb.KKEngine(w.array, w.params, w.receive, w.grid, frames=1)
    p = w.params
    rf = torch.from_numpy(configs.noise_rf(p.num_transmits, w.array.num_elements, p.num_samples)[None]).cuda()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            eng.run(rf)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        eng.run(rf)
    torch.cuda.synchronize()
    ref = eng.iq.clone()
    g.replay(); torch.cuda.synchronize()
    same = bool(torch.equal(ref, eng.iq))
    def t(fn, n=200):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(n): fn()
        torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
    eager = t(lambda: eng.run(rf))
    graph = t(lambda: g.replay())
    res[w.name] = {"eager_ms": eager, "graph_ms": graph, "bit_identical": same}
print(json.dumps(res))
