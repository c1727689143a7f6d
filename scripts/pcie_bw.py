"""Raw pinned host<->device copy bandwidth on the box (the ceiling of the
bench's e2e leg)."""
import json

import torch

n = 1 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(n // 8, dtype=torch.uint8).pin_memory()
d2 = torch.empty(n // 8, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}
for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)),
                 ("d2h", lambda: h.copy_(d, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record()
    torch.cuda.synchronize()
    res[name + "_GBps"] = 5 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9
# h2d with a concurrent 1/8-size d2h (the e2e leg's mix)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
with torch.cuda.stream(s1):
    for _ in range(5):
        d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    for _ in range(5):
        h2.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(s1)
torch.cuda.current_stream().wait_stream(s2)
e1.record()
torch.cuda.synchronize()
res["h2d_with_d2h_GBps"] = 5 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9
print(json.dumps(res))
