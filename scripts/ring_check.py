"""Stage-1 ring mode (kkb_decomposer_set_ring): bit-identity with the
three-kernel path and decomposition time for several (slots, consumer CTAs).
Prints JSON lines.  usage: python scripts/ring_check.py [frames]"""
import json, os, statistics, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import ctypes
    import torch
    import paper_2603_22496_b200 as kb
    from paper_2603_22496_b200 import _lib, configs

    F = int(sys.argv[1]) if len(sys.argv) > 1 else 400
    w = configs.config4(frames=F)
    arr, p, rx, g = w.array, w.params, w.receive, w.grid
    base = np.stack([configs.noise_rf(p.num_transmits, arr.num_elements, p.num_samples, seed=s) for s in range(8)])
    rf = torch.empty((F, p.num_transmits, arr.num_elements, p.num_samples), dtype=torch.float32, device="cuda")
    for f0 in range(0, F, 8):
        rf[f0:f0 + 8].copy_(torch.from_numpy(base[: min(8, F - f0)]))
    eng = kb.KKEngine(arr, p, rx, g, frames=F, want_db=False)

    def timed(reps=5):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        eng.decompose(rf)
        for a, b in ev:
            a.record()
            eng.decompose(rf)
            b.record()
        torch.cuda.synchronize()
        return statistics.median(a.elapsed_time(b) for a, b in ev)

    t_ref = timed()
    ref = eng.traces.clone()
    print(json.dumps({"mode": "three-kernel", "frames": F, "decompose_ms": t_ref}), flush=True)
    for R, ctas in ((4, 74), (8, 74), (8, 148), (4, 148), (4, 37), (6, 110)):
        _lib.call("kkb_decomposer_set_ring", eng._dec, R, ctas)
        eng.traces.zero_()
        t = timed()
        flag = ctypes.c_int(0)
        _lib.call("kkb_decomposer_ring_error", eng._dec, ctypes.byref(flag))
        same = bool(torch.equal(eng.traces, ref))
        print(json.dumps({"mode": "ring", "slots": R, "consumer_ctas": ctas, "frames": F, "decompose_ms": t,
                          "bit_identical": same, "ring_error": flag.value}), flush=True)
    _lib.call("kkb_decomposer_set_ring", eng._dec, 0, 0)
    eng.close()


if __name__ == "__main__":
    main()
