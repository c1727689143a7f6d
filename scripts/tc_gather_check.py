"""Tensor-core gather (KKB_KK_INST=tc) vs the FMA gather: agreement and
launch time on the bench workload and the other shapes.  Prints JSON lines."""
import ctypes, json, os, statistics, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2603_22496_b200 import _device as dev, _lib, configs
    from paper_2603_22496_b200.beamform import build_kk_luts_device

    def run(kp, traces, F, P, inst, reps=5):
        if inst:
            os.environ["KKB_KK_INST"] = inst
        else:
            os.environ.pop("KKB_KK_INST", None)
        NMT = traces[0].numel()
        iq = torch.empty((F, P), dtype=torch.complex64, device="cuda")
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        _lib.call("kkb_kk_plan_run", kp, dev.ptr(traces), F, NMT, dev.ptr(iq), _lib.KKB_OUT_C64, P, None, None,
                  dev.stream_handle())
        for a, b in ev:
            a.record()
            _lib.call("kkb_kk_plan_run", kp, dev.ptr(traces), F, NMT, dev.ptr(iq), _lib.KKB_OUT_C64, P, None,
                      None, dev.stream_handle())
            b.record()
        torch.cuda.synchronize()
        ran = _lib.KKB_KK_INST_NAMES[_lib.last_instance() & 15]
        os.environ.pop("KKB_KK_INST", None)
        return iq, statistics.median(a.elapsed_time(b) for a, b in ev), ran

    for name, w, F, linear in (("config4", configs.config4(frames=400), 400, 1), ("config4", configs.config4(frames=64), 64, 1),
                               ("config4_nearest", configs.config4(frames=64), 64, 0),
                               ("config1", configs.config1(), 16, 1), ("config5", configs.config5(), 1, 1),
                               ("config2", configs.config2(), 16, 1)):
        p, rx, g = w.params, w.receive, w.grid
        N, M, T = p.num_transmits, rx.num_angles, p.num_samples
        fs = w.array.sampling_frequency
        luts = build_kk_luts_device(g, p.transmit_angles, rx.angles, p.sound_speed)
        kp = ctypes.c_void_p()
        _lib.call("kkb_kk_plan_create", dev.ptr(luts["lut_tx_x"]), dev.ptr(luts["lut_tx_z"]), dev.ptr(luts["lut_rx_x"]),
                  dev.ptr(luts["lut_rx_z"]), N, M, T, g.nx, g.nz, None, float(fs), float((0.0 - p.start_time) * fs),
                  linear, dev.stream_handle(), ctypes.byref(kp))
        gen = torch.Generator(device="cuda").manual_seed(1)
        traces = torch.view_as_complex(torch.randn((F, N, M, T, 2), generator=gen, device="cuda"))
        P = g.nx * g.nz
        ref, t_ref, ran_ref = run(kp, traces, F, P, None)
        got, t_tc, ran_tc = run(kp, traces, F, P, "tc")
        err = float((torch.linalg.vector_norm(got - ref) / torch.linalg.vector_norm(ref)).item())
        print(json.dumps({"shape": name, "frames": F, "linear": linear, "fma_instance": ran_ref, "fma_ms": t_ref,
                          "tc_instance": ran_tc, "tc_ms": t_tc, "rel_l2_tc_vs_fma": err,
                          "window_check": _lib.load().kkb_kk_plan_window_check(kp),
                          "device_error": _lib.take_device_error()}), flush=True)
        _lib.load().kkb_kk_plan_destroy(kp)


if __name__ == "__main__":
    main()
