"""FMA vs tensor-core gather launch time over batch sizes (config 4 and 2,
linear and nearest): the data behind kk_gather.cu's dispatch rule.
Prints JSON lines; usage: python scripts/tc_gather_sweep.py [out.jsonl]"""
import ctypes, json, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2603_22496_b200 import _device as dev, _lib, configs
    from paper_2603_22496_b200.beamform import build_kk_luts_device

    out = open(sys.argv[1], "w") if len(sys.argv) > 1 else None

    def run(kp, traces, F, P, inst, reps=7):
        os.environ["KKB_KK_INST"] = inst
        NMT = traces[0].numel()
        iq = torch.empty((F, P), dtype=torch.complex64, device="cuda")
        inten = torch.empty((F, P), dtype=torch.float32, device="cuda")
        fmax = torch.zeros(F, dtype=torch.int32, device="cuda")
        args = lambda: (kp, dev.ptr(traces), F, NMT, dev.ptr(iq), _lib.KKB_OUT_C64, P, dev.ptr(inten), dev.ptr(fmax),
                        dev.stream_handle())
        _lib.call("kkb_kk_plan_run", *args())
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for a, b in ev:
            a.record()
            _lib.call("kkb_kk_plan_run", *args())
            b.record()
        torch.cuda.synchronize()
        ran = _lib.KKB_KK_INST_NAMES[_lib.last_instance() & 15]
        os.environ.pop("KKB_KK_INST", None)
        return iq, statistics.median(a.elapsed_time(b) for a, b in ev), ran

    for name, mk in (("config4", lambda F: configs.config4(frames=F)), ("config2", lambda F: configs.config2())):
        w = mk(1)
        p, rx, g = w.params, w.receive, w.grid
        N, M, T = p.num_transmits, rx.num_angles, p.num_samples
        fs = w.array.sampling_frequency
        luts = build_kk_luts_device(g, p.transmit_angles, rx.angles, p.sound_speed)
        for linear in (1, 0):
            kp = ctypes.c_void_p()
            _lib.call("kkb_kk_plan_create", dev.ptr(luts["lut_tx_x"]), dev.ptr(luts["lut_tx_z"]),
                      dev.ptr(luts["lut_rx_x"]), dev.ptr(luts["lut_rx_z"]), N, M, T, g.nx, g.nz, None, float(fs),
                      float((0.0 - p.start_time) * fs), linear, dev.stream_handle(), ctypes.byref(kp))
            for F in (8, 16, 32, 48, 64, 96, 128, 192, 256, 400):
                gen = torch.Generator(device="cuda").manual_seed(F)
                traces = torch.view_as_complex(torch.randn((F, N, M, T, 2), generator=gen, device="cuda"))
                P = g.nx * g.nz
                ref, t_fma, ran_f = run(kp, traces, F, P, "natural")
                got, t_tc, ran_t = run(kp, traces, F, P, "tc")
                err = float((torch.linalg.vector_norm(got - ref) / torch.linalg.vector_norm(ref)).item())
                rec = {"shape": name, "linear": linear, "frames": F, "fma": ran_f, "fma_ms": t_fma, "tc": ran_t,
                       "tc_ms": t_tc, "rel_l2": err}
                print(json.dumps(rec), flush=True)
                if out:
                    out.write(json.dumps(rec) + "\n")
                del traces
            _lib.load().kkb_kk_plan_destroy(kp)


if __name__ == "__main__":
    main()
