"""K5 call time at the bench shape (config 4, 400 frames, IQ + intensity +
frame max), CUDA-event median of 9 after 3 warm-ups: the number the
tensor-core gather's tuning is judged on.  KKB_LIB selects a variant build."""
import ctypes, os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2603_22496_b200 import _device as dev, _lib, configs
from paper_2603_22496_b200.beamform import build_kk_luts_device

F = int(sys.argv[1]) if len(sys.argv) > 1 else 400
MODE = sys.argv[2] if len(sys.argv) > 2 else "iq+inten+fmax"  # which outputs the epilogue writes
w = configs.config4(frames=F)
p, rx, g = w.params, w.receive, w.grid
N, M, T = p.num_transmits, rx.num_angles, p.num_samples
fs = w.array.sampling_frequency
luts = build_kk_luts_device(g, p.transmit_angles, rx.angles, p.sound_speed)
kp = ctypes.c_void_p()
_lib.call("kkb_kk_plan_create", dev.ptr(luts["lut_tx_x"]), dev.ptr(luts["lut_tx_z"]), dev.ptr(luts["lut_rx_x"]),
          dev.ptr(luts["lut_rx_z"]), N, M, T, g.nx, g.nz, None, float(fs), float((0.0 - p.start_time) * fs), 1,
          dev.stream_handle(), ctypes.byref(kp))
P = g.nx * g.nz
traces = torch.view_as_complex(torch.randn((F, N, M, T, 2), generator=torch.Generator(device="cuda").manual_seed(0),
                                           device="cuda"))
iq = torch.empty((F, P), dtype=torch.complex64, device="cuda")
inten = torch.empty((F, P), device="cuda")
fmax = torch.zeros(F, dtype=torch.int32, device="cuda")
args = (kp, dev.ptr(traces), F, N * M * T, dev.ptr(iq) if "iq" in MODE else None, _lib.KKB_OUT_C64, P,
        dev.ptr(inten) if "inten" in MODE else None, dev.ptr(fmax) if "fmax" in MODE else None, dev.stream_handle())
for _ in range(3):
    _lib.call("kkb_kk_plan_run", *args)
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(9)]
for a, b in ev:
    a.record()
    _lib.call("kkb_kk_plan_run", *args)
    b.record()
torch.cuda.synchronize()
print(os.path.basename(os.environ.get("KKB_LIB", "libkkb.so")), F, MODE, _lib.KKB_KK_INST_NAMES[_lib.last_instance() & 15],
      round(statistics.median(a.elapsed_time(b) for a, b in ev), 4))
