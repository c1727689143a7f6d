import ctypes, os, sys
sys.path.insert(0, '/root/repo')
import torch
from paper_2603_22496_b200 import _device as dev, _lib, configs
from paper_2603_22496_b200.beamform import build_kk_luts_device
F = 400
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
traces = torch.view_as_complex(torch.randn((F, N, M, T, 2), device="cuda"))
iq = torch.empty((F, P), dtype=torch.complex64, device="cuda")
inten = torch.empty((F, P), device="cuda")
fmax = torch.zeros(F + 200, dtype=torch.int32, device="cuda")  # noqa  # + profile slots (u64 220..224, past the frame maxima)
_lib.call("kkb_kk_plan_run", kp, dev.ptr(traces), F, N * M * T, dev.ptr(iq), _lib.KKB_OUT_C64, P, dev.ptr(inten), dev.ptr(fmax), dev.stream_handle())
torch.cuda.synchronize()
v = fmax.cpu().view(torch.int64)[220:235].tolist()
n = v[4]
print({"mma_warp": {"pairs": n, "dfree_wait": v[0] / n, "a_full_wait": v[1] / n, "b_full_wait": v[2] / n,
                    "issue": v[3] / n},
       "producer_thread0": {"loop": v[10] / n * 148, "a_empty_wait": v[11] / n * 148, "tab_full_wait": v[12] / n * 148},
       "tma_lane": {"loop": v[13] / n * 148, "b_empty_wait": v[14] / n * 148},
       "note": "cycles per (tile, pair); producer / TMA sums are per CTA (one thread each), scaled by the 148 CTAs"})
