"""KKRF container goldens written and read by the REFERENCE itself.

Run in the build container (needs /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_kkrf_golden.py

Writes tests/golden/kkrf/{real,analytic,compressed}.kkrf with the reference's
write_container, plus kkrf.npz holding what the reference's read_container
returns for each file and the FileFormatError text it raises for a set of
byte-level corruptions (applied identically by the tests).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))

# (label, byte offset, replacement bytes | None = truncate at offset)
CORRUPTIONS = [
    ("short_head", 40, None),
    ("magic", 0, b"KKRG"),
    ("version", 4, (2).to_bytes(2, "little")),
    ("kind", 6, bytes([3])),
    ("zero_n", 7, (0).to_bytes(4, "little")),
    ("neg_fs", 19, np.float64(-1.0).tobytes()),
    ("zero_pitch", 43, np.float64(0.0).tobytes()),
    ("short_payload", -4, None),
    ("long_payload", 10 ** 9, b"\x00\x00\x00\x00"),
]


def corrupt(blob: bytes, off: int, rep) -> bytes:
    if rep is None:
        return blob[:off] if off >= 0 else blob[:len(blob) + off]
    if off >= len(blob):
        return blob + rep
    return blob[:off] + rep + blob[off + len(rep):]


def main():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, REF_SRC)
    import kkbeam as kb
    from kkbeam import rffile

    d = os.path.join(OUT, "kkrf")
    os.makedirs(d, exist_ok=True)
    rng = np.random.default_rng(11)
    arr = kb.TransducerArray(4, 0.3e-3, 5.2e6, 20.8e6, 0.6)
    params = kb.AcquisitionParams(1540.0, kb.transmit_angles(3, np.deg2rad(10)), 8, start_time=1e-6)
    real = kb.RFVolume(rng.standard_normal((3, 4, 8)).astype(np.float32), arr, params)
    an = kb.AnalyticRF((rng.standard_normal((3, 4, 8)) + 1j * rng.standard_normal((3, 4, 8)))
                       .astype(np.complex64), arr, params)
    rx = kb.explicit_angles(np.deg2rad([-2.0, -1.0, 0.0, 1.0, 2.0]), np.deg2rad(10))
    comp = kb.CompressedRF((rng.standard_normal((3, 5, 8)) + 1j * rng.standard_normal((3, 5, 8)))
                           .astype(np.complex64), rx, params, array=None, sampling_frequency=20.8e6)
    out = {}
    for name, cont in (("real", real), ("analytic", an), ("compressed", comp)):
        path = os.path.join(d, f"{name}.kkrf")
        rffile.write_container(path, cont)
        back = rffile.read_container(path)
        out[f"{name}_data"] = back.data
        out[f"{name}_tx"] = back.params.transmit_angles
        out[f"{name}_meta"] = np.array([back.params.sound_speed, back.params.start_time,
                                        back.params.num_samples], np.float64)
        if name == "compressed":
            out[f"{name}_rx"] = back.receive_angles.angles
            out[f"{name}_fs"] = np.float64(back.sampling_frequency)
        else:
            a = back.array
            out[f"{name}_array"] = np.array([a.num_elements, a.pitch, a.center_frequency,
                                             a.sampling_frequency, a.fractional_bandwidth])
        blob = open(path, "rb").read()
        for label, off, rep in CORRUPTIONS:
            if label == "zero_pitch" and name == "compressed":
                continue
            bad = os.path.join(d, "_tmp.kkrf")
            with open(bad, "wb") as f:
                f.write(corrupt(blob, off, rep))
            try:
                rffile.read_container(bad)
                msg = "OK"
            except Exception as exc:  # noqa: BLE001 - record the reference's behaviour
                msg = f"{type(exc).__name__}: {exc}".replace(bad, "<path>")
            out[f"{name}_err_{label}"] = np.array(msg)
            os.remove(bad)
    np.savez_compressed(os.path.join(OUT, "kkrf.npz"), **out)
    print("kkrf goldens:", sorted(os.listdir(d)))


if __name__ == "__main__":
    main()
