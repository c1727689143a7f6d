"""The two K3 forms of the fused stage 1 (the one-shot `k_c2c_planes`, default,
and the opt-in persistent bulk-copy-prefetch `k_c2c_planes_pf`,
KKB_K3_PREFETCH=1) give bit-identical images on a full and a ragged last
frame group.  The switch is read once per process, so each form runs in its
own subprocess (scripts/k3_pf_check.py)."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_k3_prefetch_form_is_bit_identical(tmp_path):
    script = os.path.join(ROOT, "scripts", "k3_pf_check.py")
    outs = []
    for pf in ("0", "1"):
        out = str(tmp_path / f"k{pf}.npy")
        env = dict(os.environ, KKB_K3_PREFETCH=pf)
        r = subprocess.run([sys.executable, script, out], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout + r.stderr
        outs.append(out)
    r = subprocess.run([sys.executable, script, "--compare", *outs], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
