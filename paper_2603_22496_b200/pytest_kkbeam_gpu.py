"""pytest plugin: run the reference's own test suite with its kernels on the GPU.

    PYTHONPATH=<reference>/pkg/src:<this repo> \\
        python -m pytest -p paper_2603_22496_b200.pytest_kkbeam_gpu <reference>/pkg/tests

Rebinds kkbeam.beamform._kk_kernel / _das_kernel and
kkbeam.compress.shear_and_sum to the libkkb shims before collection
(kkbeam_plugin.install).  Direct calls to ``kb.shear_and_sum`` inside the
reference tests go through the package namespace and keep the float64
original, so those oracle comparisons stay intact.
"""

_handle = None


def pytest_configure(config):
    global _handle
    from .kkbeam_plugin import install

    _handle = install()


def pytest_terminal_summary(terminalreporter):
    from . import _lib

    terminalreporter.write_line(
        f"kkbeam kernels on the GPU: libkkb {_lib.version()}, "
        f"{_lib.launch_count()} kernel launches ({_lib.LIB_PATH})")


def pytest_unconfigure(config):
    if _handle is not None:
        _handle.restore()
