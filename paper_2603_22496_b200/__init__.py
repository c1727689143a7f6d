"""B200-native KK beamforming hot path (arXiv 2603.22496).

Drop-in for the hot path of the reference package ``kkbeam``: the same
public names, container types, sampling-scheme objects and error types for
stage 1 (analytic signal + receive decomposition) and stage 2 (delay
tables, kk / das image formation, detection and compounding), computed by
hand-written sm_100a CUDA kernels in ``libkkb.so`` (``include/kkb.h``).
``KKEngine`` is the device-resident batched pipeline for throughput.

There is no CPU fallback: without the CUDA library or a GPU the compute
entry points raise ``DeviceError``.
"""

from .bench import (STAGES, StageTimings, bench_csv_text, bench_das, bench_kk, format_bench_table,
                    noise_volume, write_bench_csv)
from .beamform import (BeamformConfig, DelayLUTSet, build_das_luts, build_kk_luts,
                       cache_model_entries, compound_coherent, compound_incoherent, das,
                       intensity, kk)
from .compress import compress, compression_ratio, guard_band_samples, shear_and_sum
from .core import (AcquisitionParams, AnalyticRF, ComplexImage, CompressedRF, ImageGrid,
                   IntensityImage, RFVolume, TransducerArray, element_positions, sample_index)
from .errors import (ConfigError, DataError, DeviceError, FileFormatError, GeometryError,
                     GuardBandError, KKBeamError, MetricError, RoiError, WindowOverflowError)
from .rffile import read_container, write_container
from .sampling import (ReceiveAngleSet, SupportSample, confocal_angles, explicit_angles, support,
                       transmit_angles, uniform_vernier_angles)
from .simulate import (Phantom, Pulse, Scatterer, make_pulse, merge_phantoms, render_rf_device,
                       simulate_rf, speckle_phantom, wire_phantom)
from .spectral import analytic_signal, one_sided_weights

__version__ = "0.1.0"


def __getattr__(name):
    # lazy: importing the engine pulls in torch
    if name in ("KKEngine", "MultiSetEngine"):
        from . import engine

        return getattr(engine, name)
    raise AttributeError(name)
