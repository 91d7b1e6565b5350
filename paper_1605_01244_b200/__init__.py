"""B200-native 3D NFFT trafo: drop-in for the hot path of the reference
package `vortexfourier` (scattered-point and rectilinear-grid evaluation of a
3D truncated Fourier series).  The evaluators run hand-written sm_100a
kernels through the C ABI in include/vfnfft.h (libvfnfft.so, built in-tree).
"""

from . import formats, pipeline
from .fourier import (
    DomainBox,
    PhysicalField,
    SpectralField,
    decompose,
    fft_workers,
    regular_grid,
    set_fft_workers,
    synthesize_regular,
)
from .nufft import (
    AccuracyWarning,
    NufftParams,
    NufftPlan,
    eval_direct,
    eval_nufft,
    map_to_torus,
    rescale_coeffs,
)
from .rectilinear import basis_matrix, eval_rectilinear
from .tube import Snapshot, TubePointCloud, computational_domain, snapshot_spectral, tube_eval

__all__ = [
    "AccuracyWarning",
    "DomainBox",
    "NufftParams",
    "NufftPlan",
    "PhysicalField",
    "Snapshot",
    "SpectralField",
    "TubePointCloud",
    "computational_domain",
    "decompose",
    "formats",
    "pipeline",
    "basis_matrix",
    "eval_direct",
    "eval_nufft",
    "eval_rectilinear",
    "fft_workers",
    "map_to_torus",
    "regular_grid",
    "rescale_coeffs",
    "set_fft_workers",
    "snapshot_spectral",
    "synthesize_regular",
    "tube_eval",
]

__version__ = "0.1.0"
