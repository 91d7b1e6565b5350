"""`import vortexfourier` for the reference's own test files: the
B200-native package under the reference's name (its hot-path API is the
same: NufftParams, NufftPlan, eval_nufft, eval_direct, map_to_torus,
rescale_coeffs, AccuracyWarning, basis_matrix, eval_rectilinear and the
DomainBox / SpectralField / PhysicalField types).  The reference's GPE
solver, vortex initial conditions and CLI are out of scope and absent."""

from paper_1605_01244_b200 import *  # noqa: F401,F403
from paper_1605_01244_b200 import __all__ as _all

from . import nufft, rectilinear, tube  # noqa: F401

__all__ = list(_all)
