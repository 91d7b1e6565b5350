"""vortexfourier.nufft for the reference tests: public API plus the private
helpers they import (_kb_beta, _kb_transform, _kb_values, _oversampled_size)."""

from paper_1605_01244_b200.nufft import *  # noqa: F401,F403
from paper_1605_01244_b200.nufft import (  # noqa: F401
    _kb_beta,
    _kb_transform,
    _kb_values,
    _oversampled_size,
)
