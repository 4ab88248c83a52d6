"""paper_2601_22137_b200 — B200-native PRISM Newton–Schulz (arXiv 2601.22137).

Thin Python binding over the C-ABI library ``libprism.so`` (include/prism.h).
The library is loaded lazily; every compute entry point fails loudly if it is
missing (there is no CPU fallback).
"""

from .binding import (  # noqa: F401
    PrismError, Options, lib, polar, sqrt_invsqrt, PRECISION, FIT, STATUS,
)

__all__ = ["PrismError", "Options", "lib", "polar", "sqrt_invsqrt", "PRECISION", "FIT", "STATUS"]
