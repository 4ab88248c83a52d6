"""paper_2601_22137_b200 — B200-native PRISM Newton–Schulz (arXiv 2601.22137).

Thin Python binding over the C-ABI library ``_lib/libprism.so``
(``include/prism.h``).  The library is loaded lazily; every compute entry
point raises if it is missing (there is no CPU fallback).
"""

from .binding import (  # noqa: F401
    FIT, PRECISION, STATUS, Handle, PrismError, default_handle, lib, lpt_partition, make_options, polar,
    polar_flops_per_iter, polar_host, sqrt_flops_per_iter, sqrt_invsqrt, sqrt_invsqrt_host, sign, sign_host, inv_root, inv_root_host,
    chebyshev_inverse, chebyshev_inverse_host, db_newton, db_newton_host,
)

__all__ = ["FIT", "PRECISION", "STATUS", "Handle", "PrismError", "default_handle", "lib", "lpt_partition",
           "make_options", "polar", "polar_flops_per_iter", "polar_host", "sqrt_flops_per_iter", "sqrt_invsqrt",
           "sqrt_invsqrt_host", "sign", "sign_host",
           "inv_root", "inv_root_host", "chebyshev_inverse", "chebyshev_inverse_host",
           "db_newton", "db_newton_host"]
