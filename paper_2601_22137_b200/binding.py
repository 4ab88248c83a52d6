"""placeholder; replaced by the ctypes binding."""
class PrismError(RuntimeError):
    pass
Options = lib = polar = sqrt_invsqrt = None
PRECISION = FIT = STATUS = {}
