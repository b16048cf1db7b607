"""GF(2) polynomial value type used by the jump API.

Mirrors the part of /root/reference/pkg/src/slprng/gf2.py that the hot path
exposes: ``GF2Poly`` (:106-175, ``.bits`` holds coefficient i in bit i),
``poly_mod_mul`` / ``poly_mod_pow`` (:208-227) and ``Gf2Error`` (:48-53).
The heavy lifting (characteristic polynomials up to degree 1024, x^J mod P)
is done by the native host library (csrc/slp_host.cpp).  The rest of the
reference's GF(2) toolkit (Berlekamp-Massey, primitivity, bit matrices) is
analysis-only and out of scope.
"""

from __future__ import annotations

from ._native import Gf2Error

__all__ = ["GF2Poly", "X", "ONE", "ZERO", "poly_mod_mul", "poly_mod_pow", "poly_weight", "Gf2Error"]

ZERO_DEGREE = float("-inf")


def _clmul(a: int, b: int) -> int:
    if a.bit_count() > b.bit_count():
        a, b = b, a
    r = 0
    i = 0
    while a:
        if a & 1:
            r ^= b << i
        a >>= 1
        i += 1
    return r


def _reduce(a: int, m: int) -> int:
    dm = m.bit_length() - 1
    while a.bit_length() - 1 >= dm:
        a ^= m << (a.bit_length() - 1 - dm)
    return a


class GF2Poly:
    """Immutable polynomial over GF(2); bit i of ``bits`` = coefficient of x^i."""

    __slots__ = ("bits",)

    def __init__(self, bits: int = 0):
        if bits < 0:
            raise ValueError("coefficient mask must be non-negative")
        object.__setattr__(self, "bits", int(bits))

    def __setattr__(self, *a):
        raise AttributeError("GF2Poly is immutable")

    @property
    def degree(self):
        return self.bits.bit_length() - 1 if self.bits else ZERO_DEGREE

    @property
    def weight(self) -> int:
        return self.bits.bit_count()

    def is_zero(self) -> bool:
        return self.bits == 0

    def coeff(self, i: int) -> int:
        return (self.bits >> i) & 1

    def __eq__(self, other):
        return isinstance(other, GF2Poly) and self.bits == other.bits

    def __hash__(self):
        return hash(("GF2Poly", self.bits))

    def __xor__(self, other):
        return GF2Poly(self.bits ^ other.bits)

    __add__ = __xor__

    def __mul__(self, other):
        return GF2Poly(_clmul(self.bits, other.bits))

    def __mod__(self, other):
        if other.bits == 0:
            raise ZeroDivisionError("polynomial modulus is zero")
        return GF2Poly(_reduce(self.bits, other.bits))

    def __repr__(self):
        return f"GF2Poly(0x{self.bits:x})"


ZERO = GF2Poly(0)
ONE = GF2Poly(1)
X = GF2Poly(2)


def poly_weight(p: GF2Poly) -> int:
    return p.weight


def _check_modulus(m: GF2Poly):
    if m.bits == 0 or m.bits == 1:
        raise ValueError("modulus must have degree >= 1")


def poly_mod_mul(a: GF2Poly, b: GF2Poly, m: GF2Poly) -> GF2Poly:
    _check_modulus(m)
    return GF2Poly(_reduce(_clmul(a.bits, b.bits), m.bits))


def poly_mod_pow(base: GF2Poly, e: int, m: GF2Poly) -> GF2Poly:
    """base**e mod m (right-to-left square and multiply)."""
    _check_modulus(m)
    if e < 0:
        raise ValueError("negative exponent")
    result = 1
    b = _reduce(base.bits, m.bits)
    while e:
        if e & 1:
            result = _reduce(_clmul(result, b), m.bits)
        e >>= 1
        if e:
            b = _reduce(_clmul(b, b), m.bits)
    return GF2Poly(result)
