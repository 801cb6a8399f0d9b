"""Exact Gaussian-rational scalar (a + b·i with a, b in Q).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Used to run the oracle recurrences in exact arithmetic so that finite
termination (r_n = 0 exactly at iteration n, SURVEY.md §8(c) pin table) can be
checked with no rounding at all.  Only +, -, *, /, conjugate, abs² and
comparison with 0 are needed by the rational-only methods (BiCGSTAB, CGNE,
BiCOR, CORS, BiCG, CGS).
"""

from fractions import Fraction


class GaussianRational:
    __slots__ = ("re", "im")

    def __init__(self, re=0, im=0):
        self.re = Fraction(re)
        self.im = Fraction(im)

    # -- helpers ---------------------------------------------------------
    @staticmethod
    def _lift(o):
        if isinstance(o, GaussianRational):
            return o
        if isinstance(o, complex):
            return GaussianRational(Fraction(o.real), Fraction(o.imag))
        if isinstance(o, (int, Fraction, float)):
            return GaussianRational(Fraction(o), 0)
        return NotImplemented

    @property
    def real(self):
        return self.re

    @property
    def imag(self):
        return self.im

    def conjugate(self):
        return GaussianRational(self.re, -self.im)

    def abs2(self):
        return self.re * self.re + self.im * self.im

    # -- arithmetic ------------------------------------------------------
    def __add__(self, o):
        o = self._lift(o)
        if o is NotImplemented:
            return o
        return GaussianRational(self.re + o.re, self.im + o.im)

    __radd__ = __add__

    def __sub__(self, o):
        o = self._lift(o)
        if o is NotImplemented:
            return o
        return GaussianRational(self.re - o.re, self.im - o.im)

    def __rsub__(self, o):
        o = self._lift(o)
        return o if o is NotImplemented else o.__sub__(self)

    def __neg__(self):
        return GaussianRational(-self.re, -self.im)

    def __mul__(self, o):
        o = self._lift(o)
        if o is NotImplemented:
            return o
        return GaussianRational(self.re * o.re - self.im * o.im,
                                self.re * o.im + self.im * o.re)

    __rmul__ = __mul__

    def __truediv__(self, o):
        o = self._lift(o)
        if o is NotImplemented:
            return o
        d = o.abs2()
        if d == 0:
            raise ZeroDivisionError("GaussianRational division by zero")
        num = self * o.conjugate()
        return GaussianRational(num.re / d, num.im / d)

    def __rtruediv__(self, o):
        o = self._lift(o)
        return o if o is NotImplemented else o.__truediv__(self)

    def __eq__(self, o):
        o = self._lift(o)
        if o is NotImplemented:
            return o
        return self.re == o.re and self.im == o.im

    def __ne__(self, o):
        r = self.__eq__(o)
        return r if r is NotImplemented else not r

    def __hash__(self):
        return hash((self.re, self.im))

    def __complex__(self):
        return complex(float(self.re), float(self.im))

    def __repr__(self):
        return f"GR({self.re}, {self.im})"


def to_exact(a):
    """numpy array of binary floating values -> object array of GaussianRational.

    The conversion is exact (``Fraction(float)`` is the exact binary value)."""
    import numpy as np
    a = np.asarray(a)
    out = np.empty(a.shape, dtype=object)
    for idx, v in np.ndenumerate(a):
        v = complex(v)
        out[idx] = GaussianRational(Fraction(v.real), Fraction(v.imag))
    return out
