"""Exact polynomial algebra for the modal DG basis on the reference triangle.

Setup-time only (never on the per-stage path).  Every basis function of the
paper is sqrt(m) times a polynomial with rational coefficients, and every
tensor entry the scheme needs is an integral of a product of such functions,
hence again rational * sqrt(m).  We therefore carry one square-free radicand
per polynomial (``RootPoly``) instead of per coefficient, which keeps
products and integrals exact with plain ``fractions.Fraction`` arithmetic.

Conventions follow the reference (``/root/reference/pkg/src/qfswe``):

* reference triangle v0=(0,0), v1=(1,0), v2=(0,1); local edge j is opposite
  vertex j and traversed counter-clockwise (symbolic.py:350-355):
  edge 0: (1-s, s), edge 1: (0, 1-s), edge 2: (s, 0);
* the basis for k <= 3 is the paper's list (PAPER.md:276-298,
  symbolic.py:413-435), in that order;
* float conversion of an exact value r*sqrt(m) is ``float(r)*sqrt(m)``
  (symbolic.py:116-119), so frozen tensors are bit-identical to the
  reference for k <= 3.

k = 4 is an extension (the reference stops at k = 3, symbolic.py:410,455):
the five degree-4 functions are exact Gram-Schmidt of x1^4, x1^3 x2,
x1^2 x2^2, x1 x2^3, x2^4 against the lower-order basis.  The scheme is
basis-invariant, so any hierarchical orthonormal completion is
admissible; this one stays inside the rational*sqrt(m) representation.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction
from functools import lru_cache

__all__ = [
    "UnsupportedOrder",
    "RootPoly",
    "EDGE_MAPS",
    "K_FUNCS",
    "MAX_ORDER",
    "monomial_integral",
    "squarefree",
    "build_basis",
    "Basis",
    "exact_float",
]

MAX_ORDER = 4
K_FUNCS = {k: (k + 1) * (k + 2) // 2 for k in range(MAX_ORDER + 1)}


class UnsupportedOrder(ValueError):
    """Polynomial order outside 0..MAX_ORDER."""


def squarefree(n: int) -> tuple[int, int]:
    """n = s*s*m with m square-free; returns (s, m)."""
    if n <= 0:
        raise ValueError("radicand must be positive")
    s, m, d = 1, n, 2
    while d * d <= m:
        while m % (d * d) == 0:
            m //= d * d
            s *= d
        d += 1
    return s, m


def exact_float(r: Fraction, m: int) -> float:
    """Correctly rounded rational times sqrt(m), the reference's conversion."""
    if r == 0:
        return 0.0
    if m == 1:
        return float(r)
    return float(r) * math.sqrt(m)


def monomial_integral(a: int, b: int) -> Fraction:
    """Exact integral of x1^a x2^b over the reference triangle: a! b!/(a+b+2)!."""
    return Fraction(math.factorial(a) * math.factorial(b), math.factorial(a + b + 2))


def _edge_power(const: int, slope: int, n: int) -> dict[int, int]:
    """(const + slope*s)^n as {power: integer coefficient}."""
    return {j: math.comb(n, j) * const ** (n - j) * slope**j
            for j in range(n + 1) if math.comb(n, j) * const ** (n - j) * slope**j}


# (x1 const, x1 slope, x2 const, x2 slope) per local edge
EDGE_MAPS = ((1, -1, 0, 1), (0, 0, 1, -1), (0, 1, 0, 0))


@dataclass(frozen=True)
class RootPoly:
    """sqrt(rad) * sum_{(a,b)} coef[(a,b)] x1^a x2^b, rad square-free."""

    rad: int
    coef: tuple  # sorted tuple of ((a, b), Fraction), no zeros

    @staticmethod
    def make(rad: int, terms: dict) -> "RootPoly":
        s, m = squarefree(rad)
        clean = {k: Fraction(v) * s for k, v in terms.items() if Fraction(v) != 0}
        return RootPoly(m if clean else 1, tuple(sorted(clean.items())))

    @property
    def terms(self) -> dict:
        return dict(self.coef)

    @property
    def degree(self) -> int:
        return max((a + b for (a, b), _ in self.coef), default=0)

    def __mul__(self, other: "RootPoly") -> "RootPoly":
        out: dict = {}
        for (a1, b1), c1 in self.coef:
            for (a2, b2), c2 in other.coef:
                key = (a1 + a2, b1 + b2)
                out[key] = out.get(key, 0) + c1 * c2
        return RootPoly.make(self.rad * other.rad, out)

    def scale(self, r: Fraction) -> "RootPoly":
        return RootPoly(self.rad, tuple((k, v * r) for k, v in self.coef if v * r != 0))

    def diff(self, var: int) -> "RootPoly":
        out = {}
        for (a, b), c in self.coef:
            if var == 1 and a:
                out[(a - 1, b)] = c * a
            elif var == 2 and b:
                out[(a, b - 1)] = c * b
        return RootPoly(self.rad if out else 1, tuple(sorted(out.items())))

    def integral(self) -> tuple[Fraction, int]:
        """Exact integral over the reference triangle as (rational, radicand)."""
        tot = sum((c * monomial_integral(a, b) for (a, b), c in self.coef), Fraction(0))
        return tot, (self.rad if tot != 0 else 1)

    def trace(self, edge: int) -> tuple[int, dict[int, Fraction]]:
        """Restriction to local edge ``edge`` as (radicand, {s power: rational})."""
        x0, x1s, y0, y1s = EDGE_MAPS[edge]
        out: dict[int, Fraction] = {}
        for (a, b), c in self.coef:
            pa = _edge_power(x0, x1s, a)
            pb = _edge_power(y0, y1s, b)
            for i, ci in pa.items():
                for j, cj in pb.items():
                    out[i + j] = out.get(i + j, 0) + c * ci * cj
        return self.rad, {n: v for n, v in out.items() if v != 0}

    def eval(self, x1, x2):
        """Floating evaluation (numpy-broadcasting)."""
        acc = 0.0
        for (a, b), c in self.coef:
            acc = acc + float(c) * x1**a * x2**b
        return acc * math.sqrt(self.rad)

    def eval_point(self, x1: float, x2: float) -> float:
        """Scalar evaluation with the reference's rounding sequence (a sum of
        float(coefficient) * x1^a * x2^b, symbolic.py:232-233), so point
        tables such as ``phi_at_vertices`` match the reference bit for bit."""
        return sum(exact_float(c, self.rad) * x1**a * x2**b for (a, b), c in self.coef)


def _paper_basis() -> list[RootPoly]:
    """The paper's k <= 3 basis, PAPER.md:276-298 (reference symbolic.py:420-435)."""
    P = RootPoly.make
    return [
        P(2, {(0, 0): 1}),
        P(1, {(0, 0): 2, (1, 0): -6}),
        P(12, {(0, 0): 1, (1, 0): -1, (0, 1): -2}),
        P(6, {(0, 0): 1, (1, 0): -8, (2, 0): 10}),
        P(3, {(0, 0): -1, (1, 0): -4, (2, 0): 5, (0, 1): 12, (0, 2): -15}),
        P(45, {(0, 0): 1, (1, 0): -4, (2, 0): 3, (0, 1): -4, (1, 1): 8, (0, 2): 3}),
        P(8, {(0, 0): -1, (1, 0): 15, (2, 0): -45, (3, 0): 35}),
        P(24, {(0, 0): -1, (1, 0): 13, (2, 0): -33, (3, 0): 21,
               (0, 1): 2, (1, 1): -24, (2, 1): 42}),
        P(40, {(0, 0): -1, (1, 0): 9, (2, 0): -15, (3, 0): 7,
               (0, 1): 6, (1, 1): -48, (2, 1): 42, (0, 2): -6, (1, 2): 42}),
        P(56, {(0, 0): -1, (1, 0): 3, (2, 0): -3, (3, 0): 1,
               (0, 1): 12, (1, 1): -24, (2, 1): 12,
               (0, 2): -30, (1, 2): 30, (0, 3): 20}),
    ]


def _inner_rational(p: RootPoly, q: RootPoly) -> Fraction:
    """<p, q> when the result is rational (p, q share a radicand class)."""
    r, m = (p * q).integral()
    if r != 0 and m != 1:
        raise ArithmeticError("inner product is irrational")
    return r


def _gram_schmidt_degree(lower: list[RootPoly], degree: int) -> list[RootPoly]:
    """Exact orthonormal completion of P_degree against ``lower``."""
    new: list[RootPoly] = []
    for b in range(degree + 1):
        a = degree - b
        resid = {(a, b): Fraction(1)}
        mono = RootPoly.make(1, resid)
        for f in lower + new:
            # <mono, f> f = (r sqrt(m)) (sqrt(m) P) = r m P: rational
            r, m = (mono * f).integral()
            if r == 0:
                continue
            for key, c in f.coef:
                resid[key] = resid.get(key, 0) - r * m * c
        rp = RootPoly(1, tuple(sorted((k, v) for k, v in resid.items() if v != 0)))
        norm2 = _inner_rational(rp, rp)  # p/q
        num, den = norm2.numerator, norm2.denominator
        # rp / sqrt(num/den) = rp * sqrt(num*den) / num
        s, m = squarefree(num * den)
        new.append(RootPoly(m, tuple((k, v * s / num) for k, v in rp.coef)))
    return new


@lru_cache(maxsize=None)
def _modal(k: int) -> tuple[RootPoly, ...]:
    funcs = _paper_basis()
    if k >= 4:
        funcs = funcs + _gram_schmidt_degree(funcs, 4)
    return tuple(funcs[: K_FUNCS[k]])


@dataclass(frozen=True)
class Basis:
    """Orthonormal hierarchical modal basis of order k (reference RefBasis)."""

    order: int
    functions: tuple
    gradients: tuple

    @property
    def size(self) -> int:
        return len(self.functions)


@lru_cache(maxsize=None)
def build_basis(k: int) -> Basis:
    if k not in K_FUNCS:
        raise UnsupportedOrder(f"order {k} not supported (0..{MAX_ORDER})")
    funcs = _modal(k)
    grads = tuple((f.diff(1), f.diff(2)) for f in funcs)
    return Basis(order=k, functions=funcs, gradients=grads)
