"""Frozen reference-element tensors and the 1-D trace-space operators.

Two families of constants are produced here, both exact until the single
float conversion (``symbolic.exact_float``):

* the reference's own contraction tensors (``RefTensors``: M, S, T, G, E,
  EX, ET, ETX with the index conventions of reference tensors.py:8-16 and
  the construction of tensors.py:100-172).  For k <= 3 they are
  bit-identical to the reference; they feed parity tests and the dense
  ``RefTensors`` API.
* the operators the B200 kernels actually contract with (``TraceSpace``):
  Lambda[e, i, a] = int_0^1 phi_i|_e(s) psi_a(s) ds with psi_a the orthonormal
  Legendre polynomials on [0, 1], and J[a, b, c] = int psi_a psi_b psi_c.
  They replace the K x K (x K) edge tensors by (k+1)-sized ones:
  E[e] = Lambda_e Lambda_e^T, EX[e, f] = Lambda_e R Lambda_f^T with
  R = diag((-1)^a), ET/ETX likewise through J.

Quadrature rules mirror reference tensors.py:175-197 (collapsed
Gauss-Legendre on the triangle, Gauss-Legendre on [0, 1]).
"""

from __future__ import annotations

import csv
import math
from dataclasses import dataclass
from fractions import Fraction
from functools import lru_cache
from pathlib import Path

import numpy as np

from .symbolic import (
    EDGE_MAPS,
    K_FUNCS,
    RootPoly,
    UnsupportedOrder,
    build_basis,
    exact_float,
    monomial_integral,
    squarefree,
)

__all__ = [
    "RefTensors",
    "TraceSpace",
    "build_ref_tensors",
    "build_trace_space",
    "triangle_rule",
    "edge_rule",
    "legendre01",
    "LAMBDA_SAMPLES",
]

LAMBDA_SAMPLES = (0.0, 0.5, 1.0)


# ----------------------------------------------------------- exact helpers

def _mul_terms(p: dict, q: dict) -> dict:
    out: dict = {}
    for (a1, b1), c1 in p.items():
        for (a2, b2), c2 in q.items():
            key = (a1 + a2, b1 + b2)
            out[key] = out.get(key, 0) + c1 * c2
    return out


def _tri_integral(terms: dict) -> Fraction:
    return sum((c * monomial_integral(a, b) for (a, b), c in terms.items()), Fraction(0))


def _val(r: Fraction, rad: int) -> float:
    """exact r*sqrt(rad) (rad need not be square-free) to float64."""
    s, m = squarefree(rad)
    return exact_float(r * s, m)


def _mul1(p: dict, q: dict) -> dict:
    out: dict = {}
    for n1, c1 in p.items():
        for n2, c2 in q.items():
            out[n1 + n2] = out.get(n1 + n2, 0) + c1 * c2
    return out


def _int1(p: dict) -> Fraction:
    return sum((c / (n + 1) for n, c in p.items()), Fraction(0))


def _reverse1(p: dict) -> dict:
    """q(1-s) for q = sum c_n s^n."""
    out: dict = {}
    for n, c in p.items():
        for j in range(n + 1):
            v = c * math.comb(n, j) * (-1) ** j
            out[j] = out.get(j, 0) + v
    return {n: v for n, v in out.items() if v != 0}


def _shifted_legendre(n: int) -> dict:
    """Integer coefficients of P_n(2s-1) (psi_n = sqrt(2n+1) * this)."""
    return {j: Fraction((-1) ** (n + j) * math.comb(n, j) * math.comb(n + j, j))
            for j in range(n + 1)}


# ---------------------------------------------------------------- tensors

@dataclass(frozen=True)
class RefTensors:
    """Reference contraction tensors for one order (reference tensors.py:51-73)."""

    order: int
    M: np.ndarray
    S: np.ndarray
    T: np.ndarray
    G: np.ndarray
    E: np.ndarray
    EX: np.ndarray
    ET: np.ndarray
    ETX: np.ndarray

    @property
    def n_funcs(self) -> int:
        return self.M.shape[0]

    def as_dict(self) -> dict:
        return {"M": self.M, "S": self.S, "T": self.T, "G": self.G,
                "E": self.E, "EX": self.EX, "ET": self.ET, "ETX": self.ETX}


@lru_cache(maxsize=None)
def _volume_tensors(k: int):
    """M, S, T, G exactly (reference tensors.py:109-137)."""
    basis = build_basis(k)
    K = basis.size
    phi = basis.functions
    dphi = basis.gradients
    M = np.zeros((K, K))
    S = np.zeros((2, K, K))
    T = np.zeros((2, K, K, K))
    G = np.zeros((K, K, K))
    for p in range(K):
        for i in range(K):
            pi = _mul_terms(phi[p].terms, phi[i].terms)
            M[p, i] = _val(_tri_integral(pi), phi[p].rad * phi[i].rad)
    for l in range(2):
        for p in range(K):
            d = dphi[p][l]
            for i in range(K):
                di = _mul_terms(d.terms, phi[i].terms)
                S[l, p, i] = _val(_tri_integral(di), d.rad * phi[i].rad)
                for m in range(i, K):
                    v = _val(_tri_integral(_mul_terms(di, phi[m].terms)),
                             d.rad * phi[i].rad * phi[m].rad)
                    T[l, p, i, m] = v
                    T[l, p, m, i] = v
    for p in range(K):
        for i in range(p, K):
            pi = _mul_terms(phi[p].terms, phi[i].terms)
            for m in range(i, K):
                v = _val(_tri_integral(_mul_terms(pi, phi[m].terms)),
                         phi[p].rad * phi[i].rad * phi[m].rad)
                for a, b, c in ((p, i, m), (p, m, i), (i, p, m),
                                (i, m, p), (m, p, i), (m, i, p)):
                    G[a, b, c] = v
    return M, S, T, G


@lru_cache(maxsize=None)
def _traces(k: int):
    """Exact edge restrictions: traces[e][i] = (rad, {n: coef})."""
    basis = build_basis(k)
    return [[f.trace(e) for f in basis.functions] for e in range(3)]


@lru_cache(maxsize=None)
def build_ref_tensors(k: int) -> RefTensors:
    if k not in K_FUNCS:
        raise UnsupportedOrder(f"order {k} not supported")
    M, S, T, G = _volume_tensors(k)
    K = K_FUNCS[k]
    tr = _traces(k)
    trr = [[(rad, _reverse1(p)) for rad, p in row] for row in tr]
    E = np.zeros((3, K, K))
    ET = np.zeros((3, K, K, K))
    EX = np.zeros((3, 3, K, K))
    ETX = np.zeros((3, 3, K, K, K))
    for e in range(3):
        for p in range(K):
            rp, tp = tr[e][p]
            for i in range(K):
                ri, ti = tr[e][i]
                pi = _mul1(tp, ti)
                E[e, p, i] = _val(_int1(pi), rp * ri)
                for m in range(i, K):
                    rm, tm = tr[e][m]
                    v = _val(_int1(_mul1(pi, tm)), rp * ri * rm)
                    ET[e, p, i, m] = v
                    ET[e, p, m, i] = v
        for f in range(3):
            for p in range(K):
                rp, tp = tr[e][p]
                for i in range(K):
                    ri, ti = trr[f][i]
                    pi = _mul1(tp, ti)
                    EX[e, f, p, i] = _val(_int1(pi), rp * ri)
                    for m in range(i, K):
                        rm, tm = trr[f][m]
                        v = _val(_int1(_mul1(pi, tm)), rp * ri * rm)
                        ETX[e, f, p, i, m] = v
                        ETX[e, f, p, m, i] = v
    return RefTensors(order=k, M=M, S=S, T=T, G=G, E=E, EX=EX, ET=ET, ETX=ETX)


@dataclass(frozen=True)
class TraceSpace:
    """1-D trace-space operators of one order.

    Lam[e, i, a]   = int_0^1 phi_i|_e psi_a            (3, K, k+1)
    J[a, b, c]     = int_0^1 psi_a psi_b psi_c          (k+1)^3
    psi_at[a, s]   = psi_a(s) at LAMBDA_SAMPLES         (k+1, 3)
    """

    order: int
    Lam: np.ndarray
    J: np.ndarray
    psi_at: np.ndarray

    @property
    def n_trace(self) -> int:
        return self.J.shape[0]


@lru_cache(maxsize=None)
def build_trace_space(k: int) -> TraceSpace:
    if k not in K_FUNCS:
        raise UnsupportedOrder(f"order {k} not supported")
    K = K_FUNCS[k]
    NT = k + 1
    leg = [_shifted_legendre(a) for a in range(NT)]
    tr = _traces(k)
    Lam = np.zeros((3, K, NT))
    for e in range(3):
        for i in range(K):
            rad, t = tr[e][i]
            for a in range(NT):
                Lam[e, i, a] = _val(_int1(_mul1(t, leg[a])), rad * (2 * a + 1))
    J = np.zeros((NT, NT, NT))
    for a in range(NT):
        for b in range(NT):
            ab = _mul1(leg[a], leg[b])
            for c in range(NT):
                J[a, b, c] = _val(_int1(_mul1(ab, leg[c])),
                                  (2 * a + 1) * (2 * b + 1) * (2 * c + 1))
    psi_at = np.array([[float(legendre01(a, s)) for s in LAMBDA_SAMPLES] for a in range(NT)])
    return TraceSpace(order=k, Lam=Lam, J=J, psi_at=psi_at)


def legendre01(a: int, s):
    """Orthonormal Legendre psi_a on [0, 1], floating evaluation."""
    coeffs = _shifted_legendre(a)
    acc = 0.0
    for n, c in coeffs.items():
        acc = acc + float(c) * np.asarray(s, dtype=float) ** n
    return math.sqrt(2 * a + 1) * acc


# ------------------------------------------------------- quadrature rules

def triangle_rule(degree: int) -> tuple[np.ndarray, np.ndarray]:
    """Collapsed Gauss rule exact to ``degree`` (reference tensors.py:175-190)."""
    n = (degree + 3) // 2
    x, w = np.polynomial.legendre.leggauss(n)
    a = 0.5 * (x + 1.0)
    wa = 0.5 * w
    A, Bm = np.meshgrid(a, a, indexing="ij")
    WA, WB = np.meshgrid(wa, wa, indexing="ij")
    pts = np.column_stack([A.ravel(), (Bm * (1.0 - A)).ravel()])
    return pts, (WA * WB * (1.0 - A)).ravel()


def edge_rule(degree: int) -> tuple[np.ndarray, np.ndarray]:
    """Gauss-Legendre on [0, 1] exact to ``degree`` (reference tensors.py:193-197)."""
    x, w = np.polynomial.legendre.leggauss(degree // 2 + 1)
    return 0.5 * (x + 1.0), 0.5 * w


def edge_point(edge: int, s):
    """Reference coordinates of edge parameter s on local edge ``edge``."""
    x0, x1s, y0, y1s = EDGE_MAPS[edge]
    s = np.asarray(s, dtype=float)
    return x0 + x1s * s, y0 + y1s * s


# ------------------------------------------------- verification and dumps

@dataclass(frozen=True)
class TensorReport:
    """Deviation of the frozen tensors from quadrature (reference tensors.py:200-204)."""

    order: int
    max_abs_dev: float
    max_rel_dev: float


def verify_tensors(t: RefTensors) -> TensorReport:
    """Re-derive every tensor with degree-exact floating quadrature and report
    the largest deviation (reference tensors.py:207-254; relative deviations
    are scaled by the largest entry of each tensor)."""
    k = t.order
    basis = build_basis(k)
    K = basis.size
    pts, wts = triangle_rule(3 * k + 1)
    x1, x2 = pts[:, 0], pts[:, 1]
    vals = np.array([f.eval(x1, x2) for f in basis.functions])                     # [i, q]
    grads = np.array([[basis.gradients[i][l].eval(x1, x2) * np.ones_like(x1) for l in range(2)]
                      for i in range(K)])                                          # [i, l, q]
    sq, wq = edge_rule(3 * k)
    tr = np.array([[f.eval(*edge_point(e, sq)) * np.ones_like(sq) for f in basis.functions]
                   for e in range(3)])                                             # [e, i, q]
    trr = np.array([[f.eval(*edge_point(e, 1.0 - sq)) * np.ones_like(sq) for f in basis.functions]
                    for e in range(3)])
    quad = {
        "M": np.einsum("pq,iq,q->pi", vals, vals, wts),
        "S": np.einsum("plq,iq,q->lpi", grads, vals, wts),
        "T": np.einsum("plq,iq,mq,q->lpim", grads, vals, vals, wts),
        "G": np.einsum("pq,iq,mq,q->pim", vals, vals, vals, wts),
        "E": np.einsum("epq,eiq,q->epi", tr, tr, wq),
        "EX": np.einsum("epq,fiq,q->efpi", tr, trr, wq),
        "ET": np.einsum("epq,eiq,emq,q->epim", tr, tr, tr, wq),
        "ETX": np.einsum("epq,fiq,fmq,q->efpim", tr, trr, trr, wq),
    }
    max_abs = max_rel = 0.0
    for name, frozen in t.as_dict().items():
        dev = float(np.abs(frozen - quad[name]).max())
        max_abs = max(max_abs, dev)
        scale = float(np.abs(quad[name]).max())
        max_rel = max(max_rel, dev / scale if scale > 0.0 else dev)  # k = 0: S = T = 0
    return TensorReport(order=k, max_abs_dev=max_abs, max_rel_dev=max_rel)


_CSV_INDEX = {
    "M": ["p", "i"], "S": ["l", "p", "i"], "T": ["l", "p", "i", "m"], "G": ["p", "i", "m"],
    "E": ["e", "p", "i"], "EX": ["e", "eN", "p", "i"], "ET": ["e", "p", "i", "m"],
    "ETX": ["e", "eN", "p", "i", "m"],
}


def dump_tensors_csv(t: RefTensors, out_dir) -> list:
    """One CSV per tensor, ``<name>_k<order>.csv``, header = index names +
    ``value``, entries in C order with %.17g (reference tensors.py:257-275)."""
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    paths = []
    for name, arr in t.as_dict().items():
        path = out_dir / f"{name}_k{t.order}.csv"
        idx = np.indices(arr.shape).reshape(arr.ndim, -1).T
        with open(path, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(_CSV_INDEX[name] + ["value"])
            w.writerows([*map(int, row), f"{v:.17g}"] for row, v in zip(idx, arr.ravel()))
        paths.append(path)
    return paths


def load_tensors_csv(order: int, in_dir) -> RefTensors:
    """Inverse of dump_tensors_csv (shapes from the order)."""
    ref = build_ref_tensors(order)
    arrs = {}
    for name, arr in ref.as_dict().items():
        out = np.zeros(arr.shape)
        with open(Path(in_dir) / f"{name}_k{order}.csv", newline="") as fh:
            rd = csv.reader(fh)
            next(rd)
            for row in rd:
                out[tuple(int(v) for v in row[:-1])] = float(row[-1])
        arrs[name] = out
    return RefTensors(order=order, **arrs)
