"""Literal-constant CUDA generation for the per-order element operators.

The paper's thesis (reference codegen.py:219-398) is to
unroll every reference-tensor contraction into straight-line code with the
tensor entries as literals and the zero entries dropped.  This module does
the same for the B200 kernels, emitting one header per order k,
``csrc/generated/qf_order{k}.cuh``, that defines ``qf::Ord<k>`` with:

  vel_matrix  A[p<=m] = sum_i H_i G[p,i,m]           (packed, column-major)
  vol_xi      r = S1 alpha + S2 beta                    (xi row, Eq. 15)
  vol_uv      factorised stiffness-triple rows          (U/V rows, Eq. 16)
  trace<J>    t_a = sum_i Lambda_J[i,a] f_i             (1-D trace moments)
  lift<J>     r_p -= s sum_a Lambda_J[p,a] F_a
  jprod       (x*y)_a = sum J[a,b,c] x_b y_c            (trace products)
  samples     trace values at s = 0, 1/2, 1             (lambda samples)
  quad_project / gauss_moments  forcing and Dirichlet-data quadrature
  hb_dref     reference gradient of the P1 bathymetry

Constants come from the exact tensors (``tensors.py``); output is
deterministic byte-for-byte so the build is reproducible.
"""

from __future__ import annotations

import math
from pathlib import Path

import numpy as np

from .symbolic import K_FUNCS, MAX_ORDER, build_basis
from .tensors import (LAMBDA_SAMPLES, build_ref_tensors, build_trace_space, edge_rule,
                      legendre01, triangle_rule)

GEN_DIR = Path(__file__).resolve().parent / "csrc" / "generated"
TOL = 1e-15
# orders whose (input-outer, split) volume kernel takes the pressure rows from
# vol_press instead of the y_l = T_l w contraction (measured: k = 4 faster,
# k = 3 row-outer slower)
PRESS_MINK = 4
QF_LITERAL_ORDERS = tuple(int(x) for x in __import__("os").environ.get("QF_LITERAL_ORDERS", "3").split(",") if x)


def lit(v: float) -> str:
    s = repr(float(v))
    if "e" not in s and "." not in s and "inf" not in s and "nan" not in s:
        s += ".0"
    return s


# Constant pool of the order being generated.  Coefficients are emitted as
# references P{k}[i] into a __constant__ array with compile-time indices, so
# ptxas feeds them to DFMA/DMUL as constant-bank operands (c[0x3][...])
# instead of materialising each 64-bit literal with two UMOV/IMAD.MOV.
_POOL: dict | None = None
_POOL_NAME = "P"


def coef(v: float) -> str:
    """Pool reference for |v| (callers handle the sign)."""
    v = abs(float(v))
    if _POOL is None:
        return lit(v)
    if v not in _POOL:
        _POOL[v] = len(_POOL)
    return f"{_POOL_NAME}[{_POOL[v]}]"


def scoef(v: float) -> str:
    """Signed pool reference."""
    return coef(v) if v >= 0 else f"-{coef(v)}"


def _sum(terms: list[tuple[float, str]]) -> str:
    """Linear combination with pooled coefficients; +-1 folded."""
    if not terms:
        return "0.0"
    out = []
    for i, (c, x) in enumerate(terms):
        if c == 1.0:
            t = x
            sign = "+"
        elif c == -1.0:
            t = x
            sign = "-"
        elif c < 0:
            t = f"{coef(c)} * {x}"
            sign = "-"
        else:
            t = f"{coef(c)} * {x}"
            sign = "+"
        if i == 0:
            out.append(t if sign == "+" else f"-{t}")
        else:
            out.append(f" {sign} {t}")
    return "".join(out)


def _nz(a) -> bool:
    return abs(a) > TOL


def _gen_press(w, rt, K, NH):
    """vol_press<P0, P1>: pressure rows from symmetric products (see gen_order)."""
    w("  template <int P0 = 0, int P1 = K, class RT> static __device__ __forceinline__ void"
      " vol_press(const double* xi, const double* hb, bool hbl, double g22, double g21,"
      " double g12, double g11, RT rU, RT rV) {")
    w("    constexpr unsigned R = (1u << P1) - (1u << P0);")
    w("    double p1[K], p2[K];")
    w("    #pragma unroll\n    for (int p = 0; p < K; ++p) { p1[p] = 0.0; p2[p] = 0.0; }")

    def _press_block(pairs, xa, xb, half_diag):
        for (i, m) in pairs:
            ent = []
            for p in range(K):
                f = 0.5 if (half_diag and i == m) else 1.0
                c1, c2 = f * rt.T[0, p, i, m], f * rt.T[1, p, i, m]
                if _nz(c1) or _nz(c2):
                    ent.append((p, c1, c2))
            if not ent:
                continue
            mask = sum(1 << p for p, _, _ in ent)
            w(f"    if constexpr (({mask}u & R) != 0u) {{ const double q = {xa}[{i}] * {xb}[{m}];")
            for p, c1, c2 in ent:
                st = []
                if _nz(c1):
                    st.append(f"p1[{p}] = fma({scoef(c1)}, q, p1[{p}]);")
                if _nz(c2):
                    st.append(f"p2[{p}] = fma({scoef(c2)}, q, p2[{p}]);")
                w(f"      if constexpr (P0 <= {p} && {p} < P1) {{ {' '.join(st)} }}")
            w("    }")

    _press_block([(i, m) for i in range(K) for m in range(i, K)], "xi", "xi", True)
    w("    if (hbl) {")
    _press_block([(i, m) for i in range(K) for m in range(NH)], "xi", "hb", False)
    w("    }")
    for p in range(K):
        w(f"    if constexpr (P0 <= {p} && {p} < P1) {{ rU[{p}] = fma(g22, p1[{p}], fma(-g21, p2[{p}], rU[{p}]));"
          f" rV[{p}] = fma(g11, p2[{p}], fma(-g12, p1[{p}], rV[{p}])); }}")
    w("  }")


def gen_order(k: int) -> str:
    K = K_FUNCS[k]
    NT = k + 1
    NH = 1 if k == 0 else 3
    rt = build_ref_tensors(k)
    ts = build_trace_space(k)
    basis = build_basis(k)
    qp, qw = triangle_rule(2 * k + 2)
    NQ = len(qw)
    gs, gw = edge_rule(2 * (k + 2) - 1)
    NG = len(gw)
    phi_q = np.array([[f.eval(x, y) for (x, y) in qp] for f in basis.functions])  # (K, NQ)
    global _POOL, _POOL_NAME
    # measured per order (round 1): pooled constants win for k = 0, 1, 2, 4;
    # for k = 3 literals give ptxas a better register allocation
    _POOL, _POOL_NAME = ({} if k not in QF_LITERAL_ORDERS else None), f"qf_pool{k}"
    L = []
    w = L.append
    w(f"template <> struct Ord<{k}> {{")
    w(f"  static constexpr int K = {K}, NT = {NT}, NH = {NH}, NQ = {NQ}, NG = {NG};")
    # ---- velocity matrix
    w("  static __device__ __forceinline__ void vel_matrix(const double* __restrict__ H, double* __restrict__ A) {")
    for m in range(K):
        for p in range(m + 1):
            terms = [(rt.G[p, i, m], f"H[{i}]") for i in range(K) if _nz(rt.G[p, i, m])]
            w(f"    A[{m * (m + 1) // 2 + p}] = {_sum(terms)};")
    w("  }")
    # ---- LDL^T velocity solve in scalar registers (no local arrays)
    # (qU, qV: register arrays, or strided row views read where the forward
    # substitution first needs them)
    w("  template <class Q>")
    w("  static __device__ __forceinline__ bool vel_solve(const double* __restrict__ H,"
      " const Q& qU, const Q& qV, double sd, double* uo, double* vo) {")
    for m in range(K):
        for p in range(m + 1):
            terms = [(rt.G[p, i, m], f"H[{i}]") for i in range(K) if _nz(rt.G[p, i, m])]
            w(f"    double a{p}_{m} = {_sum(terms)};")
    w("    bool ok = true;")
    for j in range(K):
        w(f"    ok = ok && (a{j}_{j} != 0.0) && isfinite(a{j}_{j}); const double d{j} = 1.0 / a{j}_{j};")
        for i in range(j + 1, K):
            w(f"    const double l{i}_{j} = a{j}_{i} * d{j};")
            for m in range(i, K):
                w(f"    a{i}_{m} = fma(-l{i}_{j}, a{j}_{m}, a{i}_{m});")
    for i in range(K):
        tu = " ".join(f"yu{i} = fma(-l{i}_{j}, yu{j}, yu{i}); yv{i} = fma(-l{i}_{j}, yv{j}, yv{i});"
                      for j in range(i))
        w(f"    double yu{i} = qU[{i}], yv{i} = qV[{i}]; {tu}")
    for i in range(K - 1, -1, -1):
        w(f"    yu{i} *= d{i}; yv{i} *= d{i};")
        for m in range(i + 1, K):
            w(f"    yu{i} = fma(-l{m}_{i}, yu{m}, yu{i}); yv{i} = fma(-l{m}_{i}, yv{m}, yv{i});")
        w(f"    uo[{i}] = sd * yu{i}; vo[{i}] = sd * yv{i}; ok = ok && isfinite(yu{i}) && isfinite(yv{i});")
    w("    return ok;")
    w("  }")
    # ---- xi row
    w("  template <class RT> static __device__ __forceinline__ void vol_xi(const double* al, const double* be, RT r) {")
    for p in range(K):
        terms = [(rt.S[0, p, i], f"al[{i}]") for i in range(K) if _nz(rt.S[0, p, i])]
        terms += [(rt.S[1, p, i], f"be[{i}]") for i in range(K) if _nz(rt.S[1, p, i])]
        w(f"    r[{p}] = {_sum(terms)};")
    w("  }")
    # ---- U/V rows
    w("  template <class RT, class CT> static __device__ __forceinline__ void vol_uv(CT cU, CT cV,"
      " CT xi, const double* a, const double* b, const double* wv,")
    w("      double g22, double g21, double g12, double g11, RT rU, RT rV) {")
    for p in range(K):
        w(f"    {{ double su = 0.0, sv = 0.0;")
        for i in range(K):
            zt = [(rt.T[0, p, i, m], f"a[{m}]") for m in range(K) if _nz(rt.T[0, p, i, m])]
            zt += [(rt.T[1, p, i, m], f"b[{m}]") for m in range(K) if _nz(rt.T[1, p, i, m])]
            y1 = [(rt.T[0, p, i, m], f"wv[{m}]") for m in range(K) if _nz(rt.T[0, p, i, m])]
            y2 = [(rt.T[1, p, i, m], f"wv[{m}]") for m in range(K) if _nz(rt.T[1, p, i, m])]
            if not (zt or y1 or y2):
                continue
            w("      {")
            if zt:
                w(f"        const double z = {_sum(zt)};")
                w(f"        su = fma(z, cU[{i}], su); sv = fma(z, cV[{i}], sv);")
            if y1 and y2:
                w(f"        const double y1 = {_sum(y1)}, y2 = {_sum(y2)};")
                w(f"        su = fma(xi[{i}], fma(g22, y1, -g21 * y2), su);")
                w(f"        sv = fma(xi[{i}], fma(g11, y2, -g12 * y1), sv);")
            elif y1:
                w(f"        const double y1 = {_sum(y1)};")
                w(f"        su = fma(xi[{i}] * g22, y1, su); sv = fma(-xi[{i}] * g12, y1, sv);")
            elif y2:
                w(f"        const double y2 = {_sum(y2)};")
                w(f"        su = fma(-xi[{i}] * g21, y2, su); sv = fma(xi[{i}] * g11, y2, sv);")
            w("      }")
        w(f"      rU[{p}] = su; rV[{p}] = sv; }}")
    w("  }")
    # ---- U/V rows, input-outer order (volume_kernel, k >= 3): only a, b, wv
    # and the accumulators stay live; cU_i, cV_i, xi_i are fetched once each
    # (the caller pre-scales them by 1/(detB sqrt(detB)) through its view).
    # outputs [P0, P1) only (the volume kernel splits the output rows across
    # launches to bound the live accumulators); an input block is emitted only
    # if one of its outputs is in range (mask), so no dead loads remain
    def _has(i, p):
        return any(_nz(rt.T[l, p, i, m]) for l in range(2) for m in range(K))
    masks = [sum(1 << p for p in range(K) if _has(i, p)) for i in range(K)]
    cnt = [sum(2 * sum(_nz(rt.T[l, p, i, m]) for l in range(2) for m in range(K)) for i in range(K))
           for p in range(K)]
    for G in (2, 3, 4):  # output split points balanced by term count
        tot, acc, cuts = sum(cnt), 0, [0]
        for p in range(K):
            acc += cnt[p]
            if len(cuts) < G and acc >= tot * len(cuts) / G:
                cuts.append(p + 1)
        cuts += [K] * (G + 1 - len(cuts))
        w(f"  static constexpr int VOL_PSPLIT{G}[{G + 1}] = {{{', '.join(map(str, cuts))}}};")
    w("  template <int P0 = 0, int P1 = K, bool PRESS = true, class RT, class CT> static __device__"
      " __forceinline__ void vol_uv_acc(CT cU, CT cV, CT xi, const double* a, const double* b,"
      " const double* wv,")
    w("      double g22, double g21, double g12, double g11, RT rU, RT rV) {")
    w("    constexpr unsigned R = (1u << P1) - (1u << P0);")
    for i in range(K):
        w(f"    if constexpr (({masks[i]}u & R) != 0u) {{ const double ci = cU[{i}], vi = cV[{i}], xq = xi[{i}];")
        for p in range(K):
            zt = [(rt.T[0, p, i, m], f"a[{m}]") for m in range(K) if _nz(rt.T[0, p, i, m])]
            zt += [(rt.T[1, p, i, m], f"b[{m}]") for m in range(K) if _nz(rt.T[1, p, i, m])]
            y1 = [(rt.T[0, p, i, m], f"wv[{m}]") for m in range(K) if _nz(rt.T[0, p, i, m])]
            y2 = [(rt.T[1, p, i, m], f"wv[{m}]") for m in range(K) if _nz(rt.T[1, p, i, m])]
            if not (zt or y1 or y2):
                continue
            w(f"      if constexpr (P0 <= {p} && {p} < P1) {{")
            if zt:
                w(f"        const double z = {_sum(zt)};")
                w(f"        rU[{p}] = fma(z, ci, rU[{p}]); rV[{p}] = fma(z, vi, rV[{p}]);")
            if (y1 or y2) and k >= PRESS_MINK:
                w("        if constexpr (PRESS) {")
            if y1 and y2:
                w(f"        const double y1 = {_sum(y1)}, y2 = {_sum(y2)};")
                w(f"        rU[{p}] = fma(xq, fma(g22, y1, -g21 * y2), rU[{p}]);")
                w(f"        rV[{p}] = fma(xq, fma(g11, y2, -g12 * y1), rV[{p}]);")
            elif y1:
                w(f"        const double y1 = {_sum(y1)};")
                w(f"        rU[{p}] = fma(xq * g22, y1, rU[{p}]); rV[{p}] = fma(-xq * g12, y1, rV[{p}]);")
            elif y2:
                w(f"        const double y2 = {_sum(y2)};")
                w(f"        rU[{p}] = fma(-xq * g21, y2, rU[{p}]); rV[{p}] = fma(xq * g11, y2, rV[{p}]);")
            if (y1 or y2) and k >= PRESS_MINK:
                w("        }")
            w("      }")
        w("    }")
    w("  }")
    # ---- pressure rows from the symmetric products (k >= 3 volume): with
    # T_l[p, i, m] symmetric in (i, m),
    #   pi_l[p] = T_l : (xi (x) (xi / 2 + hb))
    #           = sum_{i<m} T_l[p,i,m] xi_i xi_m + 1/2 sum_i T_l[p,i,i] xi_i^2
    #             + sum_{i, m<NH} T_l[p,i,m] xi_i hb_m
    # (about half the multiply-adds of the y_l = T_l w contraction), then
    # U_p += g22 pi_1 - g21 pi_2, V_p += g11 pi_2 - g12 pi_1 (rows [P0, P1))
    # (generated for the orders whose volume kernel uses it only, so the
    # other orders' constant pools and register allocation are unchanged)
    if k >= min(PRESS_MINK, MMA_MINK):
        _gen_press(w, rt, K, NH)
    # ---- traces and lifts
    for j in range(3):
        # explicit fma chains: the same trace is evaluated by the element's own
        # thread and by a neighbour's thread; pinning the rounding sequence
        # keeps both bit-identical whatever the surrounding code (no
        # context-dependent contraction / CSE)
        w(f"  static __device__ __forceinline__ void trace{j}(const double* f, double* t) {{")
        for a in range(NT):
            terms = [(ts.Lam[j, i, a], i) for i in range(K) if _nz(ts.Lam[j, i, a])]
            if not terms:
                w(f"    t[{a}] = 0.0;")
                continue
            c0, i0 = terms[0]
            expr = f"__dmul_rn({scoef(c0)}, f[{i0}])"
            for c, i in terms[1:]:
                expr = f"__fma_rn({scoef(c)}, f[{i}], {expr})"
            w(f"    t[{a}] = {expr};")
        w("  }")
        w(f"  template <class RT> static __device__ __forceinline__ void lift{j}(const double* F, double s, RT r) {{")
        for p in range(K):
            terms = [(ts.Lam[j, p, a], f"F[{a}]") for a in range(NT) if _nz(ts.Lam[j, p, a])]
            if terms:
                w(f"    r[{p}] = fma(-s, {_sum(terms)}, r[{p}]);")
        w("  }")
    w("  template <int J> static __device__ __forceinline__ void trace(const double* f, double* t) {")
    w("    if (J == 0) trace0(f, t); else if (J == 1) trace1(f, t); else trace2(f, t);")
    w("  }")
    w("  template <int J, class RT> static __device__ __forceinline__ void lift(const double* F, double s, RT r) {")
    w("    if (J == 0) lift0(F, s, r); else if (J == 1) lift1(F, s, r); else lift2(F, s, r);")
    w("  }")
    w("  static __device__ __forceinline__ void trace_dyn(int j, const double* f, double* t) {")
    w("    if (j == 0) trace0(f, t); else if (j == 1) trace1(f, t); else trace2(f, t);")
    w("  }")
    # ---- J products
    w("  static __device__ __forceinline__ void jprod(const double* x, const double* y, double* o) {")
    for a in range(NT):
        terms = []
        for b in range(NT):
            for c in range(b, NT):
                v = ts.J[a, b, c]
                if not _nz(v):
                    continue
                if b == c:
                    terms.append((v, f"x[{b}] * y[{c}]"))
                else:
                    terms.append((v, f"(x[{b}] * y[{c}] + x[{c}] * y[{b}])"))
        w(f"    o[{a}] = {_sum(terms)};")
    w("  }")
    # ---- samples
    w("  static __device__ __forceinline__ void samples(const double* t, double* v) {")
    for si, s in enumerate(LAMBDA_SAMPLES):
        terms = [(float(legendre01(a, s)), f"t[{a}]") for a in range(NT) if _nz(float(legendre01(a, s)))]
        w(f"    v[{si}] = {_sum(terms)};")
    w("  }")
    # ---- bathymetry reference gradient (P1 part)
    w("  static __device__ __forceinline__ void hb_dref(const double* hb, double& d1, double& d2) {")
    if NH == 3:
        g1 = [float(basis.gradients[i][0].eval(0.0, 0.0)) for i in range(3)]
        g2 = [float(basis.gradients[i][1].eval(0.0, 0.0)) for i in range(3)]
        w(f"    d1 = {_sum([(g1[i], f'hb[{i}]') for i in range(3) if _nz(g1[i])])};")
        w(f"    d2 = {_sum([(g2[i], f'hb[{i}]') for i in range(3) if _nz(g2[i])])};")
    else:
        w("    (void)hb; d1 = 0.0; d2 = 0.0;")
    w("  }")
    # ---- forcing quadrature: fn(x1, x2, f0, f1, f2) then r_f[p] += P[p][q] * f
    w("  template <class Fn> static __device__ __forceinline__ void quad_project(Fn&& fn,"
      " double* r0, double* r1, double* r2) {")
    for q in range(NQ):
        w(f"    {{ double f0, f1, f2; fn({lit(qp[q, 0])}, {lit(qp[q, 1])}, f0, f1, f2);")
        for p in range(K):
            c = phi_q[p, q] * qw[q]
            if _nz(c):
                w(f"      r0[{p}] = fma({lit(c)}, f0, r0[{p}]); r1[{p}] = fma({lit(c)}, f1, r1[{p}]);"
                  f" r2[{p}] = fma({lit(c)}, f2, r2[{p}]);")
        w("    }")
    w("  }")
    # ---- Dirichlet ghost moments: fn(s, vals[5]) at Gauss points
    w("  template <class Fn> static __device__ __forceinline__ void gauss_moments(Fn&& fn, double* mom) {")
    w(f"    #pragma unroll\n    for (int i = 0; i < 5 * NT; ++i) mom[i] = 0.0;")
    for gi in range(NG):
        w(f"    {{ double v[5]; fn({lit(gs[gi])}, v);")
        for a in range(NT):
            c = float(legendre01(a, gs[gi])) * gw[gi]
            w(f"      for (int f = 0; f < 5; ++f) mom[f * NT + {a}] = fma({lit(c)}, v[f], mom[f * NT + {a}]);")
        w("    }")
    w("  }")
    w("};")
    pool = sorted((_POOL or {}).items(), key=lambda kv: kv[1])
    _POOL = None
    head = [f"// Generated by paper_1904_08684_b200/codegen.py for order k={k}. Do not edit.",
            "#pragma once", "namespace qf {",
            f"__constant__ double qf_pool{k}[{max(len(pool), 1)}] = {{"]
    vals = [lit(v) for v, _ in pool] or ["0.0"]
    for i0 in range(0, len(vals), 4):
        head.append("  " + ", ".join(vals[i0:i0 + 4]) + ",")
    head.append("};")
    L[:0] = head
    # ---- tables for the looped (non-unrolled) edge and quadrature code:
    # Lam[3][K][NT] | QX[NQ] | QY[NQ] | P[NQ][K] (P = w_q phi_p(q)) | GS[NG] |
    # GPSI[NT][NG] (psi_a(s_g) w_g, Dirichlet ghost moments) | PHI[NQ][K] (phi_p(q)) |
    # QW[NQ] (w_q, error quadrature) | QR1, QR2[NQ] (quadrature points minus the centroid)
    gpsi = np.array([[float(legendre01(a, gs[g])) * gw[g] for g in range(NG)] for a in range(NT)])
    # (entries the literal trace code skips are zeroed, so a table-driven
    # trace reproduces its bits)
    lam_t = np.where(np.abs(ts.Lam) > TOL, ts.Lam, 0.0)
    tab = list(lam_t.ravel()) + list(qp[:, 0]) + list(qp[:, 1]) + \
        list((phi_q * qw[None, :]).T.ravel()) + list(gs) + list(gpsi.ravel()) + \
        list(phi_q.T.ravel()) + list(qw) + list(qp[:, 0] - 1.0 / 3.0) + list(qp[:, 1] - 1.0 / 3.0)
    w(f"__constant__ double c_tab{k}[{len(tab)}] = {{")
    for i0 in range(0, len(tab), 4):
        w("  " + ", ".join(lit(v) for v in tab[i0:i0 + 4]) + ",")
    w("};")
    w(f"template <> struct Tabs<{k}> {{")
    o_p = 3 * K * NT + 2 * NQ
    o_gs = o_p + NQ * K
    w(f"  static constexpr int L = 0, QX = {3 * K * NT}, QY = {3 * K * NT + NQ}, P = {o_p}, "
      f"GS = {o_gs}, GPSI = {o_gs + NG}, PHI = {o_gs + NG + NT * NG}, "
      f"QW = {o_gs + NG + NT * NG + NQ * K}, QR1 = {o_gs + NG + NT * NG + NQ * K + NQ}, "
      f"QR2 = {o_gs + NG + NT * NG + NQ * K + 2 * NQ}, SIZE = {len(tab)};")
    w(f"  static __device__ __forceinline__ const double* ptr() {{ return c_tab{k}; }}")
    w("};")
    if k >= MMA_MINK:
        L.extend(_gen_mma(k, rt, K))
    w("}  // namespace qf")
    return "\n".join(L) + "\n"


# orders whose volume advection Z[p,i] = sum_m T1[p,i,m] a_m + T2[p,i,m] b_m
# runs on the FP64 tensor cores (mma.sync.m8n8k4.f64, vol_mma_kernel)
MMA_MINK = 3
MMA_PREFETCH = int(__import__("os").environ.get("QF_MMA_PREFETCH", "4"))


def mma_layout(k: int, rt=None):
    """Fragment plan of the FP64-MMA volume advection for order k.

    GEMM per element tile of 8: D[el, n] = sum_kk A[el, kk] B[kk, n] with
    A[el, kk] = (a; b)_kk of element el (kk = l K + m, l = 0: a_m, 1: b_m),
    B[kk, n] = T[l, p, 8 ch + n, m] for output row p and input chunk ch, so
    D[el, n] = Z_el[p, 8 ch + n].  Returns (NKS, frags) with frags a list of
    (p, ch, s, values[32]) -- the m8n8k4 B fragment of k-step s, lane-major
    (lane holds B[lane % 4][lane // 4]) -- all-zero fragments dropped."""
    rt = rt or build_ref_tensors(k)
    T = rt.T
    K = T.shape[1]
    nks = (2 * K + 3) // 4
    nch = (K + 7) // 8
    frags = []
    for p in range(K):
        for ch in range(nch):
            for s in range(nks):
                vals = []
                for lane in range(32):
                    kk, i = 4 * s + lane % 4, 8 * ch + lane // 4
                    v = float(T[kk // K, p, i, kk % K]) if (kk < 2 * K and i < K) else 0.0
                    vals.append(v if _nz(v) else 0.0)
                if any(v != 0.0 for v in vals):
                    frags.append((p, ch, s, vals))
    return nks, frags


def _gen_mma(k: int, rt, K: int) -> list:
    nks, frags = mma_layout(k, rt)
    nch = (K + 7) // 8
    L = [f"// FP64 tensor-core volume advection, order {k}: {len(frags)} nonzero m8n8k4 B fragments",
         f"// (of {K * nch * nks}), {nks} k-steps over (a; b), {nch} input chunks of 8 (codegen.mma_layout)",
         f"__device__ const double qf_vmma{k}[{len(frags) * 32}] = {{"]
    for (_, _, _, vals) in frags:
        for i0 in range(0, 32, 4):
            L.append("  " + ", ".join(lit(v) for v in vals[i0:i0 + 4]) + ",")
    L.append("};")
    L.append(f"template <> struct Mma<{k}> {{")
    L.append(f"  static constexpr int K = {K}, NKS = {nks}, NCH = {nch}, NF = {len(frags)};")
    L.append(f"  static __device__ __forceinline__ const double* table() {{ return qf_vmma{k}; }}")
    L.append("  // pu[t][p] += sum_i Z_t[p,i] cu[t][i-slot] (likewise pv): sB = the fragment table in")
    L.append("  // shared memory, A[t][s] = this lane's (a; b) entry of k-step s for tile t,")
    L.append("  // cu/cv[t][2 ch + j] = c_U/c_V of input 8 ch + 2 (lane % 4) + j of the lane's element")
    L.append("  template <int NT> static __device__ __forceinline__ void adv(const double* sB, int lane,")
    L.append("      const double (&A)[NT][NKS], const double (&cu)[NT][2 * NCH], const double (&cv)[NT][2 * NCH],")
    L.append("      double (&pu)[NT][K], double (&pv)[NT][K]) {")
    # flat fragment order; the B fragment of step j + MMA_PREFETCH is loaded
    # while step j multiplies (volatile shared loads and MMAs keep this
    # order, so ptxas cannot hoist all NF loads and spill)
    seq = [(f, p, ch, s_) for f, (p, ch, s_, _) in enumerate(frags)]
    D = MMA_PREFETCH
    L.append(f"    double bq[{D}];")
    for j in range(min(D, len(seq))):
        L.append(f"    bq[{j}] = lds64(sB + {seq[j][0] * 32} + lane);")
    L.append("    double d0[NT], d1[NT];")
    for j, (f, p, ch, s_) in enumerate(seq):
        first = j == 0 or (seq[j - 1][1], seq[j - 1][2]) != (p, ch)
        last = j + 1 == len(seq) or (seq[j + 1][1], seq[j + 1][2]) != (p, ch)
        if first:
            L.append("    #pragma unroll")
            L.append("    for (int t = 0; t < NT; ++t) { d0[t] = 0.0; d1[t] = 0.0; }")
        L.append(f"    {{ const double b = bq[{j % D}];")
        if j + D < len(seq):
            L.append(f"      bq[{j % D}] = lds64(sB + {seq[j + D][0] * 32} + lane);")
        L.append("      #pragma unroll")
        L.append(f"      for (int t = 0; t < NT; ++t) dmma(d0[t], d1[t], A[t][{s_}], b); }}")
        if last:
            L.append("    #pragma unroll")
            L.append(f"    for (int t = 0; t < NT; ++t) {{ pu[t][{p}] = fma(d1[t], cu[t][{2 * ch + 1}], fma(d0[t], cu[t][{2 * ch}], pu[t][{p}]));"
                     f" pv[t][{p}] = fma(d1[t], cv[t][{2 * ch + 1}], fma(d0[t], cv[t][{2 * ch}], pv[t][{p}])); }}")
    L.append("  }")
    L.append("};")
    return L


def generate(out_dir: Path = GEN_DIR, orders=range(MAX_ORDER + 1)) -> list[Path]:
    out_dir.mkdir(parents=True, exist_ok=True)
    paths = []
    for k in orders:
        p = out_dir / f"qf_order{k}.cuh"
        src = gen_order(k)
        if not p.exists() or p.read_text() != src:
            p.write_text(src)
        paths.append(p)
    return paths


def term_counts(k: int) -> dict:
    """Multiply-add counts of the generated operators (for DESIGN.md / roofline)."""
    src = gen_order(k)
    return {"lines": src.count("\n"), "literals": src.count("fma(") + src.count(" * ")}


if __name__ == "__main__":
    for p in generate():
        print(p, p.stat().st_size)
