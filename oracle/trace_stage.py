"""CPU ORACLE (test infrastructure only): the B200 kernel algorithm in NumPy.

``qfswe_oracle`` restates the reference's dense formulation; this module
restates the *reformulated* algorithm the sm_100a kernels implement, on the
same structure-of-arrays tables (``paper_1904_08684_b200.layout``):

* velocity: A = sum_i H_i G[:, i, :], Cholesky-free LDL^T-equivalent dense
  solve, u = sqrt(detB) A^-1 q (reference solver.py:315-336);
* volume: factorised stiffness-triple contraction
  Z[p,i] = sum_m T1[p,i,m] a_m + T2[p,i,m] b_m;
* edges: owner-computes Lax-Friedrichs flux in 1-D trace space (Lambda, J),
  lambda from sample values of the trace moments;
* Dirichlet ghosts as Gauss moments of the exact data, walls as mirrors.

It exists to (1) check the reformulation against the dense oracle on the
CPU, and (2) drive the multi-rank halo logic under ``gloo`` in the CPU test
suite, where no GPU is available.  It is never part of the product path.
"""

from __future__ import annotations

import math

import numpy as np

from . import qfswe_oracle as O

SAMPLES = np.array([0.0, 0.5, 1.0])


def legendre01(a, s):
    c = np.zeros(a + 1)
    c[a] = 1.0
    return math.sqrt(2 * a + 1) * np.polynomial.legendre.legval(2 * np.asarray(s) - 1, c)


class TraceOps:
    """Trace-space operators by quadrature (independent of the product's exact ones)."""

    def __init__(self, k):
        self.k, self.NT = k, k + 1
        b = O.Basis(k)
        self.K = b.K
        s, w = O.gauss_line(k + 3)
        psi = np.array([legendre01(a, s) for a in range(self.NT)])     # (NT, Q)
        self.Lam = np.array([np.einsum("iq,aq,q->ia", b.trace(e, s), psi, w) for e in range(3)])
        self.J = np.einsum("aq,bq,cq,q->abc", psi, psi, psi, w)
        self.psi_s = np.array([legendre01(a, SAMPLES) for a in range(self.NT)])  # (NT, 3)
        self.R = (-1.0) ** np.arange(self.NT)
        t = O.build_tensors(k)
        self.S, self.T, self.G = t.S, t.T, t.G
        n = (2 * k + 2 + 3) // 2
        qx, qy, qw = O.gauss_triangle(n)
        self.qref = np.column_stack([qx, qy])
        self.qproj = b.eval(qx, qy) * qw                               # (K, Q)
        sg, wg = O.gauss_line(k + 2)
        self.gs, self.gw = sg, wg
        self.gpsi = np.array([legendre01(a, sg) for a in range(self.NT)]) * wg  # (NT, NG)


def jprod(J, x, y):
    return np.einsum("abc,b...,c...->a...", J, x, y)


class TraceStage:
    """One RHS / RK stage on SoA tables for elements [0, n_own)."""

    def __init__(self, k, geo, nbr, hb, n_own, scn, bnd_elem=None, bnd_local=None):
        self.ht = np.zeros((0, 6, k + 1))  # halo trace rows of the current stage input
        self.ops = TraceOps(k)
        self.k = k
        self.geo, self.nbr, self.hb, self.n = geo, nbr, hb, n_own
        self.scn = scn
        self.bnd_elem = bnd_elem if bnd_elem is not None else np.zeros(0, np.int64)
        self.bnd_local = bnd_local if bnd_local is not None else np.zeros(0, np.int64)

    # geometry of elements idx
    def _geom(self, idx):
        B11, B12, B21, B22 = (self.geo[r, idx] for r in range(4))
        det = B11 * B22 - B12 * B21
        return B11, B12, B21, B22, det, np.sqrt(det)

    def _hbfull(self, idx):
        K = self.ops.K
        h = np.zeros((K, len(idx)))
        h[: self.hb.shape[0]] = self.hb[:, idx]
        return h

    def velocity(self, c, idx=None):
        idx = np.arange(self.n) if idx is None else idx
        H = self._hbfull(idx) + c[0][:, idx]
        A = np.einsum("ie,pim->epm", H, self.ops.G)
        q = np.stack([c[1][:, idx], c[2][:, idx]], axis=2).transpose(1, 0, 2)  # (e,K,2)
        sol = np.linalg.solve(A, q.transpose(0, 1, 2))
        sd = self._geom(idx)[5]
        return (sol * sd[:, None, None]).transpose(2, 1, 0)  # (2, K, e)

    def ghost_table(self, t, n_own_elem):
        """Per Dirichlet slot: ghost moments (5, NT) and sample (H, |u.n|) (2, 3)."""
        ops = self.ops
        el, loc = self.bnd_elem, self.bnd_local
        nb = len(el)
        mom = np.zeros((nb, 5, ops.NT))
        smp = np.zeros((nb, 2, 3))
        if nb == 0:
            return mom, smp
        B11, B12, B21, B22 = (self.geo[r, el] for r in range(4))
        a1x, a1y = self.geo[4, el], self.geo[5, el]
        for j in range(3):
            rows = np.flatnonzero(loc == j)
            if not len(rows):
                continue
            x1, x2 = O.edge_xy(j, ops.gs)
            X = a1x[rows, None] + B11[rows, None] * x1 + B12[rows, None] * x2
            Y = a1y[rows, None] + B21[rows, None] * x1 + B22[rows, None] * x2
            vals = self.scn.exact_with_velocity(X, Y, t)
            for f in range(5):
                mom[rows, f] = vals[f] @ ops.gpsi.T
            x1, x2 = O.edge_xy(j, SAMPLES)
            X = a1x[rows, None] + B11[rows, None] * x1 + B12[rows, None] * x2
            Y = a1y[rows, None] + B21[rows, None] * x1 + B22[rows, None] * x2
            xi, Uq, Vq, uu, uv = self.scn.exact_with_velocity(X, Y, t)
            d = (np.stack([B11[rows], B21[rows]]) * [[-1], [1]] if j == 0 else None)
            dref = {0: (-1.0, 1.0), 1: (0.0, -1.0), 2: (1.0, 0.0)}[j]
            dx = B11[rows] * dref[0] + B12[rows] * dref[1]
            dy = B21[rows] * dref[0] + B22[rows] * dref[1]
            ln = np.hypot(dx, dy)
            n1, n2 = dy / ln, -dx / ln
            del d
            smp[rows, 0] = self.scn.hb(X, Y) + xi
            smp[rows, 1] = np.abs(uu * n1[:, None] + uv * n2[:, None])
        return mom, smp

    def rhs(self, c, u, t, terms=7, lam_out=None):
        """c (3, K, ld), u (2, K, ld) -> rhs (3, K, n) for owned elements."""
        ops, scn, g = self.ops, self.scn, self.scn.g
        K, NT, n = ops.K, ops.NT, self.n
        idx = np.arange(n)
        B11, B12, B21, B22, det, sd = self._geom(idx)
        xi, cU, cV = c[0][:, :n], c[1][:, :n], c[2][:, :n]
        uu, uv = u[0][:, :n], u[1][:, :n]
        hbf = self._hbfull(idx)
        out = np.zeros((3, K, n))
        if terms & 1:  # volume
            alpha = B22 * cU - B12 * cV
            beta = -B21 * cU + B11 * cV
            out[0] += (ops.S[0] @ alpha + ops.S[1] @ beta) / det
            a = B22 * uu - B12 * uv
            b = -B21 * uu + B11 * uv
            Z = np.einsum("pim,me->pie", ops.T[0], a) + np.einsum("pim,me->pie", ops.T[1], b)
            w = 0.5 * xi + (hbf if scn.hb_mode == "linear" else 0.0)
            pi1 = g * np.einsum("pim,ie,me->pe", ops.T[0], xi, w)
            pi2 = g * np.einsum("pim,ie,me->pe", ops.T[1], xi, w)
            d32 = det * sd
            out[1] += (np.einsum("pie,ie->pe", Z, cU) + B22 * pi1 - B21 * pi2) / d32
            out[2] += (np.einsum("pie,ie->pe", Z, cV) - B12 * pi1 + B11 * pi2) / d32
        if terms & 4:  # source
            gx = self._hbgrad(idx)
            out[1] += -scn.tau_bf * cU + scn.f_c * cV + g * gx[0] * xi
            out[2] += -scn.tau_bf * cV - scn.f_c * cU + g * gx[1] * xi
            if scn.forcing is not None or scn.mass_source is not None:
                x = self.geo[4, :n, None] + B11[:, None] * ops.qref[:, 0] + B12[:, None] * ops.qref[:, 1]
                y = self.geo[5, :n, None] + B21[:, None] * ops.qref[:, 0] + B22[:, None] * ops.qref[:, 1]
                if scn.forcing is not None:
                    Fx, Fy = scn.forcing(x, y, t)
                    out[1] += sd * (ops.qproj @ Fx.T)
                    out[2] += sd * (ops.qproj @ Fy.T)
                if scn.mass_source is not None:
                    out[0] += sd * (ops.qproj @ scn.mass_source(x, y, t).T)
        if terms & 2:
            mom, smp = self.ghost_table(t, n)
            for j in range(3):
                self._edge(j, c, u, out, idx, (B11, B12, B21, B22, det, sd), mom, smp, lam_out)
        return out

    def _hbgrad(self, idx):
        if self.hb.shape[0] < 3:
            return np.zeros((2, len(idx)))
        b = O.Basis(1)
        g0 = b.grad(np.zeros(1), np.zeros(1))[:3, :, 0]
        d1, d2 = g0[:, 0] @ self.hb[:3, idx], g0[:, 1] @ self.hb[:3, idx]
        B11, B12, B21, B22, det, sd = self._geom(idx)
        sc = det * sd
        return np.stack([(B22 * d1 - B21 * d2) / sc, (-B12 * d1 + B11 * d2) / sc])

    def _traces(self, j, fields, idx, sd):
        """Physical trace moments (NT, e) on local edge(s) j (scalar or per element)."""
        L = self.ops.Lam[j]  # (K, NT) or (e, K, NT)
        if L.ndim == 2:
            return [np.einsum("ia,ie->ae", L, f) / sd for f in fields]
        return [np.einsum("eia,ie->ae", L, f) / sd for f in fields]

    def _edge(self, j, c, u, out, idx, gm, mom, smp, lam_out):
        ops, scn, g = self.ops, self.scn, self.scn.g
        B11, B12, B21, B22, det, sd = gm
        n = len(idx)
        dref = {0: (-1.0, 1.0), 1: (0.0, -1.0), 2: (1.0, 0.0)}[j]
        dx = B11 * dref[0] + B12 * dref[1]
        dy = B21 * dref[0] + B22 * dref[1]
        ln = np.hypot(dx, dy)
        n1, n2 = dy / ln, -dx / ln
        hbK = self._hbfull(idx)
        lin = scn.hb_mode == "linear"
        own = self._traces(j, [c[0][:, :n], c[1][:, :n], c[2][:, :n], u[0][:, :n], u[1][:, :n],
                               hbK], idx, sd)
        code = self.nbr[j, :n].astype(np.int64)
        inner = code >= 0
        halo = inner & ((code & 3) == 3)  # other partition's element: row of self.ht
        hrow = np.where(halo, code >> 2, 0)
        nb = np.where(inner & ~halo, code >> 2, 0)
        jn = np.where(inner & ~halo, code & 3, 0)
        v = np.where(inner, 0, -1 - code)
        kind = v & 1
        slot = v >> 1
        # neighbour side
        sdn = self._geom(nb)[5]
        hbn = self._hbfull(nb)
        oth = self._traces(jn, [c[0][:, nb], c[1][:, nb], c[2][:, nb], u[0][:, nb], u[1][:, nb],
                                hbn], nb, sdn)
        if halo.any():
            for f in range(6):
                oth[f][:, halo] = self.ht[hrow[halo], f].T
        oth = [ops.R[:, None] * f for f in oth]
        # boundary ghosts
        bd = ~inner & (kind == 0)
        bw = ~inner & (kind == 1)
        if bd.any():
            s_ = slot[bd]
            for f in range(5):
                oth[f][:, bd] = mom[s_, f].T
            oth[5][:, bd] = own[5][:, bd]
        if bw.any():
            qn = n1[bw] * own[1][:, bw] + n2[bw] * own[2][:, bw]
            vn = n1[bw] * own[3][:, bw] + n2[bw] * own[4][:, bw]
            oth[0][:, bw] = own[0][:, bw]
            oth[1][:, bw] = own[1][:, bw] - 2 * n1[bw] * qn
            oth[2][:, bw] = own[2][:, bw] - 2 * n2[bw] * qn
            oth[3][:, bw] = own[3][:, bw] - 2 * n1[bw] * vn
            oth[4][:, bw] = own[4][:, bw] - 2 * n2[bw] * vn
            oth[5][:, bw] = own[5][:, bw]
        # lambda from samples
        def samp(tr):
            H = ops.psi_s.T @ (tr[5] + tr[0])
            un = np.abs(ops.psi_s.T @ (n1 * tr[3] + n2 * tr[4]))
            return H, un
        Ho, uo = samp(own)
        Hn, un_ = samp([ops.R[:, None] * f for f in oth])  # back to neighbour frame
        if bd.any():
            Hn[:, bd] = smp[slot[bd], 0].T
            un_[:, bd] = smp[slot[bd], 1].T
        if (np.minimum(Ho.min(axis=0), Hn.min(axis=0)) <= 0).any():
            raise O.DryState("non-positive depth at an edge sample")
        sp_ = lambda H, un: un + np.sqrt(np.maximum(g * H, 0.0))  # noqa: E731
        lam = np.maximum(sp_(Ho, uo).max(axis=0), sp_(Hn, un_).max(axis=0))
        if lam_out is not None:
            lam_out[j, :n] = lam
        # flux in trace space
        def side(tr):
            unn = n1 * tr[3] + n2 * tr[4]
            wv = 0.5 * tr[0] + (tr[5] if lin else 0.0)
            P = g * jprod(ops.J, tr[0], wv)
            return jprod(ops.J, tr[1], unn), jprod(ops.J, tr[2], unn), P
        A1, C1, P1 = side(own)
        A2, C2, P2 = side(oth)
        Fx = 0.5 * (n1 * (own[1] + oth[1]) + n2 * (own[2] + oth[2])) + 0.5 * lam * (own[0] - oth[0])
        FU = 0.5 * (A1 + A2 + n1 * (P1 + P2)) + 0.5 * lam * (own[1] - oth[1])
        FV = 0.5 * (C1 + C2 + n2 * (P1 + P2)) + 0.5 * lam * (own[2] - oth[2])
        if not lin:
            raise NotImplementedError("hb_mode='const' edge term")
        L = ops.Lam[j]
        s = ln / sd
        for f, F in enumerate((Fx, FU, FV)):
            out[f] -= s * (L @ F)

    def halo_traces(self, c, u, items):
        """Halo trace rows (n, 6, NT) of (element items >> 2, edge items & 3),
        the neighbour-side traces ``_edge`` computes for in-partition
        neighbours (the multi-rank CPU tests exchange these)."""
        items = np.asarray(items, dtype=np.int64)
        e, j = items >> 2, items & 3
        sd = self._geom(e)[5]
        tr = self._traces(j, [c[0][:, e], c[1][:, e], c[2][:, e], u[0][:, e], u[1][:, e],
                              self._hbfull(e)], e, sd)
        return np.stack(tr, axis=1).transpose(2, 1, 0)

    def stage_coeffs(self, a, b, c_in, u_in, c0, t, dt):
        """c_out = a c0 + b (c_in + dt L(c_in)) for owned elements, and its velocity."""
        n = self.n
        r = self.rhs(c_in, u_in, t)
        cn = a * c0[:, :, :n] + b * (c_in[:, :, :n] + dt * r)
        full = c_in.copy()
        full[:, :, :n] = cn
        return cn, self.velocity(full)

    def stage(self, s, c_in, u_in, c0, t, dt):
        """SSP-RK stage s (1-based) for order k; returns (c_out, u_out) owned part."""
        k = self.k
        r = self.rhs(c_in, u_in, t)
        n = self.n
        if s == 1:
            a, b = 0.0, 1.0
        elif k == 1:
            a, b = 0.5, 0.5
        elif s == 2:
            a, b = 0.75, 0.25
        else:
            a, b = 1.0 / 3.0, 2.0 / 3.0
        cn = a * c0[:, :, :n] + b * (c_in[:, :, :n] + dt * r)
        full = c_in.copy()
        full[:, :, :n] = cn
        return cn, self.velocity(full)
