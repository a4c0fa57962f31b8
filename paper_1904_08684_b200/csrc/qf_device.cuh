// Device building blocks of the per-stage RHS path (sm_100a, FP64).
//
// One thread owns one element (structure-of-arrays state, element index
// fastest, so every (field, mode) load of a warp is one coalesced 256 B
// line).  The per-order literal-constant operators come from
// generated/qf_order{k}.cuh (paper_1904_08684_b200/codegen.py).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace qf {

template <int k>
struct Ord;
template <int k>
struct Tabs;

constexpr double TWO_PI = 6.283185307179586;

enum : unsigned { BIT_DRY = 1u, BIT_SINGULAR = 2u, BIT_NONFINITE = 4u };
enum : int { TERM_VOL = 1, TERM_EDGE = 2, TERM_SRC = 4 };
enum : int { SCN_NONE = 0, SCN_MMS = 1, SCN_TRAVEL = 2, SCN_LAKE = 3 };

// static tables, passed by value
struct Tab {
  const double* __restrict__ geo;    // [6][ld]
  const double* __restrict__ hb;     // [NH][ld]
  const int* __restrict__ nbr;       // [3][ld]
  const double* __restrict__ ghost;  // [n_bnd][5*NT+6]
  int64_t ld;
};

struct Phys {
  double g, fc, tau;
  int hb_linear, kind, forcing;
  int taylor;  // element-local Taylor sincos for the MMS forcing (|2 pi dx| <= 0.06)
  double p[8];
};

// sin / cos of a small angle z (|z| <= 0.06): truncation < 1e-19 relative
__device__ __forceinline__ void sincos_small(double z, double& s, double& c) {
  const double z2 = z * z;
  s = z * fma(z2, fma(z2, fma(z2, fma(z2, 2.7557319223985893e-06, -1.984126984126984e-04),
                                   8.333333333333333e-03), -1.6666666666666666e-01), 1.0);
  c = fma(z2, fma(z2, fma(z2, fma(z2, 2.48015873015873e-05, -1.388888888888889e-03),
                               4.1666666666666664e-02), -0.5), 1.0);
}

__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }

// ------------------------------------------------------------ scenarios
// Closed forms of paper_1904_08684_b200/scenario.py (reference
// scenario.py:51-55 exact_with_velocity, :69-94 manufactured forcing).

__device__ __forceinline__ double hb_exact(const Phys& P, double x, double y) {
  return P.p[0] + P.p[1] * x + P.p[2] * y + P.p[3] * x * y;
}

__device__ __forceinline__ void exact3(const Phys& P, double x, double y, double t, double& xi,
                                       double& U, double& V) {
  if (P.kind == SCN_MMS) {
    const double A = P.p[4], au = P.p[5], av = P.p[6];
    xi = A * sinpi(2.0 * (x + y - t));
    const double H = hb_exact(P, x, y) + xi;
    U = H * au * cospi(2.0 * (x - t));
    V = H * av * sinpi(2.0 * (y - t));
  } else if (P.kind == SCN_TRAVEL) {
    const double Ca = P.p[4], Ct = P.p[5], ya = P.p[6];
    const double s = sinpi((x + y + Ct * t) / 600.0);
    xi = 2.0 + ya - 2.0 * Ca * s;
    U = 2.0 * ya + Ca * Ct * s;
    V = ya + Ca * Ct * s;
  } else if (P.kind == SCN_LAKE) {
    xi = P.p[4];
    U = 0.0;
    V = 0.0;
  } else {
    xi = U = V = 0.0;
  }
}

// Fx = U_t + (U^2/H)_x + (UV/H)_y + tau U - fc V + g H xi_x, Fy alike.
__device__ __forceinline__ void flux_forcing(const Phys& P, double H, double Hx, double Hy,
                                             double U, double Ut, double Ux, double Uy, double V,
                                             double Vt, double Vx, double Vy, double xix,
                                             double xiy, double& Fx, double& Fy) {
  const double iH = 1.0 / H, uu = U * iH, vv = V * iH;
  Fx = Ut + 2.0 * uu * Ux - uu * uu * Hx + (Uy * V + U * Vy) * iH - uu * vv * Hy + P.tau * U -
       P.fc * V + P.g * H * xix;
  Fy = Vt + (Ux * V + U * Vx) * iH - uu * vv * Hx + 2.0 * vv * Vy - vv * vv * Hy + P.tau * V +
       P.fc * U + P.g * H * xiy;
}

// Volume source of the family at (x, y): S (xi mass source), Fx, Fy.
// (st, ct) = (sin 2 pi t, cos 2 pi t) for MMS; the spatial phases use two
// sincospi per point and angle addition.
// MMS: (sx, cx, sy, cy) = sin/cos(2 pi x), sin/cos(2 pi y) supplied by the caller.
__device__ __forceinline__ void forcing_mms(const Phys& P, double x, double y, double sx,
                                            double cx, double sy, double cy, double st, double ct,
                                            double& S, double& Fx, double& Fy) {
    const double A = P.p[4], au = P.p[5], av = P.p[6];
    const double s2 = sx * ct - cx * st, c2 = cx * ct + sx * st;  // 2 pi (x - t)
    const double s3 = sy * ct - cy * st, c3 = cy * ct + sy * st;  // 2 pi (y - t)
    const double sxy = sx * cy + cx * sy, cxy = cx * cy - sx * sy;
    const double s1 = sxy * ct - cxy * st, c1 = cxy * ct + sxy * st;  // 2 pi (x + y - t)
    const double xi = A * s1, xd = TWO_PI * A * c1;                  // xi_x = xi_y = -xi_t
    const double u = au * c2, ux = -TWO_PI * au * s2;                  // u_t = -u_x
    const double v = av * s3, vy = TWO_PI * av * c3;                   // v_t = -v_y
    const double H = hb_exact(P, x, y) + xi;
    const double Hx = P.p[1] + P.p[3] * y + xd, Hy = P.p[2] + P.p[3] * x + xd, Ht = -xd;
    const double U = H * u, V = H * v;
    const double Ut = Ht * u - H * ux, Ux = Hx * u + H * ux, Uy = Hy * u;
    const double Vt = Ht * v - H * vy, Vx = Hx * v, Vy = Hy * v + H * vy;
    S = -xd + Ux + Vy;
    flux_forcing(P, H, Hx, Hy, U, Ut, Ux, Uy, V, Vt, Vx, Vy, xd, xd, Fx, Fy);
}

__device__ __forceinline__ void forcing(const Phys& P, double x, double y, double t, double st,
                                        double ct, double& S, double& Fx, double& Fy) {
  if (P.kind == SCN_MMS) {
    const double A = P.p[4], au = P.p[5], av = P.p[6];
    double sx, cx, sy, cy;
    sincospi(2.0 * x, &sx, &cx);
    sincospi(2.0 * y, &sy, &cy);
    const double s2 = sx * ct - cx * st, c2 = cx * ct + sx * st;  // 2 pi (x - t)
    const double s3 = sy * ct - cy * st, c3 = cy * ct + sy * st;  // 2 pi (y - t)
    const double sxy = sx * cy + cx * sy, cxy = cx * cy - sx * sy;
    const double s1 = sxy * ct - cxy * st, c1 = cxy * ct + sxy * st;  // 2 pi (x + y - t)
    const double xi = A * s1, xd = TWO_PI * A * c1;                  // xi_x = xi_y = -xi_t
    const double u = au * c2, ux = -TWO_PI * au * s2;                  // u_t = -u_x
    const double v = av * s3, vy = TWO_PI * av * c3;                   // v_t = -v_y
    const double H = hb_exact(P, x, y) + xi;
    const double Hx = P.p[1] + P.p[3] * y + xd, Hy = P.p[2] + P.p[3] * x + xd, Ht = -xd;
    const double U = H * u, V = H * v;
    const double Ut = Ht * u - H * ux, Ux = Hx * u + H * ux, Uy = Hy * u;
    const double Vt = Ht * v - H * vy, Vx = Hx * v, Vy = Hy * v + H * vy;
    S = -xd + Ux + Vy;
    flux_forcing(P, H, Hx, Hy, U, Ut, Ux, Uy, V, Vt, Vx, Vy, xd, xd, Fx, Fy);
  } else if (P.kind == SCN_TRAVEL) {
    const double Ca = P.p[4], Ct = P.p[5], ya = P.p[6];
    const double kk = 3.141592653589793 / 600.0;
    double s, c;
    sincospi((x + y + Ct * t) / 600.0, &s, &c);
    const double xi = 2.0 + ya - 2.0 * Ca * s, dxi = -2.0 * Ca * c * kk;
    const double U = 2.0 * ya + Ca * Ct * s, V = ya + Ca * Ct * s, dq = Ca * Ct * c * kk;
    const double H = hb_exact(P, x, y) + xi;
    S = 0.0;
    flux_forcing(P, H, P.p[1] + dxi, P.p[2] + dxi, U, Ct * dq, dq, dq, V, Ct * dq, dq, dq, dxi,
                 dxi, Fx, Fy);
  } else {
    S = Fx = Fy = 0.0;
  }
}

}  // namespace qf
