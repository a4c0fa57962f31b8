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
template <int k>
struct Mma;  // FP64 tensor-core volume advection (generated for k >= 3)

// shared-memory load kept in program order with the MMAs (see Mma<k>::adv)
__device__ __forceinline__ double lds64(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];"
               : "=d"(v)
               : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))));
  return v;
}

// D = A B + C for one m8n8k4 FP64 tile (a, b: this lane's fragments; d0/d1:
// the lane's two accumulators, updated in place)
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

constexpr double TWO_PI = 6.283185307179586;

enum : unsigned { BIT_DRY = 1u, BIT_SINGULAR = 2u, BIT_NONFINITE = 4u };
enum : int { TERM_VOL = 1, TERM_EDGE = 2, TERM_SRC = 4 };
enum : int { SCN_NONE = 0, SCN_MMS = 1, SCN_TRAVEL = 2, SCN_LAKE = 3, SCN_USER = 4 };

// static tables, passed by value
struct Tab {
  const double* __restrict__ geo;    // [6][ld]
  const double* __restrict__ hb;     // [NH][ld]
  const int* __restrict__ nbr;       // [3][ld]
  const double* __restrict__ ghost;  // [stage][n_bnd][5*NG+6] raw exact data
  const double* __restrict__ hbt;    // [3*NT+1][ld] static h_b traces (qf_static)
  int64_t ld;
  int n_bnd;
  // MMS phase-offset table of a mesh whose element Jacobians take at most
  // two values (uniform split-square meshes), or null; layout UniTab below
  const double* __restrict__ uni;
};

// uni table: [0..3] the Jacobian B of class 1 (every other element is
// class 0), [8 + c*(6*NQ+2) + 6*q + 0..5] sin z, cos z, sin w, cos w,
// sin(z+w), cos(z+w) of the class-c phase offsets z = 2 pi (B r_q)_x,
// w = 2 pi (B r_q)_y at quadrature point q (r_q minus the centroid); the
// 2-double pad puts the two class rows in different shared-memory banks
__host__ __device__ constexpr int uni_size(int nq) { return 8 + 2 * (6 * nq + 2); }

struct Phys {
  double g, fc, tau;
  int hb_linear, kind, forcing;
  int taylor;  // element-local Taylor sincos for the MMS forcing: 1 (|2 pi dx| <= 0.06), 2 (<= 0.02)
  double p[8];
};

// sin / cos of a small angle z (|z| <= 0.06): truncation < 1e-19 relative
// |z| <= 0.02: remainders z^9/9! and z^8/8! are below 1e-18
// (coefficients in the constant bank: DFMA operands instead of per-iteration
// 64-bit immediates materialised by register moves)
__constant__ double qf_taylor7[5] = {-1.984126984126984e-04, 8.333333333333333e-03,
                                     -1.6666666666666666e-01, -1.388888888888889e-03,
                                     4.1666666666666664e-02};
__device__ __forceinline__ void sincos_small7(double z, double& s, double& c) {
  const double z2 = z * z;
  s = z * fma(z2, fma(z2, fma(z2, qf_taylor7[0], qf_taylor7[1]), qf_taylor7[2]), 1.0);
  c = fma(z2, fma(z2, fma(z2, qf_taylor7[3], qf_taylor7[4]), -0.5), 1.0);
}

__device__ __forceinline__ void sincos_small(double z, double& s, double& c) {
  const double z2 = z * z;
  s = z * fma(z2, fma(z2, fma(z2, fma(z2, 2.7557319223985893e-06, -1.984126984126984e-04),
                                   8.333333333333333e-03), -1.6666666666666666e-01), 1.0);
  c = fma(z2, fma(z2, fma(z2, fma(z2, 2.48015873015873e-05, -1.388888888888889e-03),
                               4.1666666666666664e-02), -0.5), 1.0);
}

__device__ __forceinline__ double ldg(const double* p) { return __ldg(p); }

// 1/sqrt(x) for normal positive x: MUFU seed (rsqrt.approx.f64) + one
// third-order Newton step; <= 1.21 ulp, x * rsqrt_fast(x) <= 0.99 ulp from
// sqrt(x) (tools/micro/rsqrt_acc.cu).  ~6 instructions instead of the
// library's ~20 with special-case branches; used by every kernel for detB,
// edge normals and wave speeds, so all threads that evaluate the same
// quantity get the same bits.
__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-(x * y), y, 1.0);  // 1 - x y^2
  return fma(y, e * fma(0.375, e, 0.5), y);
}

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
// MMS from element-local phases: (s2,c2) = sin/cos 2pi(x-t), (s3,c3) =
// sin/cos 2pi(y-t), (s1,c1) = sin/cos 2pi(x+y-t).  With U = H u, V = H v the
// reference's manufactured forcing (scenario.py:78-93) is division-free:
//   Fx = u D + H (u_t + 2 u u_x + u v_y + g xi_x),
//   Fy = v D + H (v_t + u_x v + 2 v v_y + g xi_y),   D = H_t + u H_x + v H_y,
//   S  = xi_t + H_x u + H u_x + H_y v + H v_y   (u_y = v_x = 0).
template <bool FRIC = true>  // FRIC: friction / Coriolis terms compiled (else tau = f_c = 0)
__device__ __forceinline__ void forcing_mms(const Phys& P, double x, double y, double s1,
                                            double c1, double s2, double c2, double s3,
                                            double c3, double& S, double& Fx, double& Fy) {
  const double A = P.p[4], au = P.p[5], av = P.p[6];
  const double xi = A * s1, xd = TWO_PI * A * c1;  // xi_x = xi_y = -xi_t
  const double u = au * c2, ux = -TWO_PI * au * s2;  // u_t = -u_x
  const double v = av * s3, vy = TWO_PI * av * c3;   // v_t = -v_y
  const double H = hb_exact(P, x, y) + xi;
  const double Hx = P.p[1] + P.p[3] * y + xd, Hy = P.p[2] + P.p[3] * x + xd;
  const double D = fma(u, Hx, fma(v, Hy, -xd));
  const double gxd = P.g * xd;
  Fx = fma(u, D, H * fma(u, fma(2.0, ux, vy), gxd - ux));
  Fy = fma(v, D, H * fma(v, fma(2.0, vy, ux), gxd - vy));
  if (FRIC && (P.tau != 0.0 || P.fc != 0.0)) {  // (adding zero terms would not change the bits)
    Fx = Fx + P.tau * H * u - P.fc * H * v;
    Fy = Fy + P.tau * H * v + P.fc * H * u;
  }
  S = fma(Hx, u, fma(Hy, v, fma(H, ux + vy, -xd)));
}

__device__ __forceinline__ void forcing(const Phys& P, double x, double y, double t, double st,
                                        double ct, double& S, double& Fx, double& Fy) {
  if (P.kind == SCN_MMS) {
    double s1, c1, s2, c2, s3, c3;
    sincospi(2.0 * (x + y - t), &s1, &c1);
    sincospi(2.0 * (x - t), &s2, &c2);
    sincospi(2.0 * (y - t), &s3, &c3);
    forcing_mms(P, x, y, s1, c1, s2, c2, s3, c3, S, Fx, Fy);
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
