// User scenarios on the device: Dirichlet data and manufactured forcing of
// a reference ``custom_scenario`` (reference scenario.py:153-157, forcing
// from ``_manufacture`` :69-94), compiled per scenario into its own module.
//
// paper_1904_08684_b200/scenario.py prints the SymPy expressions as CUDA
// (struct UserScn: exact(x, y, t) -> xi, U, V, h_b; forcing(x, y, t) ->
// Fx, Fy) and instantiates the two kernels below; the module is loaded by
// qf_user_scenario (include/qfswe.h).  The kernels write exactly what the
// built-in closed-form families produce inside the library: the Dirichlet
// ghost table of ghost_kernel (reference solver.py:395-402, 636-653) and the
// projected forcing rows sqrt(detB) sum_q w_q phi_p(q) F(x_q, t) (solver.py
// :719-724), which the stage kernel adds to its source terms.
#pragma once
#include "qf_device.cuh"

namespace qf {

template <int k, class Scn>
__device__ __forceinline__ void user_ghost(const Tab& T, const int* __restrict__ bel,
                                           const int* __restrict__ bloc, int nb, int nstage,
                                           double t0, const double* t_dev, double3 toffs,
                                           double* ghost) {
  using O = Ord<k>;
  using TB = Tabs<k>;
  constexpr int NG = O::NG, NP = NG + 3;
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= nstage * nb * NP) return;
  const int pt = id % NP, slot = (id / NP) % nb, st = id / (NP * nb);
  const double toff = st == 0 ? toffs.x : (st == 1 ? toffs.y : toffs.z);
  const double t = t_dev ? t_dev[0] + toff * t_dev[1] : t0 + toff;
  const int64_t ld = T.ld;
  const int e = bel[slot], j = bloc[slot];
  const double B11 = T.geo[e], B12 = T.geo[ld + e], B21 = T.geo[2 * ld + e], B22 = T.geo[3 * ld + e];
  const double a1x = T.geo[4 * ld + e], a1y = T.geo[5 * ld + e];
  // reference edge maps (x1, x2)(s): e0 (1-s, s), e1 (0, 1-s), e2 (s, 0)
  const double x0 = j == 0 ? 1.0 : 0.0, xs = j == 0 ? -1.0 : (j == 2 ? 1.0 : 0.0);
  const double y0 = j == 1 ? 1.0 : 0.0, ys = j == 0 ? 1.0 : (j == 1 ? -1.0 : 0.0);
  const double sv = pt < NG ? TB::ptr()[TB::GS + pt] : 0.5 * (pt - NG);
  const double r1 = x0 + xs * sv, r2 = y0 + ys * sv;
  const double x = a1x + B11 * r1 + B12 * r2, y = a1y + B21 * r1 + B22 * r2;
  double xi, U, V, hb;
  Scn::exact(x, y, t, xi, U, V, hb);
  const double H = hb + xi;
  double* out = ghost + ((int64_t)st * nb + slot) * (5 * NG + 6);
  if (pt < NG) {
    out[pt] = xi;
    out[NG + pt] = U;
    out[2 * NG + pt] = V;
    out[3 * NG + pt] = U / H;
    out[4 * NG + pt] = V / H;
  } else {
    const double dx = B11 * xs + B12 * ys, dy = B21 * xs + B22 * ys;
    const double ln = sqrt(dx * dx + dy * dy);
    out[5 * NG + pt - NG] = H;
    out[5 * NG + 3 + pt - NG] = fabs((U * (dy / ln) - V * (dx / ln)) / H);
  }
}

// frc[i][ld] (i < 2K): U and V forcing rows of elements [e0, e0 + n) at
// t = t_dev[0] + toff * t_dev[1] (or t0 without t_dev); there is no xi row
// (the reference rejects a non-zero mass residual, scenario.py:72-77)
template <int k, class Scn>
__device__ __forceinline__ void user_forcing(const Tab& T, const double* t_dev, double t0,
                                             double toff, int e0, int n, double* frc) {
  using O = Ord<k>;
  using TB = Tabs<k>;
  constexpr int K = O::K, NQ = O::NQ;
  const int e = e0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= e0 + n) return;
  const double t = t_dev ? t_dev[0] + toff * t_dev[1] : t0;
  const int64_t ld = T.ld;
  const double B11 = T.geo[e], B12 = T.geo[ld + e], B21 = T.geo[2 * ld + e], B22 = T.geo[3 * ld + e];
  const double a1x = T.geo[4 * ld + e], a1y = T.geo[5 * ld + e];
  const double sd = sqrt(B11 * B22 - B12 * B21);
  const double* tab = TB::ptr();
  double rU[K], rV[K];
#pragma unroll
  for (int p = 0; p < K; ++p) rU[p] = rV[p] = 0.0;
  for (int q = 0; q < NQ; ++q) {
    const double x1 = tab[TB::QX + q], x2 = tab[TB::QY + q];
    const double x = a1x + B11 * x1 + B12 * x2, y = a1y + B21 * x1 + B22 * x2;
    double Fx, Fy;
    Scn::forcing(x, y, t, Fx, Fy);
#pragma unroll
    for (int p = 0; p < K; ++p) {
      const double w = tab[TB::P + q * K + p];
      rU[p] = fma(w, Fx * sd, rU[p]);
      rV[p] = fma(w, Fy * sd, rV[p]);
    }
  }
#pragma unroll
  for (int p = 0; p < K; ++p) {
    frc[p * ld + e] = rU[p];
    frc[(K + p) * ld + e] = rV[p];
  }
}

}  // namespace qf
