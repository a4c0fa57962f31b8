// sm_100a kernels and the C ABI (include/qfswe.h) of the per-stage RHS path.
//
// Replaces, per SSP-RK stage, the reference's solve_velocity + rhs
// (solver.py:315-741) and the RK combination (solver.py:756-764) with ONE
// fused element kernel:
//
//   load c, u (own)  -> volume terms (factorised stiffness-triple contraction)
//                    -> source terms (bathymetry gradient, friction, Coriolis,
//                       manufactured forcing by on-device quadrature)
//                    -> 3 edges: own + neighbour trace moments, lambda,
//                       Lax-Friedrichs flux in 1-D trace space, lift
//                       (owner-computes: no atomics, deterministic)
//                    -> RK axpy with the stage base c0
//                    -> velocity solve of the new state (LDL^T in registers)
//   store c_out, u_out
//
// The velocity of the new state is solved in the epilogue, so the next
// stage's neighbour gathers read (c, u) that are already consistent and the
// reference's separate solve at the start of each stage disappears.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <string>
#include <utility>
#include <vector>

#include "../../include/qfswe.h"
#include "qf_device.cuh"
#include "generated/qf_order0.cuh"
#include "generated/qf_order1.cuh"
#include "generated/qf_order2.cuh"
#include "generated/qf_order3.cuh"
#include "generated/qf_order4.cuh"

namespace qf {

#define QF_STR(x) #x
#define QF_UNROLL(n) _Pragma(QF_STR(unroll n))
// orders (bit mask) whose velocity kernel spills registers to shared memory
// instead of local memory (ptxas pragma enable_smem_spilling; only kernels
// without dynamic shared memory may use it, so not the stage kernel)
#ifndef QF_SMEMSPILL_VEL
#define QF_SMEMSPILL_VEL 0
#endif
#ifndef QF_EN_VOL
#define QF_EN_VOL 1
#endif
#ifndef QF_EN_SRC
#define QF_EN_SRC 1
#endif
#ifndef QF_EN_EDGE
#define QF_EN_EDGE 1
#endif
#ifndef QF_EUNROLL
#define QF_EUNROLL 1
#endif
// orders <= QF_EUNROLL_MAXK unroll the loop over the three edges (small
// bodies: k = 1 walls 142 -> 123 us/step, MMS 186 -> 170 at N = 512; k = 2
// walls N = 1024 1390 -> 1474, so k >= 2 keeps the rolled loop;
// profiles/r02_var_occ.txt)
#ifndef QF_EUNROLL_MAXK
#define QF_EUNROLL_MAXK 1
#endif
// the k = 2 RK-stage instances with manufactured forcing (C2) also unroll it
// (bench C2 0.1529 -> 0.1504 ms/step in three alternating runs, N = 128 +4 %,
// N = 512 / 1024 unchanged)
#ifndef QF_EUNROLL_FC2
#define QF_EUNROLL_FC2 1
#endif
#ifndef QF_QUNROLL
#define QF_QUNROLL 1
#endif

// non-CSE'd read-only load: lets a phase re-read its element's data from L1
// instead of keeping it live in registers across phases
__device__ __forceinline__ double ldv(const double* p) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

// detB with a fixed rounding sequence (no context-dependent FMA contraction),
// so every thread that needs an element's detB gets the same bits
__device__ __forceinline__ double det2(double b11, double b12, double b21, double b22) {
  return __fma_rn(b11, b22, -__dmul_rn(b12, b21));
}

struct StageArgs {
  const double* __restrict__ c;   // [3][K][ld]
  const double* __restrict__ u;   // [2][K][ld]
  const double* __restrict__ c0;  // RK base (may alias c_out)
  double* c_out;                  // rhs out (mode 0) or new state (mode 1)
  double* u_out;
  double* lam;                    // [3][ld] optional
  unsigned* err;
  const double* t_dev;            // optional {t, dt}
  double t, toff, dt, a, b;
  int e0, n, terms, mode;
  int gstage;                     // Dirichlet ghost table of this stage
  const double* vol;              // k >= 3: precomputed volume rhs [3K][ld] (volume_kernel)
  int hcap;                       // out-of-block request slots per block (multiple of BS/32)
  const int* push;                // optional fused halo push [3][ld] (see push_rows)
  double* mflux;                  // stage_kernel<k, true>: [3][ld] xi mode-0 rhs of each edge
  const qf_peer* peers;           // device table of the peers' destination buffers
  const double* lam_in;           // optional caller-supplied lambda [3][ld] (edge_rhs(state, t, lam))
  const double* frc;              // optional user-scenario forcing rows [2K][ld] (U, V; qf_user.cuh)
  const double* ht;               // halo trace table of the stage input (partitions), see HALO_J
};

// Neighbour code 4 h + HALO_J (a local-edge value no element has): the
// neighbour is owned by another partition and its trace moments on the
// shared edge arrive in row h of the halo trace table ht[h][6][NT] (xi, U,
// V, u, v, h_b in the neighbour's own edge parametrisation), pushed by the
// peer's stage epilogue or exchanged by qf_halo_traces + NCCL (SURVEY §8e:
// 6 (k + 1) doubles per cut edge instead of the neighbour's 5 K rows).
constexpr int HALO_J = 3;

// Trace moments of fields (xi, U, V, u, v) of one element on local edge j
// with the rounding sequence of the stage kernel's phase A2 (so a partition
// sees bit-identical neighbour traces), h_b from the static table:
// out[f * NT + a], f < 6.  c rows at c[i * ld], velocity rows in registers.
template <int k>
__device__ __forceinline__ void edge_traces6(const Tab& T, int64_t ld, int e, int j,
                                             const double* c, const double* uo, const double* vo,
                                             double* out, int ostride) {
  using O = Ord<k>;
  constexpr int K = O::K, NT = O::NT;
  const double* L = Tabs<k>::ptr() + Tabs<k>::L + j * K * NT;
  const double nisd = rsqrt_fast(det2(T.geo[e], T.geo[ld + e], T.geo[2 * ld + e], T.geo[3 * ld + e]));
#pragma unroll 1
  for (int fi = 0; fi < 5; ++fi) {
#pragma unroll
    for (int a = 0; a < NT; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < K; ++i) {
        const double f = fi < 3 ? c[(fi * K + i) * ld] : (fi == 3 ? uo[i] : vo[i]);
        acc = __fma_rn(L[i * NT + a], f, acc);
      }
      out[(fi * NT + a) * ostride] = __dmul_rn(acc, nisd);
    }
  }
#pragma unroll
  for (int a = 0; a < NT; ++a) out[(5 * NT + a) * ostride] = T.hbt[(j * NT + a) * ld + e];
}

// Fused halo exchange ("a trace-producer kernel stores directly
// into the peer's buffer"): the thread that computed a cut-adjacent
// element's new (c, u) also computes its trace moments on each cut edge and
// stores them into the peer's halo trace table (device pointers: same GPU,
// P2P or CUDA-IPC mapped over NVLink).  push[j][e] = (peer << 26) | row, or -1.
template <int k>
__device__ __forceinline__ void push_traces(const Tab& T, const int* __restrict__ push,
                                            const qf_peer* __restrict__ peers, int64_t ld, int e,
                                            const double* c_new, const double* uo,
                                            const double* vo) {
  constexpr int NT = Ord<k>::NT;
#pragma unroll 1
  for (int j = 0; j < 3; ++j) {
    const int d = __ldg(push + j * ld + e);
    if (d < 0) continue;
    const qf_peer pr = peers[d >> 26];
    const int64_t row = d & ((1 << 26) - 1);
    edge_traces6<k>(T, ld, e, j, c_new + e, uo, vo, pr.ht + row * 6 * NT, 1);
  }
}

// ---------------------------------------------------------------- edges
// One local edge j (runtime, loop not unrolled to keep the kernel inside the
// instruction cache); Lambda comes from the shared-memory copy of the
// per-order table (uniform j -> broadcast, neighbour j' -> at most 3 rows).
template <int k>
__device__ __forceinline__ void trace_s(const double* __restrict__ sL, int j, const double* f,
                                        double scale, double* t) {
  constexpr int K = Ord<k>::K, NT = Ord<k>::NT;
  const double* L = sL + j * K * NT;
#pragma unroll
  for (int a = 0; a < NT; ++a) {
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < K; ++i) acc = fma(L[i * NT + a], f[i], acc);
    t[a] = acc * scale;
  }
}

// literal-constant trace / lift of local edge j (switch is warp-uniform for
// the own side; for the neighbour side it is uniform on warp-homogeneous
// element orders, see the interleaved thread mapping of stage_kernel)
template <int k>
__device__ __forceinline__ void trace_lit(int j, const double* f, double scale, double* t) {
  using O = Ord<k>;
  if (j == 0)
    O::trace0(f, t);
  else if (j == 1)
    O::trace1(f, t);
  else
    O::trace2(f, t);
#pragma unroll
  for (int a = 0; a < O::NT; ++a) t[a] = __dmul_rn(t[a], scale);
}

// threads (= elements) per block of the stage kernel
#ifndef QF_BS2
#define QF_BS2 128
#endif
#ifndef QF_BS3
#define QF_BS3 128
#endif
#ifndef QF_BS4
#define QF_BS4 128
#endif
template <int k>
struct Blk {
  static constexpr int value = k <= 1 ? 128 : (k == 2 ? QF_BS2 : (k == 3 ? QF_BS3 : QF_BS4));
};

// Shared-memory trace exchange.  Phase A: every thread writes its element's
// physical trace moments (xi, U, V, u, v on local edges 0, 1, 2) to
// s_tr[((j*5 + f)*NT + a)*BS + slot]; the static h_b traces come from the
// precomputed table T.hbt (qf_static).
// Phase B: a neighbour inside the block is read from there (no gather, no
// recomputation); only neighbours outside the block are gathered from global
// memory and traced.
// out-of-block neighbour traces computed cooperatively per block (phase A2)
#ifndef QF_HCAP
#define QF_HCAP 128
#endif
// orders whose stage kernel keeps the element's own data in registers
#ifndef QF_PRE_MAXK
#define QF_PRE_MAXK 2
#endif
#ifndef QF_NOFALLBACK
#define QF_NOFALLBACK 0
#endif
// Stage-kernel instance variants (compile-time code paths; a path that cannot
// occur on a problem is compiled out: smaller register / spill footprint)
enum : int {
  V_MF = 1,     // mass-flux instrumentation output
  V_FC = 2,     // manufactured forcing
  V_DIR = 4,    // Dirichlet ghosts
  V_HBC = 8,    // hb_mode "const" terms
  V_WALL = 16,  // reflective walls
  V_TAY7 = 32,  // MMS forcing with degree-7 Taylor phases only (no generic forcing code)
  V_OVF = 64,   // request-slot overflow path (in-loop gather of out-of-block neighbours)
  V_STG = 128,  // RK-stage launch only: all terms, mode 1, no lambda output
  V_PUSH = 256, // fused halo push in the epilogue (k <= 2)
  V_FRIC = 512, // bottom friction / Coriolis source terms
  V_UNI = 1024, // MMS forcing with tabulated phase offsets only (Tab::uni, k <= 2)
  V_GENERAL = V_FC | V_DIR | V_HBC | V_WALL | V_OVF | V_PUSH | V_FRIC
};

// orders whose stage kernel also exchanges the static h_b edge traces through
// shared memory (6th trace field: own element from its P1 coefficients in
// phase A, bit-identical to qf_static; out-of-block neighbours copied from
// the table in phase A2), so the edge loop issues no global loads
// (round 2, after the stage-kernel variants: k = 2 is faster with the table
// reads -- 56 instead of 65 KB of shared memory per block, 9 fewer trace
// evaluations in phase A: C4 5.71 -> 5.48 ms/step, C2 155.9 -> 153.3 us/step,
// profiles/r02_var_occ.txt -- so the shared-memory h_b traces are off by default)
// (k = 1 likewise: walls 142.1 -> 139.6 us/step at N = 512)
#ifndef QF_HBS_MAXK
#define QF_HBS_MAXK 0
#endif
template <int k>
struct FS {
  static constexpr int value = k <= QF_HBS_MAXK ? 6 : 5;  // trace fields per edge in smem
};

// Lax-Friedrichs flux moments F[3][NT] of local edge j of element e and the
// lift scale s = edge length / sqrt(detB) (reference solver.py:561-688).
template <int k, int BS = Blk<k>::value, int V = V_GENERAL>
__device__ __forceinline__ void edge_flux(const Tab& T, const Phys& P, const StageArgs& A, int e,
                                          int j, int code, int slot, int blo, int bhi,
                                          const double* __restrict__ s_tr,
                                          const double* __restrict__ s_ht, int hslot, int HC,
                                          double B11, double B12, double B21, double B22,
                                          double isd, double (&F)[3][Ord<k>::NT], double& s) {
  using O = Ord<k>;
  constexpr int K = O::K, NT = O::NT, NH = O::NH, NF = FS<k>::value;
  constexpr bool HS = NF == 6;
  const int64_t ld = T.ld;
  // own outward normal: physical image of the reference edge direction
  const double d1 = j == 0 ? -1.0 : (j == 1 ? 0.0 : 1.0);
  const double d2 = j == 0 ? 1.0 : (j == 1 ? -1.0 : 0.0);
  const double dx = B11 * d1 + B12 * d2, dy = B21 * d1 + B22 * d2;
  const double l2 = dx * dx + dy * dy, il = rsqrt_fast(l2);
  const double n1 = dy * il, n2 = -dx * il;

  double own[6][NT], oth[6][NT];
#pragma unroll
  for (int f = 0; f < NF; ++f)
#pragma unroll
    for (int a = 0; a < NT; ++a) own[f][a] = s_tr[((j * NF + f) * NT + a) * BS + slot];
  // static h_b traces (qf_static): [j*NT + a][ld], mean depth term in row 3*NT
  if constexpr (!HS) {
#pragma unroll
    for (int a = 0; a < NT; ++a) own[5][a] = ldg(T.hbt + (j * NT + a) * ld + e);
  }
  const bool hbl = !(V & V_HBC) || P.hb_linear;
  const double hbm_o = hbl ? 0.0 : ldg(T.hbt + 3 * NT * ld + e);
  double hbm_n = hbm_o;

  bool dirichlet = false;
  const double* gp = nullptr;
  if (code >= 0) {
    const int nb = code >> 2, jn = code & 3;
    const bool halo = jn == HALO_J;  // traces of another partition's element (A.ht row nb)
    if constexpr (!HS) {
#pragma unroll
      for (int a = 0; a < NT; ++a) {
        const double v = halo ? ldg(A.ht + (int64_t)nb * 6 * NT + 5 * NT + a)
                              : ldg(T.hbt + (jn * NT + a) * ld + nb);
        oth[5][a] = (a & 1) ? -v : v;  // s -> 1-s
      }
    }
    if (!hbl) hbm_n = halo ? 0.0 : ldg(T.hbt + 3 * NT * ld + nb);
    if (!halo && nb >= blo && nb < bhi) {  // neighbour traced by its own thread in phase A
      const int ns = nb - blo;
#pragma unroll
      for (int f = 0; f < NF; ++f)
#pragma unroll
        for (int a = 0; a < NT; ++a) {
          const double v = s_tr[((jn * NF + f) * NT + a) * BS + ns];
          oth[f][a] = (a & 1) ? -v : v;  // s -> 1-s
        }
    } else if (QF_NOFALLBACK || !(V & V_OVF) || hslot >= 0) {  // out-of-block, traced in A2
#pragma unroll
      for (int f = 0; f < NF; ++f)
#pragma unroll
        for (int a = 0; a < NT; ++a) {
          const double v = s_ht[(f * NT + a) * HC + hslot];
          oth[f][a] = (a & 1) ? -v : v;  // s -> 1-s
        }
    } else if (halo) {  // request list overflow, halo neighbour: its row of the trace table
#pragma unroll
      for (int f = 0; f < NF; ++f)
#pragma unroll
        for (int a = 0; a < NT; ++a) {
          const double v = ldg(A.ht + (int64_t)nb * 6 * NT + f * NT + a);
          oth[f][a] = (a & 1) ? -v : v;  // s -> 1-s
        }
    } else {  // request list overflow (rare): gather and trace here, compact code
      const double nisd = rsqrt_fast(det2(ldg(T.geo + nb), ldg(T.geo + ld + nb),
                                     ldg(T.geo + 2 * ld + nb), ldg(T.geo + 3 * ld + nb)));
      const double* L = s_ht + NF * NT * HC + jn * K * NT;  // s_L (stage_kernel layout)
      if constexpr (HS) {
#pragma unroll
        for (int a = 0; a < NT; ++a) {
          const double v = ldg(T.hbt + (jn * NT + a) * ld + nb);
          oth[5][a] = (a & 1) ? -v : v;  // s -> 1-s
        }
      }
#pragma unroll
      for (int fi = 0; fi < 5; ++fi) {
        const double* src =
            fi < 3 ? A.c + (int64_t)fi * K * ld : A.u + (int64_t)(fi - 3) * K * ld;
        if constexpr (k <= 2) {  // loads issued together
          double f[K];
#pragma unroll
          for (int i = 0; i < K; ++i) f[i] = ldg(src + i * ld + nb);
#pragma unroll
          for (int a = 0; a < NT; ++a) {
            double acc = 0.0;
#pragma unroll
            for (int i = 0; i < K; ++i) acc = __fma_rn(L[i * NT + a], f[i], acc);
            const double v = __dmul_rn(acc, nisd);
            oth[fi][a] = (a & 1) ? -v : v;  // s -> 1-s
          }
        } else {  // rolled (register pressure at high order)
#pragma unroll
          for (int a = 0; a < NT; ++a) {
            double acc = 0.0;
#pragma unroll 1
            for (int i = 0; i < K; ++i) acc = __fma_rn(L[i * NT + a], ldg(src + i * ld + nb), acc);
            const double v = __dmul_rn(acc, nisd);
            oth[fi][a] = (a & 1) ? -v : v;  // s -> 1-s
          }
        }
      }
    }
  } else {
    const int v = -1 - code, bslot = v >> 1;
    if ((V & V_DIR) && (!(V & V_WALL) || (v & 1) == 0)) {  // Dirichlet: ghost = Gauss moments of exact data
      using TB = Tabs<k>;
      constexpr int NG = O::NG;
      dirichlet = true;
      gp = T.ghost + ((int64_t)A.gstage * T.n_bnd + bslot) * (5 * NG + 6);
      const double* gw = TB::ptr() + TB::GPSI;
#pragma unroll
      for (int f = 0; f < 5; ++f) {
        double vals[NG];
#pragma unroll
        for (int g = 0; g < NG; ++g) vals[g] = ldg(gp + f * NG + g);
#pragma unroll
        for (int a = 0; a < NT; ++a) {
          double acc = 0.0;
#pragma unroll
          for (int g = 0; g < NG; ++g) acc = fma(gw[a * NG + g], vals[g], acc);
          oth[f][a] = acc;
        }
      }
      gp += 5 * NG - 5 * NT;  // samples follow the raw values
    } else {  // reflective wall: mirror the normal components
#pragma unroll
      for (int a = 0; a < NT; ++a) {
        const double qn = n1 * own[1][a] + n2 * own[2][a];
        const double vn = n1 * own[3][a] + n2 * own[4][a];
        oth[0][a] = own[0][a];
        oth[1][a] = own[1][a] - 2.0 * n1 * qn;
        oth[2][a] = own[2][a] - 2.0 * n2 * qn;
        oth[3][a] = own[3][a] - 2.0 * n1 * vn;
        oth[4][a] = own[4][a] - 2.0 * n2 * vn;
      }
    }
#pragma unroll
    for (int a = 0; a < NT; ++a) oth[5][a] = own[5][a];
  }

  // lambda = max over both sides and s in {0, 1/2, 1} of |u.n| + sqrt(gH)
  double unO[NT], unN[NT], tmp[NT], sH[3], sU[3];
#pragma unroll
  for (int a = 0; a < NT; ++a) {
    unO[a] = n1 * own[3][a] + n2 * own[4][a];
    unN[a] = n1 * oth[3][a] + n2 * oth[4][a];
    tmp[a] = own[5][a] + own[0][a];
  }
  // sqrt(max(gH, 0)) as x * rsqrt_fast(x): ~1 ulp, identical on both sides of an edge
  auto wave = [&](double H) {
    const double x = P.g * H;
    return x > 0.0 ? x * rsqrt_fast(x) : 0.0;
  };
  double lam = 0.0, hmin = 1.0;
  O::samples(tmp, sH);
  O::samples(unO, sU);
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const double w = fabs(sU[s]) + wave(sH[s]);
    lam = w > lam ? w : lam;  // (plain selects: fmax/fmin carry NaN handling)
    hmin = sH[s] < hmin ? sH[s] : hmin;
  }
  if (dirichlet) {
#pragma unroll
    for (int s = 0; s < 3; ++s) {
      sH[s] = ldg(gp + 5 * NT + s);
      sU[s] = ldg(gp + 5 * NT + 3 + s);
    }
  } else {
#pragma unroll
    for (int a = 0; a < NT; ++a) tmp[a] = oth[5][a] + oth[0][a];
    O::samples(tmp, sH);
    O::samples(unN, sU);
  }
#pragma unroll
  for (int s = 0; s < 3; ++s) {
    const double w = fabs(sU[s]) + wave(sH[s]);
    lam = w > lam ? w : lam;  // (plain selects: fmax/fmin carry NaN handling)
    hmin = sH[s] < hmin ? sH[s] : hmin;
  }
  if (!(hmin > 0.0)) atomicOr(A.err, BIT_DRY);
  if constexpr (!(V & V_STG)) {
    if (A.lam_in) lam = A.lam_in[j * ld + e];  // reference edge_rhs(state, t, lam), solver.py:690-704
    if (A.lam) A.lam[j * ld + e] = lam;
  }

  // Lax-Friedrichs flux in trace space (reference solver.py:610-613)
  double wO[NT], wN[NT], pO[NT], pN[NT], aO[NT], aN[NT], bO[NT], bN[NT];
#pragma unroll
  for (int a = 0; a < NT; ++a) {
    wO[a] = 0.5 * own[0][a] + (hbl ? own[5][a] : 0.0);
    wN[a] = 0.5 * oth[0][a] + (hbl ? oth[5][a] : 0.0);
  }
  O::jprod(own[0], wO, pO);
  O::jprod(oth[0], wN, pN);
  O::jprod(own[1], unO, aO);
  O::jprod(oth[1], unN, aN);
  O::jprod(own[2], unO, bO);
  O::jprod(oth[2], unN, bN);
  const double hl = 0.5 * lam, g = P.g;
#pragma unroll
  for (int a = 0; a < NT; ++a) {
    double pr = pO[a] + pN[a];
    if (!hbl) pr += hbm_o * own[0][a] + hbm_n * oth[0][a];
    F[0][a] = 0.5 * (n1 * (own[1][a] + oth[1][a]) + n2 * (own[2][a] + oth[2][a])) +
              hl * (own[0][a] - oth[0][a]);
    F[1][a] = 0.5 * (aO[a] + aN[a] + g * n1 * pr) + hl * (own[1][a] - oth[1][a]);
    F[2][a] = 0.5 * (bO[a] + bN[a] + g * n2 * pr) + hl * (own[2][a] - oth[2][a]);
  }
  s = l2 * il * isd;  // edge length / sqrt(detB)
}

template <int k, int BS = Blk<k>::value, int V = V_GENERAL>
__device__ __forceinline__ void edge_term(const Tab& T, const Phys& P, const StageArgs& A, int e,
                                          int j, int code, int slot, int blo, int bhi,
                                          const double* __restrict__ s_tr,
                                          const double* __restrict__ s_ht, int hslot, int HC,
                                          double B11,
                                          double B12, double B21, double B22, double isd,
                                          double* r) {
  using O = Ord<k>;
  constexpr int K = O::K, NT = O::NT;
  double F[3][NT], s;
  edge_flux<k, BS, V>(T, P, A, e, j, code, slot, blo, bhi, s_tr, s_ht, hslot, HC, B11, B12, B21, B22,
                   isd, F, s);
  // lift: r_f[p] -= (len / sqrt(detB)) sum_a Lambda_j[p, a] F_f[a]
  if (j == 0) {
    O::lift0(F[0], s, r);
    O::lift0(F[1], s, r + K);
    O::lift0(F[2], s, r + 2 * K);
  } else if (j == 1) {
    O::lift1(F[0], s, r);
    O::lift1(F[1], s, r + K);
    O::lift1(F[2], s, r + 2 * K);
  } else {
    O::lift2(F[0], s, r);
    O::lift2(F[1], s, r + K);
    O::lift2(F[2], s, r + 2 * K);
  }
  if constexpr ((V & V_MF) != 0) {  // instrument_mass_flux: this edge's xi mode-0 rhs (solver.py:619-620)
    double m[K];
#pragma unroll
    for (int p = 0; p < K; ++p) m[p] = 0.0;
    if (j == 0)
      O::lift0(F[0], s, m);
    else if (j == 1)
      O::lift1(F[0], s, m);
    else
      O::lift2(F[0], s, m);
    A.mflux[j * T.ld + e] = m[0];
  }
}

// k >= 3: the U/V rows of the volume contraction are split into VG output
// groups (term-balanced, Ord<k>::VOL_PSPLIT*), one launch each: fewer live
// accumulators (no spills) and 1/VG of the literal code per launch
// (instruction-cache working set); group 0 also writes the xi row
#ifndef QF_VG4
#define QF_VG4 2
#endif
#ifndef QF_VG3
#define QF_VG3 1
#endif
template <int k>
struct VGroups {
  static constexpr int value = k == 4 ? QF_VG4 : (k == 3 ? QF_VG3 : 1);
};

// orders (bit mask) whose RK-stage launches use lean instances: only the
// code paths the problem can take (forcing, Dirichlet, walls, const h_b,
// friction; measured at N = 512, walls: k = 1..4 2.5-3.5 % faster; with the
// stage-only V_STG: C2 51.6 -> 48.9 us, k = 2 walls 135 -> 125 us)
#ifndef QF_LEAN_INST
#define QF_LEAN_INST 30
#endif
// orders (bit mask) whose volume kernels drop the hb_mode "const" code for
// linear h_b (k = 4: stage 944 -> 907 us at N = 512; k = 3: 355 -> 374, not used)
#ifndef QF_VLEAN_ORDERS
#define QF_VLEAN_ORDERS 16
#endif
// orders (bit mask) whose whole-mesh launches use instances without the
// request-overflow path when it cannot trigger (k = 2: C2 53.5 -> 51.9 us,
// walls 144 -> 136 us at N = 512; k = 3 -0.8 %; k = 1 walls -1.5 %; k = 4 slower)
#ifndef QF_NOOVF_ORDERS
#define QF_NOOVF_ORDERS 14
#endif
// input-outer volume kernel (k = 4): pressure rows from symmetric products
// (vol_press; measured k = 4 stage 1007 -> 966 us at N = 512; the row-outer
// k = 3 path is faster without it: 381 vs 395 us)
#ifndef QF_VPRESS
#define QF_VPRESS 1
#endif
// orders >= QF_VSPLIT solve the velocity of the new state in its own launch
#ifndef QF_VSPLIT
#define QF_VSPLIT 4
#endif
template <int k>
struct Occ {
#ifndef QF_OCC2
#define QF_OCC2 3
#endif
#ifndef QF_OCC3
#define QF_OCC3 2
#endif
#ifndef QF_OCC4
#define QF_OCC4 1
#endif
  static constexpr int value = k <= 1 ? 4 : (k == 2 ? QF_OCC2 : (k == 3 ? QF_OCC3 : QF_OCC4));
};

// Volume terms, Eqs. (15)-(16) (reference solver.py:410-485, const-h_b form
// :498-510): factorised stiffness-triple contraction in literal code.
template <int k, int V = V_GENERAL>
__device__ __forceinline__ void volume_terms(const Phys& P, double B11, double B12, double B21,
                                             double B22, double isd, double idet,
                                             const double* xi, const double* cU,
                                             const double* cV, const double* u,
                                             const double* hb, double* r) {
  using O = Ord<k>;
  constexpr int K = O::K;
    double al[K], be[K], ra[K], rb[K], wv[K];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    al[i] = B22 * cU[i] - B12 * cV[i];
    be[i] = -B21 * cU[i] + B11 * cV[i];
  }
  O::vol_xi(al, be, ra);
#pragma unroll
  for (int i = 0; i < K; ++i) {
    r[i] += ra[i] * idet;
    al[i] = B22 * u[i] - B12 * u[K + i];   // a
    be[i] = -B21 * u[i] + B11 * u[K + i];  // b
    wv[i] = 0.5 * xi[i] + ((!(V & V_HBC) || P.hb_linear) ? hb[i] : 0.0);
  }
  const double g = P.g;
  O::vol_uv(cU, cV, xi, al, be, wv, g * B22, g * B21, g * B12, g * B11, ra, rb);
  const double i32 = idet * isd;
#pragma unroll
  for (int i = 0; i < K; ++i) {
    r[K + i] += ra[i] * i32;
    r[2 * K + i] += rb[i] * i32;
  }
  if ((V & V_HBC) && !P.hb_linear) {  // paper-form constant h_b (solver.py:498-510)
    const double ghb = g * hb[0] * isd * 0.7071067811865476 * idet;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      al[i] = B22 * xi[i];
      be[i] = -B21 * xi[i];
    }
    O::vol_xi(al, be, ra);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      al[i] = -B12 * xi[i];
      be[i] = B11 * xi[i];
    }
    O::vol_xi(al, be, rb);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      r[K + i] += ghb * ra[i];
      r[2 * K + i] += ghb * rb[i];
    }
  }
}

// global -> shared 8-byte asynchronous copies (no registers held)
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;" ::: "memory");
}

// Manufactured forcing at the (k+2)^2 collapsed Gauss points of element e
// (reference solver.py:719-724, scenario.py:78-93): sink(P_q, S, Fx, Fy)
// with P_q[p] = w_q phi_p(q) and the point values already scaled by sqrt(detB).
template <int k, int V = V_GENERAL, class Sink>
__device__ __forceinline__ void forcing_quad(const Phys& P, const Tab& T, int e, double t,
                                             double B11, double B12, double B21, double B22,
                                             double sd, const double* su, Sink&& sink) {
  using TB = Tabs<k>;
  constexpr int K = Ord<k>::K, NQ = Ord<k>::NQ;
  const int64_t ld = T.ld;
  const double* s_tab = TB::ptr();
  const double a1x = ldg(T.geo + 4 * ld + e), a1y = ldg(T.geo + 5 * ld + e);
  double st, ct;
  sincospi(2.0 * t, &st, &ct);
  // MMS: sin/cos(2 pi x_q) = rotation of the centroid value by the small
  // offset angle of point q, either read from the per-mesh table (su: the
  // Jacobian takes at most two values, shared memory) or Taylor-evaluated
  // (2 sincospi per element instead of 2 per quadrature point)
  const bool uni = (V & V_UNI) ? true : (!(V & V_TAY7) && k <= 2 && su != nullptr && P.kind == SCN_MMS);
  const bool tay = !uni && ((V & V_TAY7) || (P.kind == SCN_MMS && P.taylor));
  const double* su_e = nullptr;
  if (uni)
    su_e = su + 8 + ((B11 == su[0] && B12 == su[1] && B21 == su[2] && B22 == su[3]) ? 6 * NQ + 2 : 0);
  // element phases 2 pi (x0 - t), 2 pi (y0 - t), 2 pi (x0 + y0 - t) at
  // the centroid; per point only small-angle Taylor rotations follow
  const double x0 = a1x + (B11 + B12) * (1.0 / 3.0), y0 = a1y + (B21 + B22) * (1.0 / 3.0);
  double sx0 = 0.0, cx0 = 1.0, sy0 = 0.0, cy0 = 1.0, sxy0 = 0.0, cxy0 = 1.0;
  if (tay || uni) {
    sincospi(2.0 * (x0 - t), &sx0, &cx0);
    sincospi(2.0 * (y0 - t), &sy0, &cy0);
    sincospi(2.0 * (x0 + y0 - t), &sxy0, &cxy0);
  }
  // per point: offsets (r1, r2) from the centroid (table), the physical point
  // and the small phase angles 2 pi B r
  const double t11 = TWO_PI * B11, t12 = TWO_PI * B12, t21 = TWO_PI * B21, t22 = TWO_PI * B22;
  QF_UNROLL(QF_QUNROLL)
  for (int q = 0; q < NQ; ++q) {
    const double r1 = s_tab[TB::QR1 + q], r2 = s_tab[TB::QR2 + q];
    const double x = fma(B11, r1, fma(B12, r2, x0)), y = fma(B21, r1, fma(B22, r2, y0));
    double S, Fx, Fy;
    if (uni) {
      const double* o = su_e + 6 * q;
      const double sz = o[0], cz = o[1], sw = o[2], cw = o[3], szw = o[4], czw = o[5];
      forcing_mms<(V & V_FRIC) != 0>(P, x, y, fma(sxy0, czw, cxy0 * szw), fma(cxy0, czw, -sxy0 * szw),
                  fma(sx0, cz, cx0 * sz), fma(cx0, cz, -sx0 * sz), fma(sy0, cw, cy0 * sw),
                  fma(cy0, cw, -sy0 * sw), S, Fx, Fy);
    } else if (!(V & V_UNI) && tay) {
      double sz, cz, sw, cw;
      if ((V & V_TAY7) || P.taylor == 2) {
        sincos_small7(fma(t11, r1, t12 * r2), sz, cz);
        sincos_small7(fma(t21, r1, t22 * r2), sw, cw);
      } else {
        sincos_small(fma(t11, r1, t12 * r2), sz, cz);
        sincos_small(fma(t21, r1, t22 * r2), sw, cw);
      }
      const double szw = fma(sz, cw, cz * sw), czw = fma(cz, cw, -sz * sw);
      forcing_mms<(V & V_FRIC) != 0>(P, x, y, fma(sxy0, czw, cxy0 * szw), fma(cxy0, czw, -sxy0 * szw),
                  fma(sx0, cz, cx0 * sz), fma(cx0, cz, -sx0 * sz), fma(sy0, cw, cy0 * sw),
                  fma(cy0, cw, -sy0 * sw), S, Fx, Fy);
    } else if constexpr (!(V & (V_TAY7 | V_UNI))) {
      forcing(P, x, y, t, st, ct, S, Fx, Fy);
    }
    sink(s_tab + TB::P + q * K, S * sd, Fx * sd, Fy * sd);
  }
}

// ---------------------------------------------------------- stage kernel
// dynamic shared memory: per-order table | trace exchange (3*6*NT*BS) | BS
// hc: out-of-block request slots per block (runtime, qf_create measures the mesh)
// orders (bit mask) whose stage kernel stages the element's own 3K state
// rows in shared memory with one burst of cp.async (no registers held; the
// phases read them from there instead of re-reading global memory)
#ifndef QF_CSMEM
#define QF_CSMEM 8
#endif
// orders (bit mask) whose stage kernel evaluates the volume terms itself
// (no volume_kernel launch, no vol[3K][ld] round trip through HBM)
#ifndef QF_FUSEVOL
#define QF_FUSEVOL 8
#endif
template <int k>
struct FuseVol {
  static constexpr bool value = ((QF_FUSEVOL >> k) & 1) && k >= 3;
};

template <int k>
struct CSmem {
  static constexpr bool value = ((QF_CSMEM >> k) & 1) && k > QF_PRE_MAXK;
};

template <int k>
size_t stage_smem_bytes(int hc) {
  constexpr int K = Ord<k>::K, NT = Ord<k>::NT;
  constexpr int NF = FS<k>::value;
  constexpr int NU = k <= 2 ? uni_size(Ord<k>::NQ) : 0;  // MMS phase-offset table
  constexpr int CS = CSmem<k>::value ? 3 * K * Blk<k>::value : 0;  // own state rows
  return sizeof(double) * (3 * NF * NT * Blk<k>::value + NF * NT * hc + 3 * K * NT + NU + CS) +
         sizeof(int) * (hc + 8);
}

// V: compile-time variant (V_* above)
template <int k, int V = V_GENERAL>
__global__ void __launch_bounds__(Blk<k>::value, Occ<k>::value)
    stage_kernel(Tab T, Phys P, StageArgs A) {
  using O = Ord<k>;
  using TB = Tabs<k>;
  constexpr int K = O::K, NH = O::NH, NQ = O::NQ, NT = O::NT, BS = Blk<k>::value;
  const int HC = A.hcap;
  extern __shared__ double smem[];
  constexpr int NF = FS<k>::value;  // traced fields per edge: xi U V u v (+ h_b)
  static_assert(FS<k>::value == 5 || k <= QF_PRE_MAXK, "h_b smem traces need the register preload");
  double* s_tr = smem;  // trace exchange [3 edges][NF fields][NT][BS]
  double* s_ht = s_tr + 3 * NF * NT * BS;  // out-of-block neighbour traces [NF][NT][HC]
  double* s_L = s_ht + NF * NT * HC;       // Lambda [3][K][NT] (neighbour edge varies by lane)
  constexpr int NU = k <= 2 ? uni_size(NQ) : 0;
  double* s_U = s_L + 3 * K * NT;          // MMS phase-offset table (Tab::uni), k <= 2
  constexpr bool CSM = CSmem<k>::value;
  double* s_c = s_U + NU;                  // own state rows [3K][BS] (CSM)
  int* s_req = reinterpret_cast<int*>(s_c + (CSM ? 3 * K * BS : 0));  // [HC] neighbour codes, then count
  const double* s_tab = TB::ptr();  // per-order constants (constant memory, uniform reads)
  const int slot = threadIdx.x;
  const int blo = A.e0 + blockIdx.x * BS;
  const int bhi = min(blo + BS, A.e0 + A.n);
  const int e = blo + slot;
  const bool active = e < bhi;
  const int64_t ld = T.ld;
  const int ee = active ? e : blo;  // inactive threads read a valid element
  // issue every load of the element's own data up front: one memory round
  // trip, overlapped with the table copy below
  const double B11 = ldg(T.geo + ee), B12 = ldg(T.geo + ld + ee);
  const double B21 = ldg(T.geo + 2 * ld + ee), B22 = ldg(T.geo + 3 * ld + ee);
  const bool edges = (V & V_STG) || (A.terms & TERM_EDGE) != 0;
  int code[3] = {0, 0, 0};
  // k <= 2: the element's own data is loaded once up front and stays in
  // registers; for k >= 3 (6K values) each phase re-reads it (L1/L2)
  constexpr bool PRE = k <= QF_PRE_MAXK;
  double own_f[PRE ? 6 * K : 1];
  if (edges) {
#pragma unroll
    for (int j = 0; j < 3; ++j) code[j] = __ldg(T.nbr + j * ld + ee);
    if constexpr (PRE) {
#pragma unroll
      for (int i = 0; i < 3 * K; ++i) own_f[i] = ldg(A.c + i * ld + ee);
#pragma unroll
      for (int i = 0; i < 2 * K; ++i) own_f[3 * K + i] = ldg(A.u + i * ld + ee);
#pragma unroll
      for (int i = 0; i < K; ++i) own_f[5 * K + i] = i < NH ? ldg(T.hb + i * ld + ee) : 0.0;
    }
  }
  if constexpr (CSM) {  // waited for by each thread before its first read (own rows only)
#pragma unroll 1
    for (int i = 0; i < 3 * K; ++i) cp_async8(s_c + i * BS + slot, A.c + i * ld + ee);
  }
  // own state row i: staged copy or (re-)read through L1
  auto cown = [&](int i) { return CSM ? s_c[i * BS + slot] : ldv(A.c + i * ld + e); };
  const double t = A.t_dev ? A.t_dev[0] + A.toff * A.t_dev[1] : A.t;
  const double dt = A.t_dev ? A.t_dev[1] : A.dt;
  const double det = det2(B11, B12, B21, B22), isd = rsqrt_fast(det), sd = det * isd, idet = isd * isd;
  // out-of-block neighbour requests, (neighbour, its edge) codes in per-warp
  // slot ranges (ballot prefix, no shared counter); hs[j] = slot or -1
  constexpr int NW = BS / 32;
  const int WC = HC / NW;
  int* s_cnt = s_req + HC;  // [NW] requests per warp
  int hs[3] = {-1, -1, -1};
  // MMS phase-offset table to shared memory (made visible by the barrier
  // after phase A2, before the source terms)
  const double* su = nullptr;
  if constexpr (k <= 2 && !(V & V_TAY7)) {
    if ((V & V_UNI) || ((V & V_FC) && T.uni != nullptr)) {
      for (int i = slot; i < NU; i += BS) cp_async8(s_U + i, T.uni + i);  // waited before the barrier after A2
      su = s_U;
    }
  }
  if (edges) {
    for (int i = slot; i < 3 * K * NT; i += BS) s_L[i] = s_tab[TB::L + i];
    const int lane = slot & 31, w = slot >> 5;
    int base = 0;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int nb = code[j] >> 2;
      const bool req = active && code[j] >= 0 && ((code[j] & 3) == HALO_J || nb < blo || nb >= bhi);
      const unsigned m = __ballot_sync(0xffffffffu, req);
      const int pos = base + __popc(m & ((1u << lane) - 1u));
      if (req && pos < WC) {
        s_req[w * WC + pos] = code[j];
        hs[j] = w * WC + pos;
      }
      base += __popc(m);
    }
    if (lane == 0) s_cnt[w] = min(base, WC);
  }
  // phase A2 work items: (request, field) pairs in request order; item `it`
  // -> request slot / field
  auto item = [&](int it, int& hsl, int& fi) {
    int le = it / NF, w = 0;
    fi = it - NF * le;
    while (w < NW - 1 && le >= s_cnt[w]) le -= s_cnt[w++];
    hsl = w * WC + le;
  };
  auto a2_trace = [&](int hsl, int fi, const double* f, const double* g4) {
    if ((NF == 6 && fi == 5) || (s_req[hsl] & 3) == HALO_J) {  // copied (static h_b, halo row)
#pragma unroll
      for (int a = 0; a < NT; ++a) s_ht[(fi * NT + a) * HC + hsl] = f[a];
      return;
    }
    const int cd = s_req[hsl], jn = cd & 3;
    const double nisd = rsqrt_fast(det2(g4[0], g4[1], g4[2], g4[3]));
    const double* L = s_L + jn * K * NT;
#pragma unroll
    for (int a = 0; a < NT; ++a) {
      double acc = 0.0;
#pragma unroll
      for (int i = 0; i < K; ++i) acc = __fma_rn(L[i * NT + a], f[i], acc);
      s_ht[(fi * NT + a) * HC + hsl] = __dmul_rn(acc, nisd);
    }
  };
  auto a2_load = [&](int hsl, int fi, double* f, double* g4) {
    const int nb = s_req[hsl] >> 2;
    const int jn = s_req[hsl] & 3;
    if (jn == HALO_J) {  // row nb of the halo trace table (another partition's element)
#pragma unroll
      for (int a = 0; a < NT; ++a) f[a] = ldg(A.ht + (int64_t)nb * 6 * NT + fi * NT + a);
      return;
    }
    if (NF == 6 && fi == 5) {
#pragma unroll
      for (int a = 0; a < NT; ++a) f[a] = ldg(T.hbt + (jn * NT + a) * ld + nb);
      return;
    }
    const double* src = fi < 3 ? A.c + (int64_t)fi * K * ld : A.u + (int64_t)(fi - 3) * K * ld;
#pragma unroll
    for (int i = 0; i < K; ++i) f[i] = ldg(src + i * ld + nb);
#pragma unroll
    for (int i = 0; i < 4; ++i) g4[i] = ldg(T.geo + i * ld + nb);
  };
  int nit = 0;
  // k <= 2: the first A2 item's loads are issued before phase A (one exposed
  // memory latency per block instead of two)
  constexpr bool PF = k <= 2;
  double pf[PF ? K : 1], pg[4];
  int p_h = 0, p_f = 0;
  if (edges) {
    __syncthreads();
#pragma unroll
    for (int w = 0; w < NW; ++w) nit += NF * s_cnt[w];
    if constexpr (PF) {
      if (slot < nit) {
        item(slot, p_h, p_f);
        a2_load(p_h, p_f, pf, pg);
      }
    }
  }

  if (edges && active) {
    // phase A: own trace moments on all three local edges -> shared memory
    double t3[NT], fl[PRE ? 1 : K];
#pragma unroll
    for (int fi = 0; fi < NF; ++fi) {  // (fi = 5: P1 h_b, as qf_static computes it)
      const double* f;
      if constexpr (PRE) {
        f = own_f + fi * K;
      } else {
        if (CSM && fi == 0) cp_async_wait_all();
        if (CSM && fi < 3) {
#pragma unroll
          for (int i = 0; i < K; ++i) fl[i] = s_c[(fi * K + i) * BS + slot];
        } else {
          const double* src = fi < 3 ? A.c + (int64_t)fi * K * ld : A.u + (int64_t)(fi - 3) * K * ld;
#pragma unroll
          for (int i = 0; i < K; ++i) fl[i] = ldv(src + i * ld + e);
        }
        f = fl;
      }
      O::trace0(f, t3);
#pragma unroll
      for (int a = 0; a < NT; ++a) s_tr[((0 * NF + fi) * NT + a) * BS + slot] = __dmul_rn(t3[a], isd);
      O::trace1(f, t3);
#pragma unroll
      for (int a = 0; a < NT; ++a) s_tr[((1 * NF + fi) * NT + a) * BS + slot] = __dmul_rn(t3[a], isd);
      O::trace2(f, t3);
#pragma unroll
      for (int a = 0; a < NT; ++a) s_tr[((2 * NF + fi) * NT + a) * BS + slot] = __dmul_rn(t3[a], isd);
    }
  }
  if (edges) {
    // phase A2: traces of out-of-block neighbours on the shared edge (same
    // rounding sequence as the owner's phase A), instead of divergent
    // gathers inside the edge loop
    int it0 = slot;
    if constexpr (PF) {
      if (slot < nit) a2_trace(p_h, p_f, pf, pg);
      it0 += BS;
    }
    for (int it = it0; it < nit; it += BS) {
      int hsl, fi;
      double f[K], g4[4];
      item(it, hsl, fi);
      a2_load(hsl, fi, f, g4);
      a2_trace(hsl, fi, f, g4);
    }
  }
  if constexpr (k <= 2 && !(V & V_TAY7)) {
    if (su) cp_async_wait_all();  // MMS phase-offset table
  }
  if constexpr (CSM) cp_async_wait_all();  // (phase A may not have run: rhs without edges)
  __syncthreads();
  if (!active) return;

  double r[3 * K];
#pragma unroll
  for (int i = 0; i < 3 * K; ++i) r[i] = 0.0;
  // own data: still in registers from the prologue when edges are on
  // (u is an operand of the volume terms only, which k >= 3 takes from A.vol)
  double c[3 * K], u[k <= 2 ? 2 * K : 1], hb[K];
#pragma unroll
  for (int i = 0; i < 3 * K; ++i)
    c[i] = (PRE && edges) ? own_f[PRE ? i : 0] : cown(i);
  if constexpr (k <= 2) {
#pragma unroll
    for (int i = 0; i < 2 * K; ++i)
      u[i] = (PRE && edges) ? own_f[PRE ? 3 * K + i : 0] : ldv(A.u + i * ld + e);
  }
#pragma unroll
  for (int i = 0; i < K; ++i)
    hb[i] = (PRE && edges) ? own_f[PRE ? 5 * K + i : 0] : (i < NH ? ldv(T.hb + i * ld + e) : 0.0);
  const double* xi = c;
  const double* cU = c + K;
  const double* cV = c + 2 * K;

  if constexpr (k <= 2) {
    if (QF_EN_VOL && ((V & V_STG) || (A.terms & TERM_VOL)))
      volume_terms<k, V>(P, B11, B12, B21, B22, isd, idet, xi, cU, cV, u, hb, r);
  } else if constexpr (FuseVol<k>::value) {  // k >= 3 volume terms in this kernel
    if ((V & V_STG) || (A.terms & TERM_VOL)) {
      double uu[2 * K];
#pragma unroll
      for (int i = 0; i < 2 * K; ++i) uu[i] = ldv(A.u + i * ld + e);
      volume_terms<k, V>(P, B11, B12, B21, B22, isd, idet, xi, cU, cV, uu, hb, r);
    }
  } else if (A.vol) {  // k >= 3: computed by volume_kernel (register pressure)
#pragma unroll
    for (int i = 0; i < 3 * K; ++i) r[i] += ldg(A.vol + i * ld + e);
  }
  if (QF_EN_SRC && ((V & V_STG) || (A.terms & TERM_SRC))) {  // solver.py:708-725 (+ xi mass source)
    double d1, d2;
    O::hb_dref(hb, d1, d2);
    const double i32 = idet * isd;
    const double gx = P.g * (B22 * d1 - B21 * d2) * i32, gy = P.g * (-B12 * d1 + B11 * d2) * i32;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if constexpr ((V & V_FRIC) != 0) {
        r[K + i] += -P.tau * cU[i] + P.fc * cV[i] + gx * xi[i];
        r[2 * K + i] += -P.tau * cV[i] - P.fc * cU[i] + gy * xi[i];
      } else {  // tau = f_c = 0
        r[K + i] += __dmul_rn(gx, xi[i]);
        r[2 * K + i] += __dmul_rn(gy, xi[i]);
      }
    }
    if (A.frc) {  // user scenario: forcing rows projected by its own module (qf_user.cuh)
#pragma unroll
      for (int i = 0; i < 2 * K; ++i) r[K + i] += ldg(A.frc + i * ld + e);
    }
    if ((V & V_FC) && P.forcing) {  // sqrt(detB) sum_q w_q phi_p(q) F(x_q, t), reference :719-724
      forcing_quad<k, V>(P, T, e, t, B11, B12, B21, B22, sd, su,
                      [&](const double* Pq, double S, double Fx, double Fy) {
#pragma unroll
                        for (int p = 0; p < K; ++p) {
                          const double w = Pq[p];
                          r[p] = fma(w, S, r[p]);
                          r[K + p] = fma(w, Fx, r[K + p]);
                          r[2 * K + p] = fma(w, Fy, r[2 * K + p]);
                        }
                      });
    }
  }
  if (QF_EN_EDGE && edges) {  // reference solver.py:561-706
    constexpr int EUN = (k <= QF_EUNROLL_MAXK || (QF_EUNROLL_FC2 && k == 2 && (V & V_FC) && (V & V_STG))) ? 3 : QF_EUNROLL;
#pragma unroll EUN
    for (int j = 0; j < 3; ++j)
      edge_term<k, Blk<k>::value, V>(T, P, A, e, j, code[j], slot, blo, bhi, s_tr, s_ht, hs[j], HC, B11, B12, B21,
                   B22, isd, r);
  }
  if (!(V & V_STG) && A.mode == 0) {
#pragma unroll
    for (int i = 0; i < 3 * K; ++i) A.c_out[i * ld + e] = r[i];
    return;
  }
  // SSP-RK combination (solver.py:756-764) and velocity of the new state
  bool fin = true;
#pragma unroll
  for (int i = 0; i < 3 * K; ++i) {
    double v = cown(i) + dt * r[i];
    v = A.a != 0.0 ? fma(A.a, ldg(A.c0 + i * ld + e), A.b * v) : A.b * v;
    c[i] = v;
    fin = fin && isfinite(v);
  }
#pragma unroll
  for (int i = 0; i < 3 * K; ++i) A.c_out[i * ld + e] = c[i];
  if (!fin) atomicOr(A.err, BIT_NONFINITE);
  if constexpr (k >= QF_VSPLIT) return;  // velocity_kernel follows (register pressure)
  double H[K], uo[K], vo[K];
#pragma unroll
  for (int i = 0; i < K; ++i) H[i] = c[i] + hb[i];
  if (!O::vel_solve(H, c + K, c + 2 * K, sd, uo, vo)) atomicOr(A.err, BIT_SINGULAR);
#pragma unroll
  for (int i = 0; i < K; ++i) {
    A.u_out[i * ld + e] = uo[i];
    A.u_out[(K + i) * ld + e] = vo[i];
  }
  if constexpr ((V & V_PUSH) != 0) {
    if (A.push) push_traces<k>(T, A.push, A.peers, ld, e, A.c_out, uo, vo);
  }
}

// k >= 3: the volume contraction as its own launch (the fused stage kernel
// would otherwise spill its K^3-operand working set); writes vol[3K][ld].
// strided, scaled read-only view of one state row: v[i] = s * p[i * ld]
struct GRow {
  const double* p;
  int64_t ld;
  double s;
  __device__ __forceinline__ double operator[](int i) const { return s * ldv(p + i * ld); }
};

// a row of the block's shared-memory copy of c (stride = block size)
struct SRow {
  const double* p;
  double s;
  __device__ __forceinline__ double operator[](int i) const { return s * p[i * 128]; }
};


// k >= 4: the volume kernel copies its element's 3K state rows into shared
// memory with one burst of cp.async (no registers held, every load in flight
// at once) instead of the generated code's in-loop global loads (ncu: long
// scoreboard was the top stall at 2 warps per scheduler)
#ifndef QF_VSMEM
#define QF_VSMEM 1
#endif

// minimum resident volume_kernel blocks per SM (register cap): k = 4 with 3
// (168 registers) 902 -> 875 us/stage at N = 512; k = 3 with 3: 352 -> 392 us
#ifndef QF_VOCC
#define QF_VOCC 1
#endif
#ifndef QF_VOCC4
#define QF_VOCC4 3
#endif
#ifndef QF_VOCC4G0  // k = 4 output group 0 (the larger one): 2 blocks/SM, no spills
#define QF_VOCC4G0 2    // (858 -> 848 us per k = 4 stage at N = 512 against 3 blocks/SM)
#endif
template <int k, int GRP = 0, bool HBC = true>  // HBC: hb_mode "const" code compiled
__global__ void __launch_bounds__(128, k == 4 ? (GRP == 0 ? QF_VOCC4G0 : QF_VOCC4) : QF_VOCC) volume_kernel(Tab T, Phys P, const double* __restrict__ c,
                                                     const double* __restrict__ u, int e0, int n,
                                                     double* __restrict__ vol) {
  using O = Ord<k>;
  constexpr int K = O::K, NH = O::NH;
  const int e = e0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= e0 + n) return;
  const int64_t ld = T.ld;
  const double B11 = ldg(T.geo + e), B12 = ldg(T.geo + ld + e);
  const double B21 = ldg(T.geo + 2 * ld + e), B22 = ldg(T.geo + 3 * ld + e);
  const double det = det2(B11, B12, B21, B22), isd = rsqrt_fast(det), idet = isd * isd;
  const double i32 = idet * isd, g = P.g;
  if constexpr (k == 3 && VGroups<k>::value == 1) {  // measured: row-outer is faster at k = 3
    double cc[3 * K], uu[2 * K], hb[K], r[3 * K];
#pragma unroll
    for (int i = 0; i < 3 * K; ++i) cc[i] = ldg(c + i * ld + e);
#pragma unroll
    for (int i = 0; i < 2 * K; ++i) uu[i] = ldg(u + i * ld + e);
#pragma unroll
    for (int i = 0; i < K; ++i) hb[i] = i < NH ? ldg(T.hb + i * ld + e) : 0.0;
#pragma unroll
    for (int i = 0; i < 3 * K; ++i) r[i] = 0.0;
    volume_terms<k, HBC ? V_GENERAL : 0>(P, B11, B12, B21, B22, isd, idet, cc, cc + K, cc + 2 * K,
                                         uu, hb, r);
#pragma unroll
    for (int i = 0; i < 3 * K; ++i) vol[i * ld + e] = r[i];
    return;
  }
  constexpr int VG = VGroups<k>::value, grp = GRP;
  constexpr int P0 = VG == 1 ? 0 : (VG == 2 ? O::VOL_PSPLIT2[grp] : (VG == 3 ? O::VOL_PSPLIT3[grp]
                                                                               : O::VOL_PSPLIT4[grp]));
  constexpr int P1 = VG == 1 ? K : (VG == 2 ? O::VOL_PSPLIT2[grp + 1]
                                            : (VG == 3 ? O::VOL_PSPLIT3[grp + 1]
                                                       : O::VOL_PSPLIT4[grp + 1]));
  constexpr bool SM = QF_VSMEM && k >= 4;
  __shared__ double vsm[SM ? 3 * K * 128 : 1];
  if constexpr (SM) {
#pragma unroll
    for (int i = 0; i < 3 * K; ++i) cp_async8(vsm + i * 128 + threadIdx.x, c + i * ld + e);
  }
  double r[3 * K], al[K], be[K], wv[K];
  {  // xi row and the U/V operands a, b, w
    double cU[K], cV[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      cU[i] = ldg(c + (K + i) * ld + e);
      cV[i] = ldg(c + (2 * K + i) * ld + e);
      al[i] = B22 * cU[i] - B12 * cV[i];
      be[i] = -B21 * cU[i] + B11 * cV[i];
    }
    O::vol_xi(al, be, r);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      r[i] *= idet;
      r[K + i] = 0.0;
      r[2 * K + i] = 0.0;
      const double uu = ldg(u + i * ld + e), uv = ldg(u + (K + i) * ld + e);
      al[i] = B22 * uu - B12 * uv;
      be[i] = -B21 * uu + B11 * uv;
      wv[i] = 0.5 * ldg(c + i * ld + e) + (P.hb_linear && i < NH ? ldg(T.hb + i * ld + e) : 0.0);
    }
  }
  const GRow gU{c + K * ld + e, ld, i32}, gV{c + 2 * K * ld + e, ld, i32}, gX{c + e, ld, i32};
  if constexpr (SM) {  // advection part from the shared copy, then symmetric-product pressure rows
    cp_async_wait_all();
    const double* sc = vsm + threadIdx.x;
    const SRow sU{sc + K * 128, i32}, sV{sc + 2 * K * 128, i32}, sX{sc, i32};
    O::template vol_uv_acc<P0, P1, !QF_VPRESS>(sU, sV, sX, al, be, wv, g * B22, g * B21, g * B12,
                                               g * B11, r + K, r + 2 * K);
    if constexpr (QF_VPRESS) {
      double xi[K], hb[NH];
#pragma unroll
      for (int i = 0; i < K; ++i) xi[i] = sc[i * 128];
#pragma unroll
      for (int i = 0; i < NH; ++i) hb[i] = ldg(T.hb + i * ld + e);
      const double gs = g * i32;
      O::template vol_press<P0, P1>(xi, hb, P.hb_linear != 0, gs * B22, gs * B21, gs * B12,
                                    gs * B11, r + K, r + 2 * K);
    }
  } else if constexpr (QF_VPRESS && k >= 4) {  // advection part, then symmetric-product pressure rows
    O::template vol_uv_acc<P0, P1, false>(gU, gV, gX, al, be, wv, g * B22, g * B21, g * B12,
                                          g * B11, r + K, r + 2 * K);
    double xi[K], hb[NH];
#pragma unroll
    for (int i = 0; i < K; ++i) xi[i] = ldv(c + i * ld + e);
#pragma unroll
    for (int i = 0; i < NH; ++i) hb[i] = ldg(T.hb + i * ld + e);
    const double gs = g * i32;
    O::template vol_press<P0, P1>(xi, hb, P.hb_linear != 0, gs * B22, gs * B21, gs * B12,
                                  gs * B11, r + K, r + 2 * K);
  } else {
    O::template vol_uv_acc<P0, P1>(gU, gV, gX, al, be, wv, g * B22, g * B21, g * B12, g * B11,
                                   r + K, r + 2 * K);
  }
  if (HBC && !P.hb_linear) {  // paper-form constant h_b (solver.py:498-510)
    double xi[K], ra[K], rb[K];
#pragma unroll
    for (int i = 0; i < K; ++i) xi[i] = ldg(c + i * ld + e);
    const double ghb = g * ldg(T.hb + e) * isd * 0.7071067811865476 * idet;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      al[i] = B22 * xi[i];
      be[i] = -B21 * xi[i];
    }
    O::vol_xi(al, be, ra);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      al[i] = -B12 * xi[i];
      be[i] = B11 * xi[i];
    }
    O::vol_xi(al, be, rb);
#pragma unroll
    for (int i = P0; i < P1; ++i) {
      r[K + i] += ghb * ra[i];
      r[2 * K + i] += ghb * rb[i];
    }
  }
  if constexpr (grp == 0) {
#pragma unroll
    for (int i = 0; i < K; ++i) vol[i * ld + e] = r[i];
  }
#pragma unroll
  for (int i = P0; i < P1; ++i) {
    vol[(K + i) * ld + e] = r[K + i];
    vol[(2 * K + i) * ld + e] = r[2 * K + i];
  }
}

// k >= 3 with QF_VMMA: the volume rows in two launches.
// volume_rest_kernel: xi row (vol_xi) and the pressure rows (vol_press,
// symmetric products) -- thread per element, plain FP64;
// vol_mma_kernel: the advection part of the U/V rows,
//   U_p += sum_i Z[p,i] c_U,i / (detB sqrt(detB)),  Z[p,i] = sum_m T1[p,i,m] a_m + T2[p,i,m] b_m
// (solver.py:459-482 factorised), as a GEMM on the FP64
// tensor cores: per tile of 8 elements D[el, (p, i)] = (a; b)[el, :] . T[:, (p, i)]
// with mma.sync.m8n8k4.f64 (the B fragments of T are the generated table
// Mma<k>::table(), all-zero fragments dropped), then the contraction with
// c_U / c_V in the accumulator registers and a quad reduction.  ncu on the
// thread-per-element kernel: 2 warps per scheduler at 255 registers, FP64
// pipe ~35 % busy on FFMA chains; one DMMA carries 256 multiply-adds.
// Measured (N = 512, bumps + walls): k = 4 stage 901 -> 1057 us, k = 3 352 ->
// 506 us.  vol_mma_kernel<4> 330 us with the DMMA pipe 54 % busy (long
// scoreboard: per-tile operand loads) + volume_rest_kernel 196..325 us, against
// ~480 us for the FFMA input-outer kernel pair: the contraction is bilinear in
// the element data, so the tensor cores only take the first (linear) half and
// the operand setup, pressure rows and an extra pass over the rows stay on
// the FP64 pipe they share with DMMA.  Off by default (opt-in experiment).
#ifndef QF_VMMA
#define QF_VMMA 0  // bit mask of orders (k = 3: 8, k = 4: 16)
#endif
#ifndef QF_VMMA_BPS
#define QF_VMMA_BPS 4  // resident vol_mma blocks per SM (persistent grid)
#endif
template <int k, bool HBC, bool ADD>  // ADD: U/V rows start from vol (vol_mma_kernel's advection)
__global__ void __launch_bounds__(128) volume_rest_kernel(Tab T, Phys P, const double* __restrict__ c,
                                                          int e0, int n, double* __restrict__ vol) {
  using O = Ord<k>;
  constexpr int K = O::K, NH = O::NH;
  const int e = e0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= e0 + n) return;
  const int64_t ld = T.ld;
  const double B11 = ldg(T.geo + e), B12 = ldg(T.geo + ld + e);
  const double B21 = ldg(T.geo + 2 * ld + e), B22 = ldg(T.geo + 3 * ld + e);
  const double det = det2(B11, B12, B21, B22), isd = rsqrt_fast(det), idet = isd * isd;
  const double i32 = idet * isd, g = P.g;
  double r[3 * K], xi[K], hb[NH];
  {
    double al[K], be[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const double cU = ldg(c + (K + i) * ld + e), cV = ldg(c + (2 * K + i) * ld + e);
      al[i] = B22 * cU - B12 * cV;
      be[i] = -B21 * cU + B11 * cV;
    }
    O::vol_xi(al, be, r);
  }
#pragma unroll
  for (int i = 0; i < K; ++i) {
    r[i] *= idet;
    r[K + i] = 0.0;
    r[2 * K + i] = 0.0;
    xi[i] = ldg(c + i * ld + e);
  }
#pragma unroll
  for (int i = 0; i < NH; ++i) hb[i] = ldg(T.hb + i * ld + e);
  const double gs = g * i32;
  O::template vol_press<0, K>(xi, hb, P.hb_linear != 0, gs * B22, gs * B21, gs * B12, gs * B11,
                              r + K, r + 2 * K);
  if (HBC && !P.hb_linear) {  // paper-form constant h_b (solver.py:498-510)
    double al[K], be[K], ra[K], rb[K];
    const double ghb = g * hb[0] * isd * 0.7071067811865476 * idet;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      al[i] = B22 * xi[i];
      be[i] = -B21 * xi[i];
    }
    O::vol_xi(al, be, ra);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      al[i] = -B12 * xi[i];
      be[i] = B11 * xi[i];
    }
    O::vol_xi(al, be, rb);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      r[K + i] += ghb * ra[i];
      r[2 * K + i] += ghb * rb[i];
    }
  }
#pragma unroll
  for (int i = 0; i < 3 * K; ++i) vol[i * ld + e] = (ADD && i >= K) ? vol[i * ld + e] + r[i] : r[i];
}

template <int k>
struct MmaIn {  // raw loads of one element tile (prefetched one iteration ahead)
  static constexpr int NKS = Mma<k>::NKS, NCH = Mma<k>::NCH;
  double b11, b12, b21, b22, uu[NKS], uv[NKS], cu[2 * NCH], cv[2 * NCH];
  __device__ __forceinline__ void load(const Tab& T, const double* __restrict__ c,
                                       const double* __restrict__ u, int e, int q) {
    constexpr int K = Mma<k>::K;
    const int64_t ld = T.ld;
    b11 = ldg(T.geo + e);
    b12 = ldg(T.geo + ld + e);
    b21 = ldg(T.geo + 2 * ld + e);
    b22 = ldg(T.geo + 3 * ld + e);
#pragma unroll
    for (int s = 0; s < NKS; ++s) {  // (a; b)[4 s + q] needs u_m, v_m, m = (4 s + q) mod K
      const int kk = 4 * s + q, m = kk >= K ? kk - K : kk;
      uu[s] = kk < 2 * K ? ldg(u + m * ld + e) : 0.0;
      uv[s] = kk < 2 * K ? ldg(u + (K + m) * ld + e) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < 2 * NCH; ++j) {  // inputs 8 ch + 2 q + (j & 1)
      const int i = 8 * (j >> 1) + 2 * q + (j & 1);
      cu[j] = i < K ? ldg(c + (K + i) * ld + e) : 0.0;
      cv[j] = i < K ? ldg(c + (2 * K + i) * ld + e) : 0.0;
    }
  }
};

// writes the advection part of the U/V rows [K, 3K) of vol (volume_rest_kernel<k, .., true>
// then adds the xi row and the pressure)
#ifndef QF_VMMA_MINB
#define QF_VMMA_MINB 3
#endif
template <int k>
__global__ void __launch_bounds__(128, QF_VMMA_MINB) vol_mma_kernel(Tab T, const double* __restrict__ c,
                                                      const double* __restrict__ u, int e0, int n,
                                                      double* __restrict__ vol) {
  using M = Mma<k>;
  constexpr int K = M::K, NKS = M::NKS, NCH = M::NCH, NT = 1;
  extern __shared__ double sB[];
  for (int i = threadIdx.x; i < M::NF * 32; i += blockDim.x) sB[i] = M::table()[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, q = lane & 3, row = lane >> 2;
  const int64_t ld = T.ld;
  const int ngrp = (n + 7) / 8, stride = gridDim.x * 4;
  int grp = blockIdx.x * 4 + (threadIdx.x >> 5);
  auto elem = [&](int g) { const int loc = g * 8 + row; return e0 + (loc < n ? loc : n - 1); };
  MmaIn<k> nx;
  if (grp < ngrp) nx.load(T, c, u, elem(grp), q);
  for (; grp < ngrp; grp += stride) {
    const MmaIn<k> in = nx;
    const int e = elem(grp);
    if (grp + stride < ngrp) nx.load(T, c, u, elem(grp + stride), q);
    const double det = det2(in.b11, in.b12, in.b21, in.b22), isd = rsqrt_fast(det);
    const double i32 = isd * isd * isd;
    double A[NT][NKS], cu[NT][2 * NCH], cv[NT][2 * NCH], pu[NT][K], pv[NT][K];
#pragma unroll
    for (int s = 0; s < NKS; ++s)  // a = B22 u - B12 v, b = -B21 u + B11 v
      A[0][s] = 4 * s + q < K ? in.b22 * in.uu[s] - in.b12 * in.uv[s]
                              : -in.b21 * in.uu[s] + in.b11 * in.uv[s];
#pragma unroll
    for (int j = 0; j < 2 * NCH; ++j) {
      cu[0][j] = i32 * in.cu[j];
      cv[0][j] = i32 * in.cv[j];
    }
#pragma unroll
    for (int p = 0; p < K; ++p) {
      pu[0][p] = 0.0;
      pv[0][p] = 0.0;
    }
    M::template adv<NT>(sB, lane, A, cu, cv, pu, pv);
    const bool live = grp * 8 + row < n;
#pragma unroll
    for (int p = 0; p < K; ++p) {
      double su = pu[0][p], sv = pv[0][p];
      su += __shfl_xor_sync(0xffffffffu, su, 1);
      sv += __shfl_xor_sync(0xffffffffu, sv, 1);
      su += __shfl_xor_sync(0xffffffffu, su, 2);
      sv += __shfl_xor_sync(0xffffffffu, sv, 2);
      if (live && (p & 3) == q) {
        vol[(K + p) * ld + e] = su;
        vol[(2 * K + p) * ld + e] = sv;
      }
    }
  }
}

#ifndef QF_VELOCC4
#define QF_VELOCC4 1
#endif
#ifndef QF_VLAZY
#define QF_VLAZY 4
#endif
// strided read-only view of one state row, read on use
struct QRow {
  const double* p;
  int64_t ld;
  __device__ __forceinline__ double operator[](int i) const { return ldv(p + i * ld); }
};
#ifndef QF_VELOCC3
#define QF_VELOCC3 3  // k = 3 velocity at 168 registers: 358 -> 350 us/stage (N = 512)
#endif
template <int k, bool PUSH = false>  // PUSH: fused halo push compiled
__global__ void __launch_bounds__(128, k == 4 ? QF_VELOCC4 : (k == 3 ? QF_VELOCC3 : 1))
    velocity_kernel(Tab T, const double* __restrict__ c, double* __restrict__ u, int e0, int n,
                    unsigned* err, const int* __restrict__ push = nullptr,
                    const qf_peer* __restrict__ peers = nullptr) {
  using O = Ord<k>;
  if constexpr (((QF_SMEMSPILL_VEL >> k) & 1) != 0) asm volatile(".pragma \"enable_smem_spilling\";");
  constexpr int K = O::K, NH = O::NH;
  const int e = e0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= e0 + n) return;
  const int64_t ld = T.ld;
  const double B11 = ldg(T.geo + e), B12 = ldg(T.geo + ld + e);
  const double B21 = ldg(T.geo + 2 * ld + e), B22 = ldg(T.geo + 3 * ld + e);
  const double sd = sqrt(det2(B11, B12, B21, B22));
  // k >= QF_VLAZY: the U, V rows are read where the forward substitution
  // first needs them instead of being held through the factorisation
  constexpr bool LAZY = k >= QF_VLAZY;
  constexpr int NC = LAZY ? K : 3 * K;
  double cc[NC], hb[K], uo[K], vo[K];
#pragma unroll
  for (int i = 0; i < NC; ++i) cc[i] = ldg(c + i * ld + e);
#pragma unroll
  for (int i = 0; i < K; ++i) hb[i] = i < NH ? ldg(T.hb + i * ld + e) : 0.0;
  double H[K];
#pragma unroll
  for (int i = 0; i < K; ++i) H[i] = cc[i] + hb[i];
  bool ok;
  if constexpr (LAZY) {
    const QRow qu{c + K * ld + e, ld}, qv{c + 2 * K * ld + e, ld};
    ok = O::vel_solve(H, qu, qv, sd, uo, vo);
  } else {
    ok = O::vel_solve(H, cc + K, cc + 2 * K, sd, uo, vo);
  }
  if (!ok) atomicOr(err, BIT_SINGULAR);
#pragma unroll
  for (int i = 0; i < K; ++i) {
    u[i * ld + e] = uo[i];
    u[(K + i) * ld + e] = vo[i];
  }
  if constexpr (PUSH) push_traces<k>(T, push, peers, ld, e, c, uo, vo);
}

// Dirichlet ghost data: exact (xi, U, V, u, v) at the k+2 Gauss points of
// every Dirichlet edge and (H, |u.n|) at the lambda samples (reference
// solver.py:395-402, 636-653; the pinv(E) projection of :649-653 reduces to
// the Gauss moments, taken in the stage kernel).  One thread per
// (stage, slot, point); all stages of a step in one launch (the data depend
// on time only).
template <int k>
__global__ void ghost_kernel(Tab T, Phys P, const int* __restrict__ bel,
                             const int* __restrict__ bloc, int nb, int nstage, double t0,
                             const double* t_dev, double3 toffs, double* ghost) {
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
  double xi, U, V;
  exact3(P, x, y, t, xi, U, V);
  const double H = hb_exact(P, x, y) + xi;
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

// Device-side setup: L2 projection of the initial state
// and of the bathymetry onto the normalised basis at the reference's
// degree-(2k+2) collapsed Gauss points (solver.py:139-168, 282-303), for
// meshes too large for the host NumPy path.  Field program `prog`:
//   [0] hb kind (0: bilinear from Phys.p, 1: base + amp * sum sin(k.x + phi))
//   [1] init kind (0: scenario exact data at t = 0, 1: Gaussian bumps at rest)
//   [2] n_modes  [3] n_bumps  [4] base  [5] amp
//   then n_modes x (kx, ky, phi), then n_bumps x (A, sigma, cx, cy)
// After projecting, the projected depth is checked at the quadrature points
// (DryState if H < h_min, solver.py:305-311).
template <int k>
__global__ void project_kernel(Tab T, Phys P, const double* __restrict__ prog, int n,
                               double h_min, double* __restrict__ c, double* __restrict__ hb_out,
                               unsigned* err) {
  using O = Ord<k>;
  using TB = Tabs<k>;
  constexpr int K = O::K, NH = O::NH, NQ = O::NQ;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int64_t ld = T.ld;
  const double B11 = T.geo[e], B12 = T.geo[ld + e], B21 = T.geo[2 * ld + e], B22 = T.geo[3 * ld + e];
  const double a1x = T.geo[4 * ld + e], a1y = T.geo[5 * ld + e];
  const double sd = sqrt(det2(B11, B12, B21, B22));
  const int hk = (int)prog[0], ik = (int)prog[1], nm = (int)prog[2], nbmp = (int)prog[3];
  const double* modes = prog + 6;
  const double* bumps = modes + 3 * nm;
  double acc[4][K];
#pragma unroll
  for (int f = 0; f < 4; ++f)
#pragma unroll
    for (int p = 0; p < K; ++p) acc[f][p] = 0.0;
  const double* tab = TB::ptr();
  for (int q = 0; q < NQ; ++q) {
    const double x1 = tab[TB::QX + q], x2 = tab[TB::QY + q];
    const double x = a1x + B11 * x1 + B12 * x2, y = a1y + B21 * x1 + B22 * x2;
    double hbv;
    if (hk == 1) {
      double s = 0.0;
      for (int m = 0; m < nm; ++m) s += sin(modes[3 * m] * x + modes[3 * m + 1] * y + modes[3 * m + 2]);
      hbv = prog[4] + prog[5] * s;
    } else {
      hbv = hb_exact(P, x, y);
    }
    double xi = 0.0, U = 0.0, V = 0.0;
    if (ik == 1) {
      for (int b = 0; b < nbmp; ++b) {
        const double dx = x - bumps[4 * b + 2], dy = y - bumps[4 * b + 3], s = bumps[4 * b + 1];
        xi += bumps[4 * b] * exp(-(dx * dx + dy * dy) / (2.0 * s * s));
      }
    } else {
      exact3(P, x, y, 0.0, xi, U, V);
    }
    const double v[4] = {xi, U, V, hbv};
#pragma unroll
    for (int p = 0; p < K; ++p) {
      const double w = tab[TB::P + q * K + p];
#pragma unroll
      for (int f = 0; f < 4; ++f) acc[f][p] = fma(w, v[f], acc[f][p]);
    }
  }
#pragma unroll
  for (int f = 0; f < 3; ++f)
#pragma unroll
    for (int p = 0; p < K; ++p) c[(f * K + p) * ld + e] = sd * acc[f][p];
#pragma unroll
  for (int p = 0; p < NH; ++p) hb_out[p * ld + e] = sd * acc[3][p];
  // projected depth at the quadrature points (P1 bathymetry + xi)
  bool dry = false;
  for (int q = 0; q < NQ; ++q) {
    double H = 0.0;
#pragma unroll
    for (int p = 0; p < K; ++p) {
      const double hbp = p < NH ? sd * acc[3][p] : 0.0;
      H = fma(hbp + sd * acc[0][p], tab[TB::PHI + q * K + p], H);
    }
    dry = dry || !(H / sd >= h_min);
  }
  if (dry) atomicOr(err, BIT_DRY);
}

// Static per-element-edge data derived from geometry and bathymetry:
// hbt[j*NT + a][e] = physical h_b trace moments on local edge j (the
// bathymetry part of every edge flux, read by both sides of the edge), and
// hbt[3*NT][e] = element-mean depth term of hb_mode="const".
template <int k>
__global__ void static_kernel(Tab T, int n, double* __restrict__ hbt) {
  using O = Ord<k>;
  constexpr int K = O::K, NT = O::NT, NH = O::NH;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int64_t ld = T.ld;
  const double isd = rsqrt_fast(det2(T.geo[e], T.geo[ld + e], T.geo[2 * ld + e], T.geo[3 * ld + e]));
  double f[K], t3[NT];
#pragma unroll
  for (int i = 0; i < K; ++i) f[i] = i < NH ? T.hb[i * ld + e] : 0.0;
  O::trace0(f, t3);
#pragma unroll
  for (int a = 0; a < NT; ++a) hbt[(0 * NT + a) * ld + e] = __dmul_rn(t3[a], isd);
  O::trace1(f, t3);
#pragma unroll
  for (int a = 0; a < NT; ++a) hbt[(1 * NT + a) * ld + e] = __dmul_rn(t3[a], isd);
  O::trace2(f, t3);
#pragma unroll
  for (int a = 0; a < NT; ++a) hbt[(2 * NT + a) * ld + e] = __dmul_rn(t3[a], isd);
  hbt[3 * NT * ld + e] = __dmul_rn(__dmul_rn(f[0], isd), 0.7071067811865476);
}

// Global L2 error against the scenario's exact solution (reference
// harness.py:81-98): per element
//   detB * sum_q w_q ((sum_p c[f][p] phi_p(q)) / sqrt(detB) - exact_f(x_q, t))^2
// for f = xi, U, V at the degree-(2k+2) collapsed rule; block sums in a fixed
// tree order, then one block adds the partials in block order, so the result
// is deterministic (independent of scheduling).
constexpr int L2_BS = 256;

template <int k>
__global__ void __launch_bounds__(L2_BS)
    l2err_kernel(Tab T, Phys P, const double* __restrict__ c, int e0, int n, double t,
                 double* __restrict__ part) {
  using O = Ord<k>;
  using TB = Tabs<k>;
  constexpr int K = O::K, NQ = O::NQ;
  __shared__ double s[3][L2_BS];
  const int tid = threadIdx.x, e = e0 + blockIdx.x * L2_BS + tid;
  double acc[3] = {0.0, 0.0, 0.0};
  if (e < e0 + n) {
    const int64_t ld = T.ld;
    const double B11 = T.geo[e], B12 = T.geo[ld + e], B21 = T.geo[2 * ld + e],
                 B22 = T.geo[3 * ld + e];
    const double a1x = T.geo[4 * ld + e], a1y = T.geo[5 * ld + e];
    const double det = det2(B11, B12, B21, B22), sd = sqrt(det);
    double cc[3 * K];
#pragma unroll
    for (int i = 0; i < 3 * K; ++i) cc[i] = c[i * ld + e];
    const double* tab = TB::ptr();
    for (int q = 0; q < NQ; ++q) {
      const double x1 = tab[TB::QX + q], x2 = tab[TB::QY + q];
      const double x = a1x + B11 * x1 + B12 * x2, y = a1y + B21 * x1 + B22 * x2;
      double ex[3];
      exact3(P, x, y, t, ex[0], ex[1], ex[2]);
      const double w = tab[TB::QW + q];
#pragma unroll
      for (int f = 0; f < 3; ++f) {
        double v = 0.0;
#pragma unroll
        for (int p = 0; p < K; ++p) v = fma(cc[f * K + p], tab[TB::PHI + q * K + p], v);
        const double d = v / sd - ex[f];
        acc[f] = fma(w, d * d, acc[f]);
      }
    }
#pragma unroll
    for (int f = 0; f < 3; ++f) acc[f] *= det;
  }
#pragma unroll
  for (int f = 0; f < 3; ++f) s[f][tid] = acc[f];
  __syncthreads();
  for (int h = L2_BS / 2; h > 0; h >>= 1) {
    if (tid < h) {
#pragma unroll
      for (int f = 0; f < 3; ++f) s[f][tid] += s[f][tid + h];
    }
    __syncthreads();
  }
  if (tid == 0) {
#pragma unroll
    for (int f = 0; f < 3; ++f) part[(int64_t)f * gridDim.x + blockIdx.x] = s[f][0];
  }
}

// sq[f] = sum over nb block partials (fixed order: strided per thread, tree)
__global__ void __launch_bounds__(L2_BS) l2sum_kernel(const double* __restrict__ part, int nb,
                                                      double* __restrict__ sq) {
  __shared__ double s[3][L2_BS];
  const int tid = threadIdx.x;
#pragma unroll
  for (int f = 0; f < 3; ++f) {
    double a = 0.0;
    for (int b = tid; b < nb; b += L2_BS) a += part[(int64_t)f * nb + b];
    s[f][tid] = a;
  }
  __syncthreads();
  for (int h = L2_BS / 2; h > 0; h >>= 1) {
    if (tid < h) {
#pragma unroll
      for (int f = 0; f < 3; ++f) s[f][tid] += s[f][tid + h];
    }
    __syncthreads();
  }
  if (tid == 0) {
#pragma unroll
    for (int f = 0; f < 3; ++f) sq[f] = s[f][0];
  }
}

__global__ void advance_time(double* t_dev) { t_dev[0] += t_dev[1]; }

// halo trace rows out[i][6][NT] of (element items[i] >> 2, local edge items[i] & 3)
template <int k>
__global__ void halo_trace_kernel(Tab T, const double* __restrict__ c, const double* __restrict__ u,
                                  const int* __restrict__ items, int n, double* __restrict__ out) {
  constexpr int K = Ord<k>::K, NT = Ord<k>::NT;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int e = items[i] >> 2, j = items[i] & 3;
  const int64_t ld = T.ld;
  double uo[K], vo[K];
#pragma unroll
  for (int p = 0; p < K; ++p) {
    uo[p] = u[p * ld + e];
    vo[p] = u[(K + p) * ld + e];
  }
  edge_traces6<k>(T, ld, e, j, c + e, uo, vo, out + (int64_t)i * 6 * NT, 1);
}

__global__ void pack_kernel(const double* __restrict__ aos, double* __restrict__ soa, int n, int F,
                            int K, int64_t ld, const int* __restrict__ perm) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int64_t src = perm ? perm[e] : e;
  for (int i = 0; i < F * K; ++i) soa[i * ld + e] = aos[src * F * K + i];
}

__global__ void unpack_kernel(const double* __restrict__ soa, double* __restrict__ aos, int n,
                              int F, int K, int64_t ld, const int* __restrict__ perm) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  const int64_t dst = perm ? perm[e] : e;
  for (int i = 0; i < F * K; ++i) aos[dst * F * K + i] = soa[i * ld + e];
}

__global__ void gather_kernel(const double* __restrict__ src, int64_t ld, const int* __restrict__ idx,
                              int n, int rows, double* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int s = idx[i];
  for (int r = 0; r < rows; ++r) dst[(int64_t)r * n + i] = src[r * ld + s];
}

__global__ void scatter_kernel(const double* __restrict__ src, const int* __restrict__ idx, int n,
                               int rows, double* __restrict__ dst, int64_t ld) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int d = idx[i];
  for (int r = 0; r < rows; ++r) dst[r * ld + d] = src[(int64_t)r * n + i];
}

__global__ void fill_kernel(double* buf, size_t n, double v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    buf[i] = v;
}

}  // namespace qf

// out-of-block neighbour requests of the busiest warp (blocks of BS slots
// aligned at slot 0): sizes the stage kernel's request area per mesh
template <int BS>
__global__ void request_count_kernel(const int* __restrict__ nbr, int64_t ld, int n,
                                     int* __restrict__ out) {
  const int e = blockIdx.x * BS + threadIdx.x;
  const int blo = blockIdx.x * BS, bhi = min(blo + BS, n);
  int c = 0;
  if (e < n) {
    for (int j = 0; j < 3; ++j) {
      const int code = nbr[j * ld + e], nb = code >> 2;
      c += code >= 0 && ((code & 3) == qf::HALO_J || nb < blo || nb >= bhi);
    }
  }
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) atomicMax(out, c);
}

// 1 in *out if any owned element has a reflective-wall edge (boundary code
// -1 - (2 slot + 1)): selects stage-kernel instances with the wall code
__global__ void wall_scan_kernel(const int* __restrict__ nbr, int64_t ld, int n,
                                 int* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  for (int j = 0; j < 3; ++j) {
    const int code = nbr[j * ld + e];
    if (code < 0 && ((-1 - code) & 1)) {
      *out = 1;
      return;
    }
  }
}

#ifndef QF_KERNELS_ONLY  // (tools/one_kernel.sh: a translation unit that instantiates single kernels)
// ===================================================================== ABI
using namespace qf;

struct qf_ctx {
  qf_desc d;
  Tab tab;
  Phys phys;
  unsigned* err;  // device error word
  int K, NT, block;
  int n_sm = 148;  // multiprocessors of the context's device (persistent grids)
  // cached run graph
  cudaGraphExec_t graph = nullptr;
  const void* gkey[4] = {nullptr, nullptr, nullptr, nullptr};
  int graph_launches = 0;
  cudaStream_t stream_hint = nullptr;
  double* vol = nullptr;  // k >= 3 volume-rhs scratch [3K][ld] (context-owned)
  int hcap = QF_HCAP;     // stage-kernel request slots per block (measured in qf_create)
  double* l2part = nullptr;  // qf_l2_error block partials [3][blocks] (grown on demand)
  bool walls = true;         // any reflective-wall boundary code in nbr (measured in qf_create)
  bool fits = false;         // busiest warp's requests fit hcap (whole-mesh launches never overflow)
  int l2cap = 0;
  int device = 0;            // CUDA device of the context (set around every entry point)
  // optional timing events recorded around each stage of step_impl (also
  // inside the captured run graph, as external event-record nodes)
  cudaEvent_t stage_ev[8] = {};
  int n_stage_ev = 0;
  // user scenario module (qf_user_scenario): Dirichlet data and forcing kernels
  cudaLibrary_t user_lib = nullptr;
  cudaKernel_t user_ghost = nullptr;
  cudaKernel_t user_forcing = nullptr;
  double* frc = nullptr;  // [2K][ld] forcing rows of the current stage
  const double* halo_ht = nullptr;  // halo trace table for qf_rhs / qf_stage (partitions)
};

// makes the context's device current for the duration of an entry point
// (restores the caller's device on exit)
struct DevGuard {
  int prev = -1;
  explicit DevGuard(const qf_ctx* x) {
    int cur = 0;
    if (x && cudaGetDevice(&cur) == cudaSuccess && cur != x->device && cudaSetDevice(x->device) == cudaSuccess)
      prev = cur;
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

static int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

static int cuda_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(QF_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return QF_OK;
}

#define QF_DISPATCH(order, FN, ...)        \
  switch (order) {                         \
    case 0: FN<0>(__VA_ARGS__); break;     \
    case 1: FN<1>(__VA_ARGS__); break;     \
    case 2: FN<2>(__VA_ARGS__); break;     \
    case 3: FN<3>(__VA_ARGS__); break;     \
    default: FN<4>(__VA_ARGS__); break;    \
  }

// one stage-kernel instance: the dynamic shared-memory opt-in once per instance
// (function attributes are per device: one opt-in bit per device ordinal;
// a failed opt-in is not recorded, so the launch below reports the error)
template <int k, int V>
static void stage_inst(qf_ctx* x, const StageArgs& a, cudaStream_t s, int grid, size_t smem) {
  static std::atomic<uint64_t> attr{0};
  const uint64_t bit = 1ull << (x->device & 63);
  if (!(attr.load() & bit)) {
    if (cudaFuncSetAttribute(stage_kernel<k, V>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)stage_smem_bytes<k>(QF_HCAP)) == cudaSuccess)
      attr.fetch_or(bit);
  }
  stage_kernel<k, V><<<grid, Blk<k>::value, smem, s>>>(x->tab, x->phys, a);
}

// one launch per output group (separate register allocation per group)
template <int k, bool HBC>
static void launch_volume(qf_ctx* x, const StageArgs& a, int vg, cudaStream_t s) {
  volume_kernel<k, 0, HBC><<<vg, 128, 0, s>>>(x->tab, x->phys, a.c, a.u, a.e0, a.n, x->vol);
  g_launches++;
  if constexpr (VGroups<k>::value > 1) {
    volume_kernel<k, 1, HBC><<<vg, 128, 0, s>>>(x->tab, x->phys, a.c, a.u, a.e0, a.n, x->vol);
    g_launches++;
  }
  if constexpr (VGroups<k>::value > 2) {
    volume_kernel<k, 2, HBC><<<vg, 128, 0, s>>>(x->tab, x->phys, a.c, a.u, a.e0, a.n, x->vol);
    g_launches++;
  }
  if constexpr (VGroups<k>::value > 3) {
    volume_kernel<k, 3, HBC><<<vg, 128, 0, s>>>(x->tab, x->phys, a.c, a.u, a.e0, a.n, x->vol);
    g_launches++;
  }
}

template <int k>
static void launch_stage(qf_ctx* x, const StageArgs& a_in, cudaStream_t s) {
  StageArgs a = a_in;
  if (x->user_forcing && ((a.terms & TERM_SRC) || a.mode == 1) && a.n > 0) {
    Tab tab = x->tab;
    const double* td = a.t_dev;
    double t0 = a.t, toff = a.toff;
    int e0 = a.e0, n = a.n;
    double* f = x->frc;
    void* args[] = {&tab, (void*)&td, &t0, &toff, &e0, &n, &f};
    cudaLaunchKernel((const void*)x->user_forcing, dim3((n + 127) / 128), dim3(128), args, 0, s);
    g_launches++;
    a.frc = x->frc;
  }
  if constexpr (k >= 3 && !FuseVol<k>::value) {
    if ((a.terms & TERM_VOL) && a.n > 0) {
      // one launch per input group (separate register allocation per group)
      const int vg = (a.n + 127) / 128;
      if constexpr (((QF_VMMA >> k) & 1) != 0) {
        const int ngrp = (a.n + 7) / 8;
        const int mg = std::min((ngrp + 3) / 4, x->n_sm * QF_VMMA_BPS);
        vol_mma_kernel<k><<<mg, 128, Mma<k>::NF * 32 * sizeof(double), s>>>(x->tab, a.c, a.u, a.e0,
                                                                           a.n, x->vol);
        if (x->phys.hb_linear)
          volume_rest_kernel<k, false, true><<<vg, 128, 0, s>>>(x->tab, x->phys, a.c, a.e0, a.n, x->vol);
        else
          volume_rest_kernel<k, true, true><<<vg, 128, 0, s>>>(x->tab, x->phys, a.c, a.e0, a.n, x->vol);
        g_launches += 2;
      } else {
        if (x->phys.hb_linear && ((QF_VLEAN_ORDERS >> k) & 1))
          launch_volume<k, false>(x, a, vg, s);
        else
          launch_volume<k, true>(x, a, vg, s);
      }
      a.vol = x->vol;
    }
  }
  constexpr int bs = Blk<k>::value;
  a.hcap = x->hcap;
  const size_t smem = stage_smem_bytes<k>(a.hcap);
  const int grid = (a.n + bs - 1) / bs;
  if (grid == 0) return;
  // the variant this problem needs, then the smallest compiled instance
  // that covers it (instances: see the switch).  The request-overflow path
  // is compiled out only for whole-mesh launches whose busiest warp fits the
  // request slots measured in qf_create (blocks then equal the measured ones).
  const Phys& P = x->phys;
  const bool ovf = !(x->fits && a.e0 == 0 && a.n == x->d.n_elem && ((QF_NOOVF_ORDERS >> k) & 1));
  int v = V_GENERAL;
  if (a.mflux) {
    v = V_MF | V_GENERAL;
  } else if (a.mode == 1 && !a.push && P.tau == 0.0 && P.fc == 0.0 &&
             ((QF_LEAN_INST >> k) & 1)) {
    v = (P.forcing ? V_FC : 0) | (x->d.n_bnd > 0 ? V_DIR : 0) | (P.hb_linear ? 0 : V_HBC) |
        (x->walls ? V_WALL : 0) | (ovf ? V_OVF : 0) | V_STG;
    if (P.forcing && P.kind == SCN_MMS) {
      if (k <= 2 && x->tab.uni) v |= V_UNI;
      else if (P.taylor == 2) v |= V_TAY7;
    }
  }
  if constexpr (k <= 2) {  // BASELINE MMS on a uniform split-square mesh (C1, C2)
    if (v == (V_STG | V_FC | V_DIR | V_UNI)) {
      stage_inst<k, V_STG | V_FC | V_DIR | V_UNI>(x, a, s, grid, smem);
      g_launches++;  // (k <= 2: no velocity launch follows)
      return;
    }
    if (v == (V_STG | V_FC | V_DIR | V_UNI | V_OVF)) {
      stage_inst<k, V_STG | V_FC | V_DIR | V_UNI | V_OVF>(x, a, s, grid, smem);
      g_launches++;  // (k <= 2: no velocity launch follows)
      return;
    }
  }
  switch (v) {
    case V_STG | V_FC | V_DIR | V_TAY7:  // BASELINE MMS at small element size (C2)
      stage_inst<k, V_STG | V_FC | V_DIR | V_TAY7>(x, a, s, grid, smem);
      break;
    case V_STG | V_FC | V_DIR | V_TAY7 | V_OVF:
      stage_inst<k, V_STG | V_FC | V_DIR | V_TAY7 | V_OVF>(x, a, s, grid, smem);
      break;
    case V_STG | V_FC | V_DIR:  // MMS / travelling wave, Dirichlet only (C1)
      stage_inst<k, V_STG | V_FC | V_DIR>(x, a, s, grid, smem);
      break;
    case V_STG | V_FC | V_DIR | V_OVF:
      stage_inst<k, V_STG | V_FC | V_DIR | V_OVF>(x, a, s, grid, smem);
      break;
    case V_STG | V_WALL:  // reflective walls, no forcing (C3-C5)
      stage_inst<k, V_STG | V_WALL>(x, a, s, grid, smem);
      break;
    case V_STG | V_WALL | V_OVF:  // (k = 1, 4 and partition ranges)
      stage_inst<k, V_STG | V_WALL | V_OVF>(x, a, s, grid, smem);
      break;
    case V_MF | V_GENERAL:
      stage_inst<k, V_MF | V_GENERAL>(x, a, s, grid, smem);
      break;
    default:
      stage_inst<k, V_GENERAL>(x, a, s, grid, smem);
  }
  g_launches++;
  if constexpr (k >= QF_VSPLIT) {
    if (a.mode == 1) {
      if (a.push)
        velocity_kernel<k, true><<<(a.n + 127) / 128, 128, 0, s>>>(
            x->tab, a.c_out, a.u_out, a.e0, a.n, x->err, a.push, a.peers);
      else
        velocity_kernel<k><<<(a.n + 127) / 128, 128, 0, s>>>(x->tab, a.c_out, a.u_out, a.e0, a.n,
                                                          x->err);
      g_launches++;
    }
  }
}

template <int k>
static void launch_velocity(qf_ctx* x, const double* c, double* u, int e0, int n, cudaStream_t s) {
  const int bs = 128, grid = (n + bs - 1) / bs;
  if (grid == 0) return;
  velocity_kernel<k><<<grid, bs, 0, s>>>(x->tab, c, u, e0, n, x->err);
  g_launches++;
}

template <int k>
static void launch_ghost(qf_ctx* x, double t, const double* t_dev, int nstage, double3 toffs,
                         cudaStream_t s) {
  const int nb = x->d.n_bnd;
  if (nb <= 0) return;
  const int n = nstage * nb * (Ord<k>::NG + 3);
  if (x->user_ghost) {  // user scenario module, same table layout
    Tab tab = x->tab;
    const int* bel = x->d.bnd_elem;
    const int* blc = x->d.bnd_local;
    double* gh = x->d.ghost;
    void* args[] = {&tab, &bel, &blc, (void*)&nb, &nstage, &t, (void*)&t_dev, &toffs, &gh};
    cudaLaunchKernel((const void*)x->user_ghost, dim3((n + 127) / 128), dim3(128), args, 0, s);
  } else {
    ghost_kernel<k><<<(n + 127) / 128, 128, 0, s>>>(x->tab, x->phys, x->d.bnd_elem,
                                                    x->d.bnd_local, nb, nstage, t, t_dev, toffs,
                                                    x->d.ghost);
  }
  g_launches++;
}

template <int k>
static void launch_static(qf_ctx* x, int n, cudaStream_t s) {
  if (n <= 0) return;
  static_kernel<k><<<(n + 127) / 128, 128, 0, s>>>(x->tab, n, x->d.hbt);
  g_launches++;
}

template <int k>
static void launch_project(qf_ctx* x, const double* prog, int n, double h_min, double* c,
                           double* hb) {
  if (n <= 0) return;
  project_kernel<k><<<(n + 127) / 128, 128, 0, x->stream_hint>>>(x->tab, x->phys, prog, n, h_min,
                                                                  c, hb, x->err);
  g_launches++;
}

template <int k>
static void launch_l2(qf_ctx* x, const double* c, double t, int e0, int n, int nb, double* sq,
                      cudaStream_t s) {
  l2err_kernel<k><<<nb, L2_BS, 0, s>>>(x->tab, x->phys, c, e0, n, t, x->l2part);
  l2sum_kernel<<<1, L2_BS, 0, s>>>(x->l2part, nb, sq);
  g_launches += 2;
}

template <int k>
static void launch_halo_traces(qf_ctx* x, const double* c, const double* u, const int32_t* items,
                               int n, double* out, cudaStream_t s) {
  halo_trace_kernel<k><<<(n + 127) / 128, 128, 0, s>>>(x->tab, c, u, items, n, out);
  g_launches++;
}

extern "C" {

int qf_abi_version(void) { return 3; }
const char* qf_last_error(void) { return g_last_error.c_str(); }
uint64_t qf_launch_count(void) { return g_launches.load(); }

int qf_create(const qf_desc* d, qf_ctx** out) {
  if (!d || !out) return fail(QF_E_ARG, "null argument");
  if (d->order < 0 || d->order > 4) return fail(QF_E_ARG, "order must be in 0..4");
  if (d->n_elem < 0 || d->ld < d->n_elem || d->ld % 32) return fail(QF_E_ARG, "bad n_elem/ld");
  if (!d->geo || !d->hb || !d->nbr || !d->hbt) return fail(QF_E_ARG, "missing static tables");
  if (d->n_bnd > 0 && (!d->bnd_elem || !d->bnd_local || !d->ghost))
    return fail(QF_E_ARG, "missing Dirichlet boundary tables");
  qf_ctx* x = new qf_ctx();
  x->d = *d;
  x->K = (d->order + 1) * (d->order + 2) / 2;
  {
    int dev = 0, nsm = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && nsm > 0)
      x->n_sm = nsm;
    x->device = dev;  // the caller's current device owns the tables
  }
  x->NT = d->order + 1;
  x->tab = Tab{d->geo, d->hb, d->nbr, d->ghost, d->hbt, d->ld, d->n_bnd,
               d->order <= 2 ? d->uni : nullptr};
  x->phys.g = d->g;
  x->phys.fc = d->f_c;
  x->phys.tau = d->tau_bf;
  x->phys.hb_linear = d->hb_linear;
  x->phys.kind = d->scn_kind;
  x->phys.forcing = d->has_forcing;
  x->phys.taylor = d->taylor;
  for (int i = 0; i < 8; ++i) x->phys.p[i] = d->scn_params[i];
  if (d->order >= 3 &&
      cudaMalloc(&x->vol, sizeof(double) * 3 * x->K * (size_t)d->ld) != cudaSuccess) {
    delete x;
    return fail(QF_E_CUDA, "cudaMalloc(volume scratch) failed");
  }
  if (cudaMalloc(&x->err, sizeof(unsigned)) != cudaSuccess ||
      cudaMemset(x->err, 0, sizeof(unsigned)) != cudaSuccess) {
    delete x;
    return fail(QF_E_CUDA, "cudaMalloc(error word) failed");
  }
  if (d->n_elem > 0) {  // request slots: busiest warp of the mesh, rounded up, capped
    // (ranges not aligned at slot 0 may overflow into the in-loop gather path)
    const int bs = d->order <= 1 ? Blk<1>::value : (d->order == 2 ? Blk<2>::value :
                   (d->order == 3 ? Blk<3>::value : Blk<4>::value));
    const int nw = bs / 32, grid = (d->n_elem + bs - 1) / bs;
    int h = 0;
    cudaMemset(x->err, 0, sizeof(unsigned));
    if (bs == 128)
      request_count_kernel<128><<<grid, 128>>>(d->nbr, d->ld, d->n_elem, (int*)x->err);
    else if (bs == 64)
      request_count_kernel<64><<<grid, 64>>>(d->nbr, d->ld, d->n_elem, (int*)x->err);
    else if (bs == 256)
      request_count_kernel<256><<<grid, 256>>>(d->nbr, d->ld, d->n_elem, (int*)x->err);
    if (cudaMemcpy(&h, x->err, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemset(x->err, 0, sizeof(unsigned)) != cudaSuccess) {
      cudaFree(x->err);
      delete x;
      return fail(QF_E_CUDA, "request count failed");
    }
    const int wc = std::min(std::max((h + 3) / 4 * 4, 4), QF_HCAP / nw);
    x->hcap = wc * nw;
    x->fits = h <= wc;
    int w = 0;
    wall_scan_kernel<<<(d->n_elem + 255) / 256, 256>>>(d->nbr, d->ld, d->n_elem, (int*)x->err);
    if (cudaMemcpy(&w, x->err, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemset(x->err, 0, sizeof(unsigned)) != cudaSuccess) {
      cudaFree(x->err);
      delete x;
      return fail(QF_E_CUDA, "wall scan failed");
    }
    x->walls = w != 0;
  }
  *out = x;
  return QF_OK;
}

void qf_destroy(qf_ctx* x) {
  if (!x) return;
  DevGuard guard(x);
  if (x->graph) cudaGraphExecDestroy(x->graph);
  if (x->vol) cudaFree(x->vol);
  if (x->l2part) cudaFree(x->l2part);
  if (x->frc) cudaFree(x->frc);
  if (x->user_lib) cudaLibraryUnload(x->user_lib);
  cudaFree(x->err);
  delete x;
}

int qf_velocity(qf_ctx* x, const double* c, double* u, int32_t e0, int32_t n, void* stream) {
  if (!x || !c || !u) return fail(QF_E_ARG, "null argument");
  DevGuard guard(x);
  if (n < 0) {
    e0 = 0;
    n = x->d.n_elem;
  }
  QF_DISPATCH(x->d.order, launch_velocity, x, c, u, e0, n, (cudaStream_t)stream);
  return cuda_check("velocity_kernel");
}

int qf_static(qf_ctx* x, int32_t n, void* stream) {
  if (!x) return fail(QF_E_ARG, "null ctx");
  DevGuard guard(x);
  QF_DISPATCH(x->d.order, launch_static, x, n, (cudaStream_t)stream);
  return cuda_check("static_kernel");
}

int qf_project(qf_ctx* x, const double* prog, int32_t n, double h_min, double* c, double* hb,
               void* stream) {
  if (!x || !prog || !c || !hb) return fail(QF_E_ARG, "null argument");
  DevGuard guard(x);
  x->stream_hint = (cudaStream_t)stream;
  QF_DISPATCH(x->d.order, launch_project, x, prog, n, h_min, c, hb);
  QF_DISPATCH(x->d.order, launch_static, x, n, (cudaStream_t)stream);
  return cuda_check("project_kernel");
}

int qf_l2_error(qf_ctx* x, const double* c, double t, int32_t e0, int32_t n, double* sq,
                void* stream) {
  if (!x || !c || !sq) return fail(QF_E_ARG, "null argument");
  DevGuard guard(x);
  if (x->phys.kind == SCN_NONE || x->phys.kind == SCN_USER)
    return fail(QF_E_ARG, "scenario has no built-in device exact solution");
  if (n < 0) {
    e0 = 0;
    n = x->d.n_elem;
  }
  const int nb = std::max((n + L2_BS - 1) / L2_BS, 1);
  if (nb > x->l2cap) {
    if (x->l2part) cudaFree(x->l2part);
    x->l2part = nullptr;
    x->l2cap = 0;
    if (cudaMalloc(&x->l2part, sizeof(double) * 3 * (size_t)nb) != cudaSuccess)
      return fail(QF_E_CUDA, "cudaMalloc(l2 partials) failed");
    x->l2cap = nb;
  }
  QF_DISPATCH(x->d.order, launch_l2, x, c, t, e0, n, nb, sq, (cudaStream_t)stream);
  return cuda_check("l2err_kernel");
}

int qf_ghost(qf_ctx* x, double t, void* stream) {
  if (!x) return fail(QF_E_ARG, "null ctx");
  DevGuard guard(x);
  QF_DISPATCH(x->d.order, launch_ghost, x, t, nullptr, 1, make_double3(0.0, 0.0, 0.0),
              (cudaStream_t)stream);
  return cuda_check("ghost_kernel");
}

int qf_ghost_dev(qf_ctx* x, const double* t_dev, double toff, void* stream) {
  if (!x || !t_dev) return fail(QF_E_ARG, "null argument");
  DevGuard guard(x);
  QF_DISPATCH(x->d.order, launch_ghost, x, 0.0, t_dev, 1, make_double3(toff, 0.0, 0.0),
              (cudaStream_t)stream);
  return cuda_check("ghost_kernel");
}

int qf_advance_time(double* t_dev, void* stream) {
  if (!t_dev) return fail(QF_E_ARG, "null argument");
  advance_time<<<1, 1, 0, (cudaStream_t)stream>>>(t_dev);
  g_launches++;
  return cuda_check("advance_time");
}

int qf_rhs(qf_ctx* x, const double* c, const double* u, double t, int32_t terms, double* rhs,
           double* lam, void* stream) {
  return qf_rhs_mass(x, c, u, t, terms, rhs, lam, nullptr, stream);
}

int qf_rhs_mass(qf_ctx* x, const double* c, const double* u, double t, int32_t terms,
                double* rhs, double* lam, double* mflux, void* stream) {
  return qf_rhs_ex(x, c, u, t, terms, rhs, lam, mflux, nullptr, stream);
}

int qf_rhs_ex(qf_ctx* x, const double* c, const double* u, double t, int32_t terms, double* rhs,
              double* lam, double* mflux, const double* lam_in, void* stream) {
  if (!x || !c || !u || !rhs) return fail(QF_E_ARG, "null argument");
  DevGuard guard(x);
  cudaStream_t s = (cudaStream_t)stream;
  if (terms & TERM_EDGE)
    QF_DISPATCH(x->d.order, launch_ghost, x, t, nullptr, 1, make_double3(0.0, 0.0, 0.0), s);
  StageArgs a{};
  a.c = c;
  a.u = u;
  a.c_out = rhs;
  a.lam = lam;
  a.mflux = (terms & TERM_EDGE) ? mflux : nullptr;
  a.lam_in = lam_in;
  a.ht = x->halo_ht;
  a.err = x->err;
  a.t = t;
  a.e0 = 0;
  a.n = x->d.n_elem;
  a.terms = terms;
  a.mode = 0;
  QF_DISPATCH(x->d.order, launch_stage, x, a, s);
  return cuda_check("stage_kernel(rhs)");
}

int qf_stage(qf_ctx* x, const double* c_in, const double* u_in, const double* c0, double* c_out,
             double* u_out, double aa, double bb, double t, double dt, const double* t_dev,
             double toff, int32_t e0, int32_t n, void* stream) {
  return qf_stage_push(x, c_in, u_in, c0, c_out, u_out, aa, bb, t, dt, t_dev, toff, e0, n,
                       x ? x->halo_ht : nullptr, nullptr, nullptr, stream);
}

int qf_stage_push(qf_ctx* x, const double* c_in, const double* u_in, const double* c0,
                  double* c_out, double* u_out, double aa, double bb, double t, double dt,
                  const double* t_dev, double toff, int32_t e0, int32_t n, const double* ht_in,
                  const int32_t* push, const qf_peer* peers, void* stream) {
  if (!x || !c_in || !u_in || !c_out || !u_out) return fail(QF_E_ARG, "null argument");
  DevGuard guard(x);
  if (push && !peers) return fail(QF_E_ARG, "push table without peer table");
  if (aa != 0.0 && !c0) return fail(QF_E_ARG, "stage base c0 required");
  if (n < 0) {
    e0 = 0;
    n = x->d.n_elem;
  }
  StageArgs a{};
  a.c = c_in;
  a.u = u_in;
  a.c0 = c0;
  a.c_out = c_out;
  a.u_out = u_out;
  a.err = x->err;
  a.t_dev = t_dev;
  a.t = t;
  a.toff = toff;
  a.dt = dt;
  a.a = aa;
  a.b = bb;
  a.e0 = e0;
  a.n = n;
  a.terms = TERM_VOL | TERM_EDGE | TERM_SRC;
  a.mode = 1;
  a.push = push;
  a.peers = peers;
  a.ht = ht_in;
  QF_DISPATCH(x->d.order, launch_stage, x, a, (cudaStream_t)stream);
  return cuda_check("stage_kernel");
}

}  // extern "C"

// t_dev = {t, dt} lives on the device so one captured step is replayable.
static void step_impl(qf_ctx* x, double* c, double* u, double* work, double* t_dev,
                      cudaStream_t s) {
  const int64_t S = (int64_t)5 * x->K * x->d.ld;  // one (c, u) state
  const int64_t CU = (int64_t)3 * x->K * x->d.ld;
  double* c1 = work;
  double* u1 = work + CU;
  double* c2 = work + S;
  double* u2 = work + S + CU;
  const int k = x->d.order;
  const int nst = k == 0 ? 1 : (k == 1 ? 2 : 3);
  const double3 toffs = k == 1 ? make_double3(0.0, 1.0, 0.0) : make_double3(0.0, 1.0, 0.5);
  QF_DISPATCH(k, launch_ghost, x, 0.0, t_dev, nst, toffs, s);
  int gst = 0;
  auto stage = [&](const double* ci, const double* ui, const double* cb, double* co, double* uo,
                   double a, double b, double toff) {
    StageArgs A{};
    A.gstage = gst++;
    A.c = ci;
    A.u = ui;
    A.c0 = cb;
    A.c_out = co;
    A.u_out = uo;
    A.err = x->err;
    A.t_dev = t_dev;
    A.toff = toff;
    A.a = a;
    A.b = b;
    A.e0 = 0;
    A.n = x->d.n_elem;
    A.terms = TERM_VOL | TERM_EDGE | TERM_SRC;
    A.mode = 1;
    A.ht = x->halo_ht;
    const int si = A.gstage;
    if (2 * si + 1 < x->n_stage_ev) cudaEventRecordWithFlags(x->stage_ev[2 * si], s, cudaEventRecordExternal);
    QF_DISPATCH(k, launch_stage, x, A, s);
    if (2 * si + 1 < x->n_stage_ev) cudaEventRecordWithFlags(x->stage_ev[2 * si + 1], s, cudaEventRecordExternal);
  };
  // SSP-RK by order (solver.py:756-764); the last stage writes in place:
  // each thread reads c0[e] before writing c_out[e] and no thread reads
  // another element's c0 or the old u in that stage.
  if (k == 0) {
    stage(c, u, nullptr, c1, u1, 0.0, 1.0, 0.0);
    cudaMemcpyAsync(c, c1, CU * sizeof(double), cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(u, u1, (S - CU) * sizeof(double), cudaMemcpyDeviceToDevice, s);
  } else if (k == 1) {
    stage(c, u, nullptr, c1, u1, 0.0, 1.0, 0.0);
    stage(c1, u1, c, c, u, 0.5, 0.5, 1.0);
  } else {
    stage(c, u, nullptr, c1, u1, 0.0, 1.0, 0.0);
    stage(c1, u1, c, c2, u2, 0.75, 0.25, 1.0);
    stage(c2, u2, c, c, u, 1.0 / 3.0, 2.0 / 3.0, 0.5);
  }
  advance_time<<<1, 1, 0, s>>>(t_dev);
  g_launches++;
}

extern "C" {

int qf_step(qf_ctx* x, double* c, double* u, double* work, double* t_dev, void* stream) {
  if (!x || !c || !u || !work || !t_dev) return fail(QF_E_ARG, "null argument");
  DevGuard guard(x);
  step_impl(x, c, u, work, t_dev, (cudaStream_t)stream);
  return cuda_check("qf_step");
}

static int kernels_per_step(qf_ctx* x) {
  const int stages = x->d.order == 0 ? 1 : (x->d.order == 1 ? 2 : 3);
  const int vol = x->d.order == 4 ? (FuseVol<4>::value ? 0 : VGroups<4>::value)
                                  : (x->d.order == 3 ? (FuseVol<3>::value ? 0 : VGroups<3>::value) : 0);
  return stages * (1 + vol + (x->d.order >= QF_VSPLIT)) + (x->d.n_bnd > 0 ? 1 : 0) + 1;
}

int qf_run(qf_ctx* x, int32_t n_steps, double* c, double* u, double* work, double* t_dev,
           int32_t use_graph, void* stream) {
  if (!x || !c || !u || !work || !t_dev) return fail(QF_E_ARG, "null argument");
  DevGuard guard(x);
  cudaStream_t s = (cudaStream_t)stream;
  if (!use_graph || x->d.order == 0) {
    for (int i = 0; i < n_steps; ++i) step_impl(x, c, u, work, t_dev, s);
    return cuda_check("qf_run");
  }
  const void* key[4] = {c, u, work, t_dev};
  if (!x->graph || memcmp(key, x->gkey, sizeof(key)) != 0) {
    if (x->graph) {
      cudaGraphExecDestroy(x->graph);
      x->graph = nullptr;
    }
    cudaStream_t cap = s;
    bool own = false;
    if (s == nullptr) {
      if (cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) != cudaSuccess)
        return fail(QF_E_CUDA, "stream create failed");
      own = true;
    }
    cudaGraph_t g;
    if (cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
      return fail(QF_E_CUDA, "begin capture failed");
    const uint64_t before = g_launches.load();
    step_impl(x, c, u, work, t_dev, cap);
    g_launches.store(before);
    if (cudaStreamEndCapture(cap, &g) != cudaSuccess) return fail(QF_E_CUDA, "end capture failed");
    cudaError_t e = cudaGraphInstantiate(&x->graph, g, 0);
    cudaGraphDestroy(g);
    if (own) cudaStreamDestroy(cap);
    if (e != cudaSuccess) return fail(QF_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
    memcpy(x->gkey, key, sizeof(key));
  }
  for (int i = 0; i < n_steps; ++i) {
    if (cudaGraphLaunch(x->graph, s) != cudaSuccess) return cuda_check("cudaGraphLaunch");
  }
  g_launches += (uint64_t)n_steps * kernels_per_step(x);
  return cuda_check("qf_run");
}

int qf_halo_table(qf_ctx* x, const double* ht) {
  if (!x) return fail(QF_E_ARG, "null ctx");
  x->halo_ht = ht;
  return QF_OK;
}

int qf_halo_traces(qf_ctx* x, const double* c, const double* u, const int32_t* items, int32_t n,
                   double* out, void* stream) {
  if (!x || !c || !u || (n > 0 && (!items || !out))) return fail(QF_E_ARG, "null argument");
  if (n <= 0) return QF_OK;
  DevGuard guard(x);
  QF_DISPATCH(x->d.order, launch_halo_traces, x, c, u, items, n, out, (cudaStream_t)stream);
  return cuda_check("halo_trace_kernel");
}

int qf_user_scenario(qf_ctx* x, const void* image, size_t size, int32_t with_forcing) {
  if (!x || !image || size == 0) return fail(QF_E_ARG, "null argument");
  DevGuard guard(x);
  (void)size;
  cudaLibrary_t lib = nullptr;
  if (cudaLibraryLoadData(&lib, image, nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess)
    return cuda_check("cudaLibraryLoadData(user scenario)");
  cudaKernel_t kg = nullptr, kf = nullptr;
  if (cudaLibraryGetKernel(&kg, lib, "qf_user_ghost") != cudaSuccess ||
      (with_forcing && cudaLibraryGetKernel(&kf, lib, "qf_user_forcing") != cudaSuccess)) {
    cudaLibraryUnload(lib);
    return cuda_check("cudaLibraryGetKernel(user scenario)");
  }
  if (with_forcing && !x->frc &&
      cudaMalloc(&x->frc, sizeof(double) * 2 * x->K * (size_t)x->d.ld) != cudaSuccess) {
    cudaLibraryUnload(lib);
    return fail(QF_E_CUDA, "cudaMalloc(user forcing rows) failed");
  }
  if (x->user_lib) cudaLibraryUnload(x->user_lib);
  x->user_lib = lib;
  x->user_ghost = kg;
  x->user_forcing = with_forcing ? kf : nullptr;
  if (x->graph) {
    cudaGraphExecDestroy(x->graph);
    x->graph = nullptr;
  }
  return QF_OK;
}

int qf_stage_events(qf_ctx* x, void* const* events, int32_t n) {
  if (!x || n < 0 || n > 8 || (n > 0 && !events)) return fail(QF_E_ARG, "bad stage event list");
  for (int i = 0; i < n; ++i) x->stage_ev[i] = (cudaEvent_t)events[i];
  x->n_stage_ev = n;
  if (x->graph) {  // re-capture with (or without) the event-record nodes
    cudaGraphExecDestroy(x->graph);
    x->graph = nullptr;
  }
  return QF_OK;
}

int qf_error(qf_ctx* x, uint32_t* bits, int32_t clear, void* stream) {
  if (!x || !bits) return fail(QF_E_ARG, "null argument");
  DevGuard guard(x);
  cudaStream_t s = (cudaStream_t)stream;
  unsigned h = 0;
  if (cudaMemcpyAsync(&h, x->err, sizeof(unsigned), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return cuda_check("qf_error");
  if (clear) cudaMemsetAsync(x->err, 0, sizeof(unsigned), s);
  *bits = h;
  return cuda_check("qf_error");
}

int qf_pack(const double* aos, double* soa, int32_t n, int32_t F, int32_t K, int64_t ld,
            const int32_t* perm, void* stream) {
  if (n <= 0) return QF_OK;
  pack_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(aos, soa, n, F, K, ld, perm);
  g_launches++;
  return cuda_check("pack_kernel");
}

int qf_unpack(const double* soa, double* aos, int32_t n, int32_t F, int32_t K, int64_t ld,
              const int32_t* perm, void* stream) {
  if (n <= 0) return QF_OK;
  unpack_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(soa, aos, n, F, K, ld, perm);
  g_launches++;
  return cuda_check("unpack_kernel");
}

int qf_gather(const double* src, int64_t ld, const int32_t* idx, int32_t n, int32_t rows,
              double* dst, void* stream) {
  if (n <= 0) return QF_OK;
  gather_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(src, ld, idx, n, rows, dst);
  g_launches++;
  return cuda_check("gather_kernel");
}

int qf_scatter(const double* src, const int32_t* idx, int32_t n, int32_t rows, double* dst,
               int64_t ld, void* stream) {
  if (n <= 0) return QF_OK;
  scatter_kernel<<<(n + 127) / 128, 128, 0, (cudaStream_t)stream>>>(src, idx, n, rows, dst, ld);
  g_launches++;
  return cuda_check("scatter_kernel");
}

// ------------------------------------------------ fused halo transport
// Stream memory operations (signal / wait on a 32-bit flag in local or
// peer memory: the GPU front-end waits, no kernel spins) and CUDA IPC
// export / import of device buffers, for the multi-process P2P transport of
// paper_1904_08684_b200/distributed.py.  Driver entry points are resolved
// through the runtime (no link-time libcuda dependency).
typedef int (*qf_pfn_value32)(void*, unsigned long long, unsigned int, unsigned int);
typedef int (*qf_pfn_addr_range)(unsigned long long*, size_t*, unsigned long long);

static void* driver_fn(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return fn;
}

int qf_signal(uint32_t* flag, uint32_t value, void* stream) {
  static qf_pfn_value32 fn = (qf_pfn_value32)driver_fn("cuStreamWriteValue32");
  if (!flag) return fail(QF_E_ARG, "null flag");
  if (!fn) return fail(QF_E_CUDA, "cuStreamWriteValue32 unavailable");
  if (fn(stream, (unsigned long long)(uintptr_t)flag, value, 0) != 0)
    return fail(QF_E_CUDA, "cuStreamWriteValue32 failed");
  return QF_OK;
}

int qf_wait(const uint32_t* flag, uint32_t value, void* stream) {
  static qf_pfn_value32 fn = (qf_pfn_value32)driver_fn("cuStreamWaitValue32");
  if (!flag) return fail(QF_E_ARG, "null flag");
  if (!fn) return fail(QF_E_CUDA, "cuStreamWaitValue32 unavailable");
  // CU_STREAM_WAIT_VALUE_GEQ = 0: wait until (int32)(*flag - value) >= 0
  if (fn(stream, (unsigned long long)(uintptr_t)flag, value, 0) != 0)
    return fail(QF_E_CUDA, "cuStreamWaitValue32 failed");
  return QF_OK;
}

// ---------------------------------------------- captured partitioned step
// (see include/qfswe.h).  The stream memory operations are captured as
// batch-memop nodes; their 32-bit values are re-based before every launch.
struct qf_graph {
  cudaGraph_t graph = nullptr;  // kept: the memop node handles belong to it
  cudaGraphExec_t exec = nullptr;
  struct MemOp {
    CUgraphNode node;
    CUDA_BATCH_MEM_OP_NODE_PARAMS params;
    std::vector<CUstreamBatchMemOpParams> ops;  // as captured
  };
  std::vector<MemOp> memops;
  uint64_t kernels = 0;  // kernel nodes (launch count per replay)
};

typedef CUresult (*qf_pfn_memop_get)(CUgraphNode, CUDA_BATCH_MEM_OP_NODE_PARAMS*);
typedef CUresult (*qf_pfn_memop_set)(CUgraphExec, CUgraphNode, const CUDA_BATCH_MEM_OP_NODE_PARAMS*);

int qf_graph_begin(void* stream) {
  if (cudaStreamBeginCapture((cudaStream_t)stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess)
    return cuda_check("cudaStreamBeginCapture");
  return QF_OK;
}

int qf_graph_end(void* stream, qf_graph** out) {
  if (!out) return fail(QF_E_ARG, "null argument");
  static qf_pfn_memop_get get = (qf_pfn_memop_get)driver_fn("cuGraphBatchMemOpNodeGetParams");
  cudaGraph_t g = nullptr;
  if (cudaStreamEndCapture((cudaStream_t)stream, &g) != cudaSuccess || !g)
    return cuda_check("cudaStreamEndCapture");
  qf_graph* q = new qf_graph();
  size_t n = 0;
  cudaGraphGetNodes(g, nullptr, &n);
  std::vector<cudaGraphNode_t> nodes(n);
  if (n) cudaGraphGetNodes(g, nodes.data(), &n);
  // (driver-level node types: the runtime's enumeration has no batch-memop type)
  typedef CUresult (*pfn_type)(CUgraphNode, CUgraphNodeType*);
  static pfn_type node_type = (pfn_type)driver_fn("cuGraphNodeGetType");
  for (cudaGraphNode_t nd : nodes) {
    CUgraphNodeType ty;
    if (!node_type || node_type((CUgraphNode)nd, &ty) != CUDA_SUCCESS) {
      cudaGraphDestroy(g);
      delete q;
      return fail(QF_E_CUDA, "cuGraphNodeGetType failed");
    }
    if (ty == CU_GRAPH_NODE_TYPE_KERNEL) q->kernels++;
    if (ty != CU_GRAPH_NODE_TYPE_BATCH_MEM_OP) continue;
    if (!get) {
      cudaGraphDestroy(g);
      delete q;
      return fail(QF_E_CUDA, "cuGraphBatchMemOpNodeGetParams unavailable");
    }
    qf_graph::MemOp m;
    m.node = (CUgraphNode)nd;
    if (get(m.node, &m.params) != CUDA_SUCCESS) {
      cudaGraphDestroy(g);
      delete q;
      return fail(QF_E_CUDA, "cuGraphBatchMemOpNodeGetParams failed");
    }
    m.ops.assign(m.params.paramArray, m.params.paramArray + m.params.count);
    q->memops.push_back(std::move(m));
  }
  cudaError_t e = cudaGraphInstantiate(&q->exec, g, 0);
  if (e != cudaSuccess) {
    cudaGraphDestroy(g);
    delete q;
    return fail(QF_E_CUDA, std::string("graph instantiate: ") + cudaGetErrorString(e));
  }
  q->graph = g;
  *out = q;
  return QF_OK;
}

int qf_graph_launch(qf_graph* q, uint32_t delta, void* stream) {
  if (!q || !q->exec) return fail(QF_E_ARG, "null graph");
  static qf_pfn_memop_set set = (qf_pfn_memop_set)driver_fn("cuGraphExecBatchMemOpNodeSetParams");
  if (!q->memops.empty() && !set) return fail(QF_E_CUDA, "cuGraphExecBatchMemOpNodeSetParams unavailable");
  for (auto& m : q->memops) {
    std::vector<CUstreamBatchMemOpParams> ops = m.ops;
    for (auto& op : ops) {
      if (op.operation == CU_STREAM_MEM_OP_WAIT_VALUE_32)
        op.waitValue.value += delta;
      else if (op.operation == CU_STREAM_MEM_OP_WRITE_VALUE_32)
        op.writeValue.value += delta;
    }
    CUDA_BATCH_MEM_OP_NODE_PARAMS p = m.params;
    p.paramArray = ops.data();
    if (set((CUgraphExec)q->exec, m.node, &p) != CUDA_SUCCESS)
      return fail(QF_E_CUDA, "cuGraphExecBatchMemOpNodeSetParams failed");
  }
  if (cudaGraphLaunch(q->exec, (cudaStream_t)stream) != cudaSuccess) return cuda_check("cudaGraphLaunch");
  g_launches += q->kernels;
  return QF_OK;
}

void qf_graph_destroy(qf_graph* q) {
  if (!q) return;
  if (q->exec) cudaGraphExecDestroy(q->exec);
  if (q->graph) cudaGraphDestroy(q->graph);
  delete q;
}

int qf_ipc_export(const void* ptr, void* handle, uint64_t* offset) {
  static qf_pfn_addr_range range = (qf_pfn_addr_range)driver_fn("cuMemGetAddressRange");
  if (!ptr || !handle || !offset) return fail(QF_E_ARG, "null argument");
  if (!range) return fail(QF_E_CUDA, "cuMemGetAddressRange unavailable");
  unsigned long long base = 0;
  size_t size = 0;
  if (range(&base, &size, (unsigned long long)(uintptr_t)ptr) != 0)
    return fail(QF_E_CUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base) != cudaSuccess) return cuda_check("cudaIpcGetMemHandle");
  memcpy(handle, &h, sizeof(h));
  *offset = (uint64_t)((uintptr_t)ptr - (uintptr_t)base);
  return QF_OK;
}

// one mapping per exported allocation (several buffers of a peer usually
// share one caching-allocator segment)
static std::vector<std::pair<std::string, void*>> g_ipc_maps;

int qf_ipc_import(const void* handle, uint64_t offset, void** ptr) {
  if (!handle || !ptr) return fail(QF_E_ARG, "null argument");
  const std::string key((const char*)handle, sizeof(cudaIpcMemHandle_t));
  void* base = nullptr;
  for (auto& m : g_ipc_maps)
    if (m.first == key) base = m.second;
  if (!base) {
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    if (cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
      return cuda_check("cudaIpcOpenMemHandle");
    g_ipc_maps.emplace_back(key, base);
  }
  *ptr = (char*)base + offset;
  return QF_OK;
}

int qf_ipc_close_all(void) {
  for (auto& m : g_ipc_maps) cudaIpcCloseMemHandle(m.second);
  g_ipc_maps.clear();
  return cuda_check("cudaIpcCloseMemHandle");
}

int qf_copy(void* dst, const void* src, size_t bytes, void* stream) {
  if (bytes == 0) return QF_OK;
  if (!dst || !src) return fail(QF_E_ARG, "null argument");
  if (cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, (cudaStream_t)stream) != cudaSuccess)
    return cuda_check("qf_copy");
  return QF_OK;
}

int qf_fill(double* buf, size_t n, double v, void* stream) {
  fill_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(buf, n, v);
  g_launches++;
  return cuda_check("fill_kernel");
}

}  // extern "C"
#endif  // QF_KERNELS_ONLY
