/*
 * qfswe.h — C ABI of the B200 (sm_100a) per-stage RHS path of the
 * quadrature-free DG shallow-water solver (arXiv 1904.08684).
 *
 * Drop-in boundary for the reference Python package `qfswe`
 * (/root/reference/pkg/src/qfswe/solver.py).  Every entry point replaces
 * one reference method; the Python host mirror
 * (paper_1904_08684_b200/solver.py) binds them with ctypes exactly as a
 * maintainer of the reference would.
 *
 * Conventions
 *  - Plain pointers and sizes only.  All `double*` / `int32_t*` arguments
 *    are DEVICE pointers owned by the caller; the context only borrows them.
 *  - State layout is structure-of-arrays, element index fastest:
 *      c[3][K][ld] (xi, U, V),  u[2][K][ld] (u, v),  rhs like c,
 *    K = (k+1)(k+2)/2, ld >= n_elem, ld % 32 == 0.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *  - Every call returns a status: QF_OK, or QF_E_* below.  Asynchronous
 *    numerical faults (dry state, singular projection, non-finite values)
 *    are latched in a device error word read with qf_error().
 *  - One context per (process, device): qf_create binds the caller's
 *    current device; every entry point taking a context makes that device
 *    current for the call and restores the caller's afterwards.  Calls on
 *    one context must be serialised by the caller (same as the reference's
 *    single-threaded Discretization).
 */
#ifndef QFSWE_H
#define QFSWE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  QF_OK = 0,
  QF_E_DRY = 1,        /* DryState          (solver.py:40-41, raised :308-311,:369-371,:403-404) */
  QF_E_SINGULAR = 2,   /* SingularProjection (solver.py:44-45, raised :330-335) */
  QF_E_NONFINITE = 3,  /* FloatingPointError (solver.py:768-769) */
  QF_E_CUDA = 4,
  QF_E_ARG = 5
};

/* error-word bits latched by the kernels */
enum { QF_BIT_DRY = 1u, QF_BIT_SINGULAR = 2u, QF_BIT_NONFINITE = 4u };

/* rhs term mask (reference rhs = element + edge + source, solver.py:727-741) */
enum { QF_TERM_VOLUME = 1, QF_TERM_EDGE = 2, QF_TERM_SOURCE = 4, QF_TERM_ALL = 7 };

/* device scenario families (paper_1904_08684_b200/scenario.py) */
enum { QF_SCN_NONE = 0, QF_SCN_MMS = 1, QF_SCN_TRAVEL = 2, QF_SCN_LAKE = 3, QF_SCN_USER = 4 };

typedef struct qf_desc {
  int32_t order;            /* k in 0..4 */
  int32_t n_elem;           /* elements this context updates (owned) */
  int64_t ld;               /* leading dimension of every [..][ld] table */
  /* static element tables (device) */
  const double* geo;        /* [6][ld]: B11, B12, B21, B22, a1x, a1y      (mesh.py:259-282) */
  const double* hb;         /* [NH][ld]: P1 bathymetry, NH = 1 (k=0) or 3 (solver.py:139-168) */
  const int32_t* nbr;       /* [3][ld]: neighbour codes (layout.py)        (mesh.py:79-107) */
  int32_t n_bnd;            /* Dirichlet boundary slots */
  const int32_t* bnd_elem;  /* [n_bnd] */
  const int32_t* bnd_local; /* [n_bnd] */
  double* ghost;            /* [3][n_bnd][5*(k+2)+6] scratch: exact data per RK stage */
  double* hbt;              /* [3*(k+1)+1][ld] static h_b edge traces, filled by qf_static */
  /* physics (scenario.py:34-49) */
  double g, f_c, tau_bf;
  int32_t hb_linear;        /* hb_mode == "linear" */
  int32_t scn_kind;         /* QF_SCN_* */
  double scn_params[8];
  int32_t has_forcing;      /* momentum forcing + xi mass source of the family */
  int32_t taylor;           /* MMS: 1 if max |2 pi (x_q - x_centroid)| <= 0.06 on this mesh, 2 if
                               <= 0.02, so the forcing may use element-local Taylor sin/cos of
                               degree 9 resp. 7 (truncation < 1e-18); 0 = libm sincospi */
  int32_t block;            /* threads per block (0 = default) */
  const double* uni;        /* MMS, k <= 2: phase-offset table when the element Jacobians take at
                               most two values (uniform split-square meshes), else NULL; layout:
                               [0..3] class-1 B, then per class c (offset 8 + c*(6*NQ+2)) and
                               quadrature point q: sin z, cos z, sin w, cos w, sin(z+w), cos(z+w)
                               with (z, w) = 2 pi B (r_q - centroid), NQ = (k+2)^2 */
} qf_desc;

typedef struct qf_ctx qf_ctx;

/* Destination of the fused halo push in one peer partition: its halo trace
 * table for the stage output, ht[row][6][k+1] (trace moments of xi, U, V,
 * u, v, h_b on the cut edge, in the sender's edge parametrisation); device
 * pointer on the same GPU, peer-accessible, or mapped with qf_ipc_import. */
typedef struct qf_peer {
  double* ht;
} qf_peer;

/* Discretization.__init__ (solver.py:103-124): bind tables, validate. */
int qf_create(const qf_desc* desc, qf_ctx** out);
void qf_destroy(qf_ctx* ctx);

/* Discretization.solve_velocity (solver.py:315-336): u for elements
 * [e0, e0+n) of state c (n < 0: all owned elements). */
int qf_velocity(qf_ctx* ctx, const double* c, double* u, int32_t e0, int32_t n, void* stream);

/* Derived static tables (h_b edge traces) from geo and hb for the first n
 * slots; call after hb is final (qf_project calls it itself). */
int qf_static(qf_ctx* ctx, int32_t n, void* stream);

/* Device-side setup (project_initial / P1 bathymetry, solver.py:139-168,
 * 282-303): project the field program `prog` (see qf_kernels.cu) onto the
 * basis for the first n element slots: c[3][K][ld] and hb[NH][ld]; latches
 * QF_BIT_DRY if the projected depth falls below h_min at a quadrature point. */
int qf_project(qf_ctx* ctx, const double* prog, int32_t n, double h_min, double* c, double* hb,
               void* stream);

/* Dirichlet ghost data at time t into stage table 0 (solver.py:395-402, 636-653);
 * qf_stage reads table 0, qf_step/qf_run fill all stage tables themselves. */
int qf_ghost(qf_ctx* ctx, double t, void* stream);
/* The same at the device time t_dev[0] + toff * t_dev[1] (t_dev = {t, dt}),
 * and the time advance t_dev[0] += t_dev[1]: what a partitioned step needs
 * to be replayable as a captured graph (qf_graph_*). */
int qf_ghost_dev(qf_ctx* ctx, const double* t_dev, double toff, void* stream);
int qf_advance_time(double* t_dev, void* stream);

/* Discretization.rhs / element_rhs / edge_rhs / source_rhs / compute_lambda
 * (solver.py:340-741): rhs = sum of the masked terms at time t.
 * lam (optional, [3][ld]): lambda of each element's local edges. */
int qf_rhs(qf_ctx* ctx, const double* c, const double* u, double t, int32_t terms,
           double* rhs, double* lam, void* stream);

/* qf_rhs with Discretization.instrument_mass_flux (solver.py:123-124,
 * 619-620, 696-701): mflux (device [3][ld]) receives, per element and local
 * edge, that edge's contribution to the element's xi mode-0 rhs (times
 * sqrt(detB)/sqrt(2) = the element's mass rate through the edge). */
int qf_rhs_mass(qf_ctx* ctx, const double* c, const double* u, double t, int32_t terms,
                double* rhs, double* lam, double* mflux, void* stream);

/* qf_rhs_mass with a caller-supplied lambda (reference edge_rhs(state, t,
 * lam), solver.py:690-704): lam_in (device [3][ld], may be NULL) is the
 * Lax-Friedrichs speed each element uses on its local edges instead of the
 * recomputed one (both sides of an edge must carry the same value). */
int qf_rhs_ex(qf_ctx* ctx, const double* c, const double* u, double t, int32_t terms,
              double* rhs, double* lam, double* mflux, const double* lam_in, void* stream);

/* One SSP-RK stage (solver.py:750-764) for elements [e0, e0+n):
 *   c_out = a*c0 + b*(c_in + dt*rhs(c_in, u_in, t)),  u_out = velocity(c_out).
 * t_dev (optional device [2] = {t_step, dt}) overrides t: t = t_dev[0] + toff*t_dev[1]. */
int qf_stage(qf_ctx* ctx, const double* c_in, const double* u_in, const double* c0,
             double* c_out, double* u_out, double a, double b, double t, double dt,
             const double* t_dev, double toff, int32_t e0, int32_t n, void* stream);

/* qf_stage on a partition, with the halo exchange fused into the stage
 * (SURVEY §8e).  Neighbour codes 4 h + 3 (layout.py) name row h of the
 * halo trace table ht_in (device, rows of 6 (k+1) doubles: the trace
 * moments of the other partition's element on the shared edge for the
 * stage input).  push (device int32 [3][ld], may be NULL): per element and
 * local cut edge the destination (peer << 26) | row; the thread that
 * computes a cut-adjacent element's new (c, u) also computes its trace
 * moments on that edge and stores them into the peer's table (peers: device
 * qf_peer table indexed by peer).  Ordering with the peers' next stage is
 * the caller's (stream order on one GPU, qf_signal / qf_wait across
 * processes). */
int qf_stage_push(qf_ctx* ctx, const double* c_in, const double* u_in, const double* c0,
                  double* c_out, double* u_out, double a, double b, double t, double dt,
                  const double* t_dev, double toff, int32_t e0, int32_t n, const double* ht_in,
                  const int32_t* push, const qf_peer* peers, void* stream);

/* Halo trace rows for the NCCL transport: out[i][6][k+1] = trace moments of
 * element items[i] >> 2 on its local edge items[i] & 3 of state (c, u), with
 * the stage kernel's rounding (bit-identical to what the fused push stores). */
int qf_halo_traces(qf_ctx* ctx, const double* c, const double* u, const int32_t* items,
                   int32_t n, double* out, void* stream);

/* Halo trace table used by qf_rhs / qf_velocity-free operators on a
 * partition (the stage input of qf_stage_push is explicit); NULL clears. */
int qf_halo_table(qf_ctx* ctx, const double* ht);

/* Stream-ordered 32-bit flag write (local or peer memory) and wait until
 * (int32)(*flag - value) >= 0: cross-process stage ordering of the fused
 * halo push (stream memory operations, no spinning kernel). */
int qf_signal(uint32_t* flag, uint32_t value, void* stream);
int qf_wait(const uint32_t* flag, uint32_t value, void* stream);

/* One partitioned step as a replayable CUDA graph.  qf_graph_begin starts a
 * capture on `stream`; the caller then enqueues the step exactly as it
 * would run it -- qf_ghost_dev, qf_stage_push with t_dev, qf_wait /
 * qf_signal (captured as memory-operation nodes), on this and on streams
 * forked from and joined back to it with events -- and qf_graph_end
 * instantiates the graph.  The flag values of a step grow with the stage
 * count, so qf_graph_launch(g, delta, stream) first adds `delta` (stages
 * completed since the capture) to the value of every captured wait / write
 * node, then launches.  One host call per step instead of ~10 per stage. */
typedef struct qf_graph qf_graph;
int qf_graph_begin(void* stream);
int qf_graph_end(void* stream, qf_graph** out);
int qf_graph_launch(qf_graph* g, uint32_t delta, void* stream);
void qf_graph_destroy(qf_graph* g);

/* CUDA IPC of device buffers: handle (64 bytes) + offset of ptr inside its
 * allocation; import maps a peer's allocation once per process. */
int qf_ipc_export(const void* ptr, void* handle, uint64_t* offset);
int qf_ipc_import(const void* handle, uint64_t offset, void** ptr);
int qf_ipc_close_all(void);

/* Discretization.step (solver.py:745-770): one SSP-RK step in place on
 * (c, u); `u` must hold velocity(c) on entry (qf_velocity).  `work` holds
 * 2 * 5 * K * ld doubles.  t_dev: device [2] = {t, dt}; advanced by dt. */
int qf_step(qf_ctx* ctx, double* c, double* u, double* work, double* t_dev, void* stream);

/* Discretization.run (solver.py:772-780): n_steps steps, captured once in a
 * CUDA graph (use_graph != 0) and replayed. */
int qf_run(qf_ctx* ctx, int32_t n_steps, double* c, double* u, double* work, double* t_dev,
           int32_t use_graph, void* stream);

/* State <-> device layout: aos [E][F][K] (reference State.c / State.u)
 * <-> soa [F][K][ld].  perm (optional, device int32 [n]): device slot d holds
 * aos row perm[d] (locality order of the element tables); NULL = identity. */
int qf_pack(const double* aos, double* soa, int32_t n_elem, int32_t F, int32_t K, int64_t ld,
            const int32_t* perm, void* stream);
int qf_unpack(const double* soa, double* aos, int32_t n_elem, int32_t F, int32_t K, int64_t ld,
              const int32_t* perm, void* stream);

/* gather / scatter rows for halo exchange: dst[r][i] = src[r][idx[i]] (rows
 * of length ld / n_idx) and the inverse scatter. */
int qf_gather(const double* src, int64_t ld_src, const int32_t* idx, int32_t n_idx,
              int32_t rows, double* dst, void* stream);
int qf_scatter(const double* src, const int32_t* idx, int32_t n_idx, int32_t rows,
               double* dst, int64_t ld_dst, void* stream);

/* harness.l2_error (harness.py:81-98) on the device: sq[0..2] (DEVICE, 3
 * doubles) = squared global L2 errors of xi, U, V of state c against the
 * scenario's exact solution at time t over elements [e0, e0+n) (n < 0: all
 * owned), at the degree-(2k+2) collapsed Gauss rule; deterministic
 * reduction order.  QF_E_ARG if the scenario family has no device exact
 * solution (QF_SCN_NONE).  The L2 norms are sqrt(sq) (after an allreduce-sum
 * over partitions). */
int qf_l2_error(qf_ctx* ctx, const double* c, double t, int32_t e0, int32_t n, double* sq,
                void* stream);

/* User scenario (reference custom_scenario, scenario.py:153-157): `image`
 * is a cubin / fatbin built from the SymPy fields of the scenario (see
 * csrc/qf_user.cuh) exporting the kernels qf_user_ghost, with the Dirichlet
 * data in the layout of the built-in families, and, with with_forcing,
 * qf_user_forcing, the projected momentum forcing rows the stage kernels add.  Replaces the
 * context's closed-form family for boundary data and forcing. */
int qf_user_scenario(qf_ctx* ctx, const void* image, size_t size, int32_t with_forcing);

/* Timing hooks (bench.py): events[2i], events[2i+1] (cudaEvent_t, timing
 * enabled) are recorded around RK stage i of every qf_step / qf_run step,
 * inside the captured run graph as event-record nodes, so per-stage kernel
 * times come from the same graph replay as the step time.  n = 0 clears. */
int qf_stage_events(qf_ctx* ctx, void* const* events, int32_t n);

/* Read (and optionally clear) the error word; synchronises `stream`. */
int qf_error(qf_ctx* ctx, uint32_t* bits, int32_t clear, void* stream);

/* Stream-ordered copy of `bytes` between device buffers (local, peer or
 * IPC-mapped; the initial halo trace rows of the fused transport). */
int qf_copy(void* dst, const void* src, size_t bytes, void* stream);

/* Fill n doubles with v (L2 flush for timing). */
int qf_fill(double* buf, size_t n, double v, void* stream);

/* Number of kernel launches issued through this library (all contexts). */
uint64_t qf_launch_count(void);
const char* qf_last_error(void);
/* 3: + qf_ghost_dev, qf_advance_time, qf_graph_* (round 2); 2: + qf_desc.uni */
int qf_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* QFSWE_H */
