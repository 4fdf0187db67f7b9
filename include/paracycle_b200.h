/*
 * paracycle_b200 -- C ABI of the B200-native PTL-cycled parabolic-operator path.
 *
 * This is the drop-in boundary under the reference Python package's operator
 * API.  Every entry point returns an int status (PC_OK == 0);
 * the message of the last failure of the calling thread is pc_last_error().
 * No torch types cross this boundary: plain pointers, sizes and doubles.
 *
 * Reference interfaces replaced (file:line in /root/reference):
 *   pc_grid_create / pc_field_*     mesh.Grid / mesh.Field / mesh.pinned_mask
 *                                   (pkg/src/paracycle/mesh.py:89-239, :311-324)
 *   pc_op_create_scalar,
 *   pc_op_create_viscous            operators.ScalarDiffusionConfig +
 *                                   apply_scalar_diffusion
 *   pc_op_create_aligned,
 *   pc_op_freeze                    operators.AlignedConductionConfig +
 *                                   apply_aligned_conduction
 *   pc_op_apply                     DiffusionOperator.apply / F(u)
 *   pc_op_euler_dt                  operators.estimate_euler_dt
 *   pc_ptl                          ptl.compute_ptl
 *   pc_sts_count / pc_sts_table     schemes.rkg2_iteration_count,
 *                                   rkg2_coefficients, RKL2 analogues
 *   pc_step_sts                     schemes.step_rkl2 / step_rkg2
 *   pc_step_euler                   schemes.step_euler
 *   pc_step_be, pc_pcg_solve        schemes.step_backward_euler + linsolve.pcg_solve
 *                                   with build_jacobi
 *   pc_cycle                        ptl.cycle_operator; small scalar
 *                                   grids run the whole loop in one persistent launch
 *   pc_op_set_preconditioner        linsolve.Preconditioner kind:
 *                                   point Jacobi (PC1) or the r-line block Jacobi that
 *                                   stands in for the sequential ILU0 (PC2, :201-222)
 *
 * Device layout: every field component is one contiguous fp64 array
 * [n0 + 2][n1][n2] (axis 2 = phi fastest) whose first and last axis-0 planes
 * are ghost planes used only by slab decomposition; host buffers are either
 * the reference Field layout (AoS, component innermost, PC_LAYOUT_AOS) or
 * component-major (PC_LAYOUT_SOA), interior only.
 */
#ifndef PARACYCLE_B200_H
#define PARACYCLE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum pc_status {
  PC_OK = 0,
  PC_E_INVALID = 1,    /* bad argument / contract violation (ValueError)           */
  PC_E_INDEFINITE = 2, /* PCG breakdown p^T A p <= 0, or non-positive Jacobi diag  */
  PC_E_DIVERGED = 3,   /* NaN/Inf in the PCG residual                               */
  PC_E_BLOWUP = 4,     /* non-finite STS stage; pc_last_error_info() = stage        */
  PC_E_CAP = 5,        /* max_cycles reached; records hold the partial report       */
  PC_E_CUDA = 6,
  PC_E_NCCL = 7,
  PC_E_DOMAIN = 8,     /* non-positive T0 for aligned conduction      */
  PC_E_NOTCONV = 9     /* PCG hit max_iter inside a cycle                           */
};

enum pc_layout { PC_LAYOUT_AOS = 0, PC_LAYOUT_SOA = 1 };
enum pc_scheme { PC_RKL2 = 0, PC_RKG2 = 1, PC_BE = 2, PC_EULER = 3 };
enum pc_floor { PC_FLOOR_EULER = 0, PC_FLOOR_FRACTION = 1 };

typedef struct pc_ctx pc_ctx;
typedef struct pc_grid pc_grid;
typedef struct pc_field pc_field;
typedef struct pc_op pc_op;

/* one row of ptl.CycleReport (CSV :391-392) */
typedef struct pc_cycle_record {
  int64_t cycle;    /* 1-based */
  double dt;        /* cycle time step                                  */
  double ptl_raw;   /* raw PTL, or +inf when unlimited                  */
  double relres;    /* final relative residual (BE), 0 for STS          */
  int32_t limited;  /* 1 if the PTL was limited (finite)                */
  int32_t iters;    /* STS stage count s, or PCG iterations             */
} pc_cycle_record;

const char* pc_last_error(void);
int64_t pc_last_error_info(void); /* e.g. the blow-up stage */
int pc_version(void);

/* ---- context: one per GPU (rank).  nranks > 1 enables r-slab decomposition
 * over NCCL; nccl_uid points to an ncclUniqueId (128 bytes) or NULL. */
int pc_ctx_create(int device, int nranks, int rank, const void* nccl_uid, pc_ctx** out);
int pc_ctx_destroy(pc_ctx* ctx);
/* test hook: rank `rank` of an nranks r-slab decomposition WITHOUT a
   communicator -- collectives are skipped (local reductions, no halo
   exchange) and the caller sets the axis-0 ghost planes with
   pc_field_set_ghost; used to check the slab kernels on one GPU */
int pc_ctx_create_detached(int device, int nranks, int rank, pc_ctx** out);
/* slab decomposition axis of a multi-rank context: 0 = r-slabs (default,
   axis-0 ghost planes), 2 = phi-slabs (BASELINE C4's split: each rank owns
   phi columns [k0, k0 + n) of every plane and keeps one ghost column on each
   side, exchanged over a periodic NCCL ring).  Set before creating grids. */
int pc_ctx_set_decomposition(pc_ctx* ctx, int axis);
int pc_ctx_sync(pc_ctx* ctx);
int pc_nccl_unique_id(void* out128); /* fills a fresh ncclUniqueId */

/* ---- grid.  shape = LOCAL (n0, n1, n2).  iflags (PC_GRID_NFLAGS ints):
 *  [0..2] periodic per axis, [3..8] pinned lo/hi per axis (Dirichlet),
 *  [9] ghost_lo0 (a lower axis-0 neighbour rank exists), [10] ghost_hi0,
 *  [11] global n0, [12] global axis-0 offset of this slab, [13] spherical,
 *  [14] phi-slab (local columns 0 and n2-1 are ghost columns: pinned, zero
 *  weight), [15] global n2, [16] global phi offset of local column 1.
 * tables: pc_grid_table_size(shape) doubles in the order documented in
 * paper_2403_01004_b200/geometry.py (TABLE_ORDER); 2-D tables carry axis-0
 * ghost rows (n0 + 2 rows). */
#define PC_GRID_NFLAGS 17
int64_t pc_grid_table_size(const int64_t shape[3]);
int pc_grid_create(pc_ctx* ctx, const int64_t shape[3], const int32_t* iflags,
                   const double* tables, int64_t ntables, pc_grid** out);
int pc_grid_destroy(pc_grid* g);

/* ---- fields (device-resident, SoA) */
int pc_field_create(pc_grid* g, int ncomp, pc_field** out);
int pc_field_destroy(pc_field* f);
int pc_field_upload(pc_field* f, const double* host, int layout);
int pc_field_download(const pc_field* f, double* host, int layout);
/* asynchronous variants on the context's copy stream (no reference
   counterpart; they let split_advance move the next operator's state while
   the current one computes).  They start after the work already queued on the
   context; every later library call using the field waits for the copy on
   the device.  The host buffer must stay valid and unchanged until
   pc_field_wait(f) returns (or the field is destroyed, which waits). */
int pc_field_upload_async(pc_field* f, const double* host, int layout);
int pc_field_download_async(pc_field* f, double* host, int layout);
int pc_field_wait(pc_field* f);
/* axis-0 planes [i0, i0 + n) of every component, SoA [ncomp][n][n1][n2] (full-size
   parity checks read a window without moving the whole field) */
int pc_field_download_planes(const pc_field* f, int64_t i0, int64_t n, double* host);
int pc_field_copy(pc_field* dst, const pc_field* src);
int pc_field_fill(pc_field* f, double value);
int pc_field_exchange_halo(pc_field* f); /* axis-0 ghost planes (no-op on 1 rank) */
/* number of owned nodes x components failing a domain test, summed over all
   ranks: PC_TEST_POSITIVE counts !(x > 0), PC_TEST_NONNEG !(x >= 0),
   PC_TEST_FINITE !isfinite(x) (NaN fails all three).  Replaces the host-side
   `np.any(~(rho > 0))` validation of the operator constructors
   (reference: SPEC.md:89-93, ValueError for rho <= 0) with one pass over HBM. */
enum pc_field_test { PC_TEST_POSITIVE = 0, PC_TEST_NONNEG = 1, PC_TEST_FINITE = 2 };
int pc_field_count(const pc_field* f, int test, int64_t* count);
/* write ghost plane -1 (side 0) or n0 (side 1) of every component from a host
   SoA plane [ncomp][n1][n2] */
int pc_field_set_ghost(pc_field* f, int side, const double* host);
/* phi-slab test hook: write both ghost columns of every component from host
   [ncomp][2][n0 * n1] (side 0 = column 0, side 1 = column n2 - 1) */
int pc_field_set_ghost_cols(pc_field* f, const double* host);
/* pin / unpin a host buffer so uploads and downloads run at full PCIe speed */
int pc_host_register(void* ptr, size_t bytes);
int pc_host_unregister(void* ptr);
/* page-locked host allocations (the Python layer caches them for downloads) */
int pc_host_alloc(size_t bytes, void** out);
int pc_host_free(void* ptr);

/* ---- operators.
 * scalar:  F = (1/rho) div(D grad u), D = nu*rho nodal (field) or D_const when
 *          D == NULL; rho == NULL means 1; vector_metric rotates 3-component
 *          spherical vectors.
 * aligned: F = pref/rho div(c b b.grad T), c = kappa0 f_c(r_i) T0^{5/2},
 *          T0 floored at T_floor; fc_table (n0 + 2 doubles incl. ghosts) or NULL. */
int pc_op_create_scalar(pc_grid* g, int ncomp, int vector_metric, double D_const,
                        const pc_field* D, const pc_field* rho, pc_op** out);
/* viscosity F = (1/rho) div(nu rho grad u) with a density FIELD and constant
 * nu: the face coefficient nu*rho is formed per node from rho (no D array). */
int pc_op_create_viscous(pc_grid* g, int ncomp, int vector_metric, double nu, const pc_field* rho,
                         pc_op** out);
int pc_op_create_aligned(pc_grid* g, const pc_field* bhat, const pc_field* rho,
                         double pref, double kappa0, const double* fc_table,
                         double T_floor, pc_op** out);
/* freeze the lagged state (aligned: c from T0; T0 ignored for scalar) and
 * evaluate the Gershgorin bound and the Jacobi diagonal. */
int pc_op_freeze(pc_op* op, const pc_field* T0);
int pc_op_destroy(pc_op* op);
/* BE+PCG preconditioner: PC_PC_JACOBI (SPEC PC1, default) or PC_PC_LINE_R
   (block Jacobi over r-lines, Thomas solves; aligned operator, one rank) --
   a GPU substitute for the SPEC's sequential ILU0 (PC2) */
#define PC_PC_JACOBI 0
#define PC_PC_LINE_R 1
int pc_op_set_preconditioner(pc_op* op, int pc);
/* lagged-T0 cadence of an aligned operator inside pc_cycle: 0 = frozen by the
   caller once per outer step (SPEC default), 1 = re-frozen at T0 := u at the
   start of every cycle (coefficients and Gershgorin bound; SPEC.md:385
   "per-cycle refresh available via config") */
int pc_op_set_refresh(pc_op* op, int per_cycle);
int pc_op_apply(pc_op* op, const pc_field* u, pc_field* F);
int pc_op_euler_dt(pc_op* op, double* dt_euler);
/* -J_ii per node (pinned rows 0), the Jacobi building block */
int pc_op_diagonal(pc_op* op, pc_field* out);

/* ---- PTL (Eq. 5).  *limited = 0 means unlimited (ptl = +inf). kidx = AoS
 * linear index of the |F| maximum (ties -> lowest). */
int pc_ptl(pc_grid* g, const pc_field* u, const pc_field* F, double eps_rel, int check_all,
           double* ptl, int* limited, int64_t* kidx);

/* ---- STS counts and tables (host only, no GPU needed) */
int pc_sts_count(int kind, double dt, double dt_euler, int make_odd);
/* out[5*(k-1) + {0..4}] = mu_k, nu_k, (1-mu_k)-nu_k, mut_k*dt, gam_k*dt */
int pc_sts_table(int kind, int s, double dt, double* out);

/* ---- steps (u updated in place) */
int pc_step_sts(pc_op* op, pc_field* u, double dt, int kind, int s, const pc_field* y0);
int pc_step_euler(pc_op* op, pc_field* u, double dt);
int pc_step_be(pc_op* op, pc_field* u, double dt, double tol, int max_iter,
               int* iters, double* relres, int* converged);
/* general Jacobi-PCG on A x = (diag_a - dt J) x = b, diag_a == NULL means I */
int pc_pcg_solve(pc_op* op, double dt, const pc_field* diag_a, const pc_field* b,
                 pc_field* x, double tol, int max_iter, int* iters, double* relres,
                 int* converged);

/* ---- the cycle loop (ptl.cycle_operator).  dt_euler <= 0 uses the frozen
 * operator's bound.  rec receives min(n, rec_cap) records.  use_ptl: 0 no PTL
 * (one cycle of the whole outer_dt), 1 dynamic re-evaluation every cycle
 * (PAPER.md:77), 2 static first-PTL cycling (the first cycle's PTL reused by
 * every cycle). */
int pc_cycle(pc_op* op, pc_field* u, double outer_dt, int scheme, int make_odd,
             double tol, int max_iter, double eps_rel, int check_all, int use_ptl,
             int floor_mode, double floor_fraction, int64_t max_cycles, double dt_euler,
             pc_cycle_record* rec, int64_t rec_cap, int64_t* n_rec);

/* ---- seeded synthetic inputs in HBM (configs.py recipes, bit-identical):
 * tables are over the GLOBAL grid (prof/ir3/rho: n0 values, c2/st: n1,
 * acc: ncomp x n1 x n2); noise = configs.hash_normal(seed, stream, global index). */
int pc_gen_temperature(pc_field* T, uint64_t seed, int stream, double sigma, const double* prof);
int pc_gen_dipole(pc_field* b, uint64_t seed, int stream0, double eps, const double* ir3, const double* c2,
                  const double* st);
int pc_gen_harmonic(pc_field* v, const double* acc, double checker);
int pc_gen_radial(pc_field* f, const double* tab);

/* ---- instrumentation (enabled by pc_ctx_enable_timing): device time of the
 * fused STS stage kernels (k >= 2) and of the PCG iteration kernels, their
 * launch count, and the total number of kernels this context launched. */
int pc_ctx_stats(pc_ctx* ctx, double* stage_ms, int64_t* stage_launches, int64_t* launches_total);
int pc_ctx_reset_stats(pc_ctx* ctx);
/* per hot-loop kind (0 scalar/vector STS stages k >= 2, 1 aligned STS stages,
 * 2 scalar PCG iterations, 3 aligned PCG iterations, 4/5 the fused stage-1+2
 * launch of the 7-point march without/with the u1 write, 6/7 the same for the
 * aligned TMA march): device ms, launches and cell-updates (local cells x
 * stages / iterations; the fused launches count both stages) */
int pc_ctx_stats_kind(pc_ctx* ctx, int kind, double* ms, int64_t* launches, int64_t* cell_updates);
int pc_ctx_enable_timing(pc_ctx* ctx, int on);
/* CUDA events on the context stream: record mark id (0..15); elapsed ms */
int pc_ctx_mark(pc_ctx* ctx, int id);
int pc_ctx_elapsed(pc_ctx* ctx, int id0, int id1, double* ms);

#ifdef __cplusplus
}
#endif
#endif
