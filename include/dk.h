/*
 * dk.h — C ABI of the B200-native deflated-GMRES hot path (paper_1510_02148_b200).
 *
 * This is the drop-in boundary for the reference `defkrylov` package's solver path.
 * The reference is pure Python; it exposes no FFI.  Each entry point below replaces a
 * Python call on that path (citations are into /root/reference/pkg/src/defkrylov/):
 *
 *   dk_op_create / dk_op_spmv        <- SparseMatrix + spmv          (sparse.py:21-106)
 *                                       Preconditioner.jacobi/apply  (krylov.py:33-43)
 *   dk_defl_create                   <- build_context                (deflation.py:71-89)
 *                                       dense_lu (SingularCoarseMatrix) (sparse.py:121-137)
 *   dk_defl_apply_p1/p2/reconstruct  <- DeflationContext.apply_p1/apply_p2/reconstruct
 *                                                                    (deflation.py:61-68)
 *   dk_gmres                         <- _run_cycles via gmres / pdgmres
 *                                                                    (krylov.py:107-266,
 *                                                                     physics.py:183-198)
 *   dk_dense_lu / dk_lu_solve        <- dense_lu / lu_solve          (sparse.py:109-145)
 *   dk_levelset_labels_device        <- subdomain_levelset_partition / levelset_partition
 *                                       (6-connected components + first-occurrence order)
 *                                                                    (physics.py:44-143)
 *
 * Conventions
 *  - Every function returns an int status: DK_OK (0), DK_EINVAL (1, a ValueError in the
 *    Python API), DK_ESINGULAR (2, SingularCoarseMatrix), DK_ECUDA (3), DK_EUNSUPPORTED (4).
 *    dk_last_error() returns a thread-local message for the last failing call.
 *  - Vector arguments (double / int32) may be HOST or DEVICE pointers (CUDA unified virtual
 *    addressing decides); the library copies them into its own HBM buffers.  Outputs are
 *    written to the pointer given, host or device.  Nothing is mutated in place.
 *  - An operator handle owns its device buffers (operator, Krylov basis V, scratch) and one
 *    CUDA stream.  Calls on one handle must be serialised (the reference is single-threaded
 *    per solve); different handles are independent.
 *  - There is no CPU fallback: without a usable sm_100 device every compute call fails with
 *    DK_ECUDA.
 */
#ifndef DK_H_
#define DK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DK_OK 0
#define DK_EINVAL 1
#define DK_ESINGULAR 2
#define DK_ECUDA 3
#define DK_EUNSUPPORTED 4

#define DK_MAX_DIAGONALS 7

#define DK_AP_A 0  /* A_p = A      (deflation.py:84, the default) */
#define DK_AP_AM 1 /* A_p = A M^-1 (deflation.py:50-51,84)       */

#define DK_WARNING_NONE 0
#define DK_WARNING_BREAKDOWN 1 /* SolveReport.warning == "breakdown" (krylov.py:192-194) */

typedef struct dk_op dk_op;     /* DIA operator + right preconditioner on one device   */
typedef struct dk_defl dk_defl; /* deflation context: labels, E^-1, x* (one operator)  */

typedef struct dk_solve_info {
  int32_t iterations;   /* SolveReport.iterations                                   */
  int32_t restarts;     /* SolveReport.restarts = max(cycles - 1, 0)                */
  int32_t cycles;       /* completed GMRES cycles                                   */
  int32_t converged;    /* SolveReport.converged                                    */
  int32_t warning;      /* DK_WARNING_*                                             */
  int32_t last_cols;    /* columns of the last cycle (ArnoldiData.m)                */
  int32_t reorths;      /* selective re-orthogonalisations performed                */
  int32_t kernel_launches; /* device kernels launched by this call                  */
  double final_relres;  /* true ||b - A x|| / ||b - A x0||                          */
  double solve_seconds; /* device time of the cycle loop (CUDA events)              */
} dk_solve_info;

/* ---- library ---------------------------------------------------------------------- */
const char* dk_last_error(void);
int dk_version(void);
/* Number of visible CUDA devices (0 on a CPU-only host, never an error). */
int dk_device_count(int32_t* count);
/* Device used by handles created afterwards on the calling thread (one process per GPU). */
int dk_set_device(int32_t device);

/* ---- operator --------------------------------------------------------------------- */
/* n cells; ndiag <= 7 diagonals with distinct offsets (any order); diags is ndiag x n
 * row-major with diags[k*n + i] = A[i, i + offsets[k]] (0 where i+offsets[k] is outside
 * [0, n)).  inv_diag (length n) is the Jacobi right preconditioner 1/a_ii, or NULL for the
 * identity preconditioner.  offsets is a host pointer. */
int dk_op_create(dk_op** op, int64_t n, int32_t ndiag, const int64_t* offsets,
                 const double* diags, const double* inv_diag);
int dk_op_destroy(dk_op* op);
/* Replace the right preconditioner: inv_diag (length n, host or device) or NULL = identity. */
int dk_op_set_precond(dk_op* op, const double* inv_diag);
/* Use an external CUDA stream (cudaStream_t passed as void*); NULL restores the handle's own. */
int dk_op_set_stream(dk_op* op, void* stream);
/* y = A x (bit-identical to a CSR row-ordered sum without FMA contraction). */
int dk_op_spmv(dk_op* op, const double* x, double* y);
/* Per-kernel-class timing with CUDA events on the handle's stream (graphs disabled while on). */
int dk_op_profile(dk_op* op, int32_t enable);
/* Reads accumulated per-class device milliseconds and launch counts; returns the number of
 * classes written (<= cap); names are static strings. */
int dk_op_profile_read(dk_op* op, int32_t cap, const char** names, double* ms, int64_t* launches,
                       double* bytes);

/* ---- deflation -------------------------------------------------------------------- */
/* col_of_cell[i] in [0, d) is the deflation column of cell i (indicator basis), or -1 when
 * the cell belongs to no column.  Assembles E = Z^T A_p Z on the device, factorises it —
 * Cholesky when E is symmetric and numerically positive definite, otherwise LU with partial
 * pivoting (DK_ESINGULAR if min |U_kk| < 1e-300, sparse.py:135-136) — forms E^-1 on the fp64
 * tensor cores, and the coarse solution x* = Z E^-1 Z^T b.  b may be NULL (x* = 0). */
int dk_defl_create(dk_defl** ctx, dk_op* op, const int32_t* col_of_cell, int32_t d,
                   int32_t ap_choice, const double* b);
/* Dense (non-indicator) basis, 1 <= d <= 64 (DK_EUNSUPPORTED beyond): Z is d x n row-major
 * (row k = basis vector k), host or device.  E = Z^T A_p Z, LU with partial pivoting
 * (DK_ESINGULAR as above), E^-1, x*  (deflation.py:71-89). */
int dk_defl_create_dense(dk_defl** ctx, dk_op* op, const double* Z, int32_t d, int32_t ap_choice,
                         const double* b);
/* Dense basis Z = V_rows Y from the operator's last Arnoldi cycle (harmonic.py:91-94: the
 * harmonic Ritz vectors), formed on the device; Y is rows x d column-major (host or device),
 * rows <= the last cycle's columns. */
int dk_defl_create_ritz(dk_defl** ctx, dk_op* op, const double* Y, int32_t rows, int32_t d,
                        int32_t ap_choice, const double* b);
int dk_defl_destroy(dk_defl* ctx);
int dk_defl_apply_p1(dk_defl* ctx, const double* v, double* out);  /* v - A_p Z E^-1 Z^T v */
int dk_defl_apply_p2(dk_defl* ctx, const double* v, double* out);  /* v - Z E^-1 Z^T A_p v */
int dk_defl_reconstruct(dk_defl* ctx, const double* xhat, double* out); /* x* + P2 xhat */
int dk_defl_x_star(dk_defl* ctx, double* out);
/* Copies E (d x d row-major, may be NULL) and E^-1 (may be NULL) out for inspection. */
int dk_defl_coarse(dk_defl* ctx, double* E, double* Einv);
/* Setup timings in ms: [assemble E, factorisation (Cholesky if E is SPD, else pivoted LU),
   forming E^-1, x*]. */
int dk_defl_setup_ms(dk_defl* ctx, double* ms4);
/* How y = E^-1 s is applied: *kind = 0 dense GEMV of E^-1, 1 packed symmetric tiles of E^-1,
   2 two passes over the nonzero tiles of W = L^-1 in nested-dissection order (SPD E),
   3 dense-basis multi-dot; *tiles = 32 x 32 tiles streamed per application. */
int dk_defl_coarse_kind(dk_defl* ctx, int32_t* kind, int64_t* tiles);

/* ---- solver ----------------------------------------------------------------------- */
/* Restarted right-preconditioned GMRES(m) on P1 A M^-1 (ctx != NULL) or A M^-1 (ctx NULL),
 * the reference's _run_cycles semantics (krylov.py:107-236).  x0 may be NULL (zeros).
 * hist and restart_of receive iterations+1 entries (capacity max_iters+1); hbar (may be
 * NULL) receives the last cycle's pristine Hessenberg, (m+1) x m column-major. */
int dk_gmres(dk_op* op, dk_defl* ctx, const double* b, const double* x0, int32_t m, double tol,
             int32_t max_iters, int32_t min_iters, double* x_out, double* hist,
             int32_t* restart_of, double* hbar, dk_solve_info* info);
/* Cycle control for multi-phase solves (RDGMRES: harmonic.py:163-178 switches the deflation
 * context after the first cycle).  in: stop after max_cycles cycles of this call (<= 0: no
 * limit); resume != 0 continues the counters / denominator below instead of starting a new
 * solve — with x0 == NULL from the operator's device-resident iterate of the previous call
 * (x_out of a deflated call is the reconstructed solution, the iterate stays on the device),
 * and the final relative residual keeps referring to the first call's x0.
 * out: the state to resume from. */
typedef struct dk_cycle_ctl {
  int32_t max_cycles;
  int32_t resume;
  int32_t iterations;
  int32_t cycles;
  int32_t warning;    /* 1: breakdown recorded */
  int32_t has_prev;   /* a previous restart residual exists */
  int32_t converged;  /* out */
  int32_t running;    /* out: another cycle would run */
  double denom;       /* convergence denominator: the first restart residual norm */
  double prev_beta;   /* the last restart residual norm */
} dk_cycle_ctl;
/* dk_gmres with cycle control; gram (may be NULL) receives V_{cols+1}^T V_cols of the last
 * cycle, (m+1) x m column-major (the re-orthogonalisation test's Gram matrix). */
int dk_gmres_ex(dk_op* op, dk_defl* ctx, const double* b, const double* x0, int32_t m, double tol,
                int32_t max_iters, int32_t min_iters, double* x_out, double* hist,
                int32_t* restart_of, double* hbar, double* gram, dk_solve_info* info,
                const dk_cycle_ctl* ctl_in, dk_cycle_ctl* ctl_out);
/* The restart loop of the last dk_gmres / dk_gmres_ex call (krylov.py:127 `while not converged
 * and it < max_iters`): host_syncs = host synchronisations inside the cycle loop; device_loop
 * = 1 when the cycles ran as the body of a CUDA conditional WHILE graph node, the device
 * deciding each restart (one host read after the loop), 0 when the host read the state after
 * every cycle (first cycle of a one-off solve, event-profiled solves, DK_NO_LOOP_GRAPH). */
int dk_op_solve_stats(dk_op* op, int32_t* host_syncs, int32_t* device_loop);
/* Copies basis vector i of the last cycle (normalised, length n) out; i <= last_cols. */
int dk_last_basis_vector(dk_op* op, int32_t i, double* out);

/* ---- deflation-vector construction ------------------------------------------------ */
/* Labels of the 6-connected components of equal `band` value inside each subdomain box
 * (px x py x pz near-equal boxes, remainders to the leading blocks; physics.py:57-78),
 * numbered by first occurrence in linear cell order ix + nx*(iy + ny*iz)
 * (physics.py:44-54, 119-143).  band is int64 per cell (-1 = zero-permeability band).
 * Writes labels[n], *ncomp, and comp_band[ncomp] (the band of each component, capacity n).
 * Computed on the current device: lock-free union-find whose roots are the component
 * minima, then a prefix scan over the roots.  Pointers may be host or device memory.
 * Without a device: DK_ECUDA (no host fallback). */
int dk_levelset_labels_device(int64_t nx, int64_t ny, int64_t nz, const int64_t* band,
                              int32_t px, int32_t py, int32_t pz, int64_t* labels,
                              int64_t* ncomp, int64_t* comp_band);

/* ---- dense LU (the reference's public LU helpers) ------------------------------------ */
/* dense_lu (sparse.py:121-137): P A = L U with partial pivoting on the device.  a is n x n
 * row-major; lu receives the combined factors in LAPACK getrf's layout (unit L strictly
 * below the diagonal, U on and above it, row-major) and piv[k] the 0-based row interchanged
 * with row k (scipy.linalg.lu_factor's convention).  *min_pivot (may be NULL) = min |U_kk|.
 * Returns DK_ESINGULAR when min |U_kk| < 1e-300 (factors are still written).
 * Host or device pointers. */
int dk_dense_lu(int64_t n, const double* a, double* lu, int32_t* piv, double* min_pivot);
/* lu_solve (sparse.py:140-145): X = A^-1 B from dk_dense_lu's factors (getrs: row
 * interchanges, unit-lower then upper triangular solves on the device).  b and x are
 * n x nrhs row-major (numpy's stacked right-hand sides); x may alias b. */
int dk_lu_solve(int64_t n, const double* lu, const int32_t* piv, int64_t nrhs, const double* b,
                double* x);

/* ---- operator assembly ------------------------------------------------------------- */
/* TPFA pressure operator on the device (testbed.py:133-211 arithmetic): diags_out is 7 x n
 * for offsets (-nx*ny, -nx, -1, 0, 1, nx, nx*ny), b_out is n.  q (sources) may be NULL.
 * Dirichlet ghost faces are applied in the given order; face ids 0..5 = xmin, xmax, ymin,
 * ymax, zmin, zmax (zmax is the reference's "top").  Host or device pointers. */
int dk_assemble_tpfa(int32_t nx, int32_t ny, int32_t nz, double dx, double dy, double dz,
                     const double* kx, const double* ky, const double* kz, const double* q,
                     int32_t nfaces, const int32_t* face_ids, const double* face_values,
                     double boundary_perm, double* diags_out, double* b_out);

#ifdef __cplusplus
}
#endif
#endif /* DK_H_ */
