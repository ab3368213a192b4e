// dk_launch.h — host-side launchers for the device kernels (one per kernel family).
#pragma once
#include <cuda_runtime.h>

#include <climits>
#include <string>
#include <vector>

#include "dk_internal.cuh"

namespace dk {

// ---- per-device properties (dk_device.cu) ----
constexpr int kMaxDevices = 64;
int current_device();
// SM count of the current device (cached per ordinal; grids are sized from it)
int num_sms();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize, bytes) for `fn` on the current device,
// once per (kernel, device) and size (static + dynamic above 48 KB needs it).  0 or a cuda
// error code.
int smem_optin(const void* fn, size_t bytes);

// Stencil modes of launch_stencil.
enum StencilMode {
  ST_APPLY = 0,  // out = A (M^-1 (scale * v))          (krylov.py:159 / deflation.py:50-51)
  ST_RESID = 1,  // out = b - A v                        (krylov.py:128, :222)
  ST_IDENT = 2,  // out = v  (restriction of v only)     (deflation.py:62 Z^T v)
};

struct RunMap {            // label-segmented restriction metadata
  const int* lab;          // guarded labels
  const int* tile_run_off; // [ntiles+1] first run id of each tile
  double* run_part;        // [nruns] per-run partial sums, label-major (slot order)
  const int* lab_run_ptr;  // [d+1] CSR: slots of each label's runs, in run order
  const int* run_slot;     // [nruns] slot of each run (unlabelled runs after the labelled)
  int d;
  const int* long_ids;     // columns with more than kShortRuns runs (summed by a warp)
  int nlong;
  const int* s_pos;        // nullptr, or the position of label L in s (coarse ordering)
  const void* pf_base;     // nullptr, or a constant stream the next kernels read (the W tile
  unsigned long long pf_bytes;  // store): the ring stencil prefetches it into L2 as it goes
};
constexpr int kShortRuns = 16;

// w = (mode) ; if rm != nullptr also run sums of w.  pre: apply the Jacobi inverse.
// scale (device scalar or nullptr) multiplies v first.  gate (device int or nullptr).
// wait (ST_APPLY only; nullptr: off): start on *wait != 0 instead of the predecessor grid's
// completion (the scale is read after it), wait for the predecessor only before exiting.
void launch_stencil(int mode, bool pre, bool write, const Dia& A, long long n_pad, const double* v,
                    const double* scale, const double* b, double* out, const RunMap* rm,
                    const int* gate, cudaStream_t s, const unsigned* wait = nullptr,
                    const double* gsig = nullptr, int ng = 0);
// Split-iteration stencil (symmetric 7-point operators only; sym7_supported): as
// launch_stencil(ST_APPLY, ..., write, rm) and also the run sums of a = A_p^T v (A v, times
// M^-1 when am) into run_part2.  Returns false when the operator is not supported.
bool sym7_supported(const Dia& A);
void launch_stencil_split(bool pre, bool am, const Dia& A, long long n_pad, const double* v,
                          const double* scale, double* out, const RunMap& rm, double* run_part2,
                          const int* gate, cudaStream_t s, const unsigned* wait,
                          const double* gsig, int ng);
// s[s_pos[L]] (s[L] without s_pos) = sum of run partials of label L, fixed order; with
// run_part2, also out2[L] = the sums of run_part2 (label order).
void launch_restrict_final(const RunMap& rm, double* s_out, const int* gate, cudaStream_t s,
                           const double* run_part2 = nullptr, double* out2 = nullptr);
// y = M x, M d x d row-major with leading dimension ld.
void launch_gemv(const double* M, int d, int ld, const double* x, double* y, const int* gate,
                 cudaStream_t s);

// Compact prolongation map of a deflation context (k_prolong_setup).
struct Prolong {
  const int* lab;             // guarded labels
  const double* own;          // guarded: sum of a cell's coefficients into its own column
  const int2* flab;           // guarded: the first two foreign labels of a cell's row (-1: none)
  const double2* fco;         // guarded: their summed coefficients
  const unsigned char* mask;  // guarded: diagonals whose label is a third (or later) foreign one
  const double* az;           // dense basis: rows A_p Z_k (stride azs), k < dz
  long long azs;
  int dz;
};
// deflation kind of a projection: none, indicator (labels), dense basis rows
enum DeflKind { DK_NONE = 0, DK_LABELS = 1, DK_DENSE = 2 };
void launch_prolong_setup(bool am, const Dia& A, const int* lab, long long n_pad, double* own,
                          int2* flab, double2* fco, unsigned char* mask,
                          unsigned long long* nmasked, cudaStream_t s);

enum ProjectMode { PJ_ITER = 0, PJ_RESTART = 1, PJ_PLAIN = 2, PJ_REDOTS = 3,
                   // split iteration: DOTS = h' = U^T w and the Gram column (no prolongation,
                   // no control); FIX = w -= A_p Z y, ||w||^2, C y slices, then the H column
                   PJ_DOTS = 4, PJ_FIX = 5 };
// w_out = w_in - A_p Z y (defl) ; ITER: dots h = V^T w, ||w_out||^2
// -> H col j + re-orthogonalisation test; RESTART: ||w_out||^2 -> restart test;
// REDOTS: corr = V^T u for the second Gram-Schmidt pass.  G = grid width (fixed per op).
void launch_project(int mode, int defl, bool am, const Dia& A, const Prolong& lab, const double* yc,
                    const double* w_in, double* w_out, const double* V, long long vstride,
                    int nvec, long long n_pad, double* part, int G, const Scal& sc, int j,
                    const int* gate, cudaStream_t s, bool pdl = true);
// dense deflation basis (rows of stride zs): s_k = Z_k . v for k < nz; y[k * ystride] = s_k,
// or y = Einv s (nz x nz, ld) when Einv != nullptr.  ticket: a zeroed device counter.
void launch_zdots(const double* v, const double* Z, long long zs, int nz, long long n_pad,
                  double* part, int G, unsigned int* ticket, const double* Einv, int ld,
                  double* y, long long ystride, const int* gate, cudaStream_t s);
// out = mode 0: xs + (xh - sum_k y_k Z_k) ; 1: sum_k y_k Z_k ; 2: xh - sum_k y_k Z_k
void launch_dense_recon(const double* Z, long long zs, int nz, const double* y, const double* xs,
                        const double* xh, double* out, long long n_pad, int mode,
                        cudaStream_t s);
// out_j = sum_{i < nrows} Y[i + j * nrows] * sigma_i * R_i for j < nout (rows R of stride rs,
// outputs of stride os): Z = V_m Y from the stored, lazily normalised Arnoldi basis
void launch_combine_rows(const double* R, long long rs, const double* sigma, int nrows,
                         const double* Y, int nout, double* out, long long os, long long n_pad,
                         cudaStream_t s);
// u = w - sum coef_i u_i (+ corr dots, norm) or the re-orthogonalisation pass.
void launch_gs(bool reorth, const double* w_in, double* u_out, const double* V, long long vstride,
               int nvec, long long n_pad, double* part, int G, const Scal& sc, int j,
               const int* gate, bool fuse, cudaStream_t s);
// the whole k_gs grid is co-resident: the second Gram-Schmidt pass may run inside it
bool gs_can_fuse(int G, const Scal& sc);
void launch_cycle_end(const Scal& sc, cudaStream_t s);
// Small problems: the cycle's m Arnoldi steps in one persistent cooperative grid (one 2048-cell
// chunk per block).  cycle_small_ok: shape and co-residency check (DK_NO_SMALL: never).
constexpr int kMaxCycleSmall = 128;
bool cycle_small_ok(long long n_pad, int m, int d);
void launch_cycle_small(int defl, bool pre, bool am, const Dia& A, const Dia& Aam,
                        const Prolong& P, const RunMap& rm, const double* Einv, int ld, double* V,
                        long long vstride, long long n_pad, double* part, double* yg,
                        const Scal& sc, cudaStream_t s);
void launch_xupdate(const Dia& A, double* x, const double* V, long long vstride, long long n_pad,
                    const Scal& sc, cudaStream_t s);
// out = xs + (xh - y[lab])   (deflation.py:64-68)
void launch_recon(const int* lab, const double* y, const double* xs, const double* xh, double* out,
                  long long n_pad, cudaStream_t s);
// out = y[lab] (0 where lab < 0)
void launch_bcast(const int* lab, const double* y, double* out, long long n_pad, cudaStream_t s);
// out = v - y[lab]
void launch_sub_bcast(const int* lab, const double* y, const double* v, double* out,
                      long long n_pad, cudaStream_t s);
// *dst = ||v||_2 over n_pad cells (deterministic).
void launch_norm(const double* v, long long n_pad, double* part, int G, unsigned int* ticket,
                 double* dst, cudaStream_t s);
void launch_init_state(const Scal& sc, double tol, int m, int max_iters, int min_iters,
                       cudaStream_t s);
void launch_resume_state(const Scal& sc, int iterations, int cycles, int warning, int has_prev,
                         double denom, double prev_beta, cudaStream_t s);
// device-decided restart loop: arm the cycle budget; the WHILE body's last kernel sets the
// loop condition (another cycle: still running and budget left)
void launch_loop_arm(const Scal& sc, int cycles, cudaStream_t s);
void launch_loop_cond(const Scal& sc, cudaGraphConditionalHandle h, cudaStream_t s);

// ---- set-up on the device (dk_setup.cu) ----
int device_levelset_labels(long long nx, long long ny, long long nz, const long long* band_in,
                           int px, int py, int pz, long long* labels_out, long long* ncomp,
                           long long* comp_band_out, cudaStream_t s, std::string& err);
int device_assemble_tpfa(int nx, int ny, int nz, double dx, double dy, double dz,
                         const double* kx, const double* ky, const double* kz, const double* q,
                         int nfaces, const int* face_ids, const double* face_values, double bperm,
                         double* diags_out, double* b_out, cudaStream_t s, std::string& err);

// ---- coarse operator (dk_coarse.cu) ----
// symmetric coarse solve from the packed upper tile triangle of E^-1 (32 x 32 tiles)
long long symv_tiles(int d);
void launch_symv_pack(const double* Einv, int d, int ld, double* P, cudaStream_t s);
void launch_symv(const double* P, int d, const double* x, double* rowpart, double* colpart,
                 double* y, const int* gate, cudaStream_t s);
void launch_symv_reduce(int d, const double* rowpart, const double* colpart,
                        const int* seg_ptr, const int* seg_slot, double* y, const int* gate,
                        cudaStream_t s);
void symv_segments(int d, std::vector<int>& ptr, std::vector<int>& slots);
int coarse_is_symmetric(const double* E, int d, int ld, cudaStream_t s);
// E (d x d, ld) = Z^T A_p Z, deterministic.  Returns 0 or a cuda error code.
int build_coarse(const Dia& A, bool am, const int* lab, long long n_pad, const RunMap& rm,
                 double* E, int ld, double* scratch_q, cudaStream_t s);
// In-place P E = L U with partial pivoting (LAPACK getrf layout, row-major; piv[k] = row
// interchanged with row k).  dominant: the pivot-free path (columns diagonally dominant).
// *min_pivot receives min |U_kk| (host).  Returns 0 or a cuda error code.
int lu_factor(double* E, int d, int ld, int* piv, bool dominant, double* min_pivot,
              cudaStream_t s);
// X <- U^-1 L^-1 P X for a d x ncols row-major block (getrs).
void lu_solve_rows(const double* E, int d, int ld, const int* piv, double* X, int ldx,
                   int ncols, bool lower_fill, cudaStream_t s);
// In-place LU with partial pivoting of E, then Einv = U^-1 L^-1 P.  *min_pivot receives
// min |U_kk| (host).  Returns 0 or a cuda error code.
int lu_and_inverse(double* E, int d, int ld, double* Einv, int* piv, double* min_pivot,
                   float* ms_lu, float* ms_inv, cudaStream_t s);
// C = beta C + alpha op(A) op(B) on the fp64 tensor cores (dk_dense.cu).  ta: A stored K x M;
// tb: B stored N x K; tri 0/1/2 = all / lower / upper tiles; kshift (INT_MIN = off): B[k][j]
// is structurally zero for k < j + kshift; kstop (INT_MIN = off): zero for k >= j + kstop
// (rounded up to the CTA tile: tile column c0 stops its K loop at c0 + BN + kstop).
void gemm_mma(bool ta, bool tb, const double* A, int lda, const double* B, int ldb, double* C,
              int ldc, int M, int N, int K, double alpha, double beta, int tri, int kshift,
              cudaStream_t s, int kstop = INT_MIN);
// Symmetric positive definite E (in L, overwritten): Cholesky, W = L^-1 (into W), then
// E^-1 = W^T W written back into L (full).  *min_diag_sq = min L_kk^2 (NaN if not SPD); when
// it is below 1e-280 the inverse is not formed and the caller falls back to LU.
// form_inverse = false stops after W = L^-1 (W holds it, L the factor).
int spd_inverse(double* L, int d, int ld, double* W, double* min_diag_sq, float* ms_fac,
                float* ms_inv, cudaStream_t s, bool form_inverse = true, bool clear_w = true);
struct NDTreeNode;
// W = L^-1 of an SPD E~ in nested-dissection order, node by node along the tree (W zeroed
// on entry; E~'s separator blocks are overwritten).  *min_diag_sq as for spd_inverse.
// With E's pattern (host CSR in label order) and iperm (label -> position), L_SD = E_SD W_D^T
// is the sparse product instead of dense GEMMs.
int nd_tree_inverse(double* E, int d, int ld, const std::vector<NDTreeNode>& tree, double* W,
                    double* min_diag_sq, cudaStream_t s, const std::vector<int>* gptr = nullptr,
                    const std::vector<int>* gcol = nullptr,
                    const std::vector<int>* iperm = nullptr);
// X = W^T W (full, d x d) for lower-triangular W
void lauum_into(const double* W, int d, int ld, double* X, cudaStream_t s);

// ---- coarse solve through W = L^-1 in nested-dissection order (dk_profile.cu) ----
// a tile stream of k_tgemv: nt 32 x 32 tiles grouped by output block (trow ascending)
struct TileGemv {
  const double* T = nullptr;   // [tiles][16][32][2]
  const int* tid = nullptr;    // storage index of stream tile t (nullptr: t itself)
  bool trans = false;          // the stream applies the stored tiles transposed
  const int* trow = nullptr;   // output block per tile
  const int* tcol = nullptr;   // input block per tile
  const int* rfirst = nullptr; // first warp of each output block
  const int* rslot = nullptr;  // partial-slot base of a block split across warps
  const int* rnp = nullptr;    // warps holding pieces of the block
  double* part = nullptr;      // [slots][32] pieces of split blocks (sentinel when empty)
  long long nt = 0;
  int nw = 0;                  // warps holding tiles (min(kTgGrid * warps per CTA, nt))
  int nrows = 0;
  // L2 persisting window over the tile store (win_bytes == 0: none; the tiles then load with
  // an evict-last hint)
  void* win_base = nullptr;
  size_t win_bytes = 0;
  const int* split_rows = nullptr;  // output blocks split across warps (NOSPIN finish)
  int nsplit = 0;
  unsigned* bar = nullptr;  // [count, generation] of the in-kernel grid barrier (fused pass 1)
  // constant streams of the kernel that follows the coarse solve (the projection's per-cell
  // prolongation inputs): this pass prefetches them into L2 while DRAM is otherwise idle
  const char* pf[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  unsigned long long pf_bytes[5] = {0, 0, 0, 0, 0};
  int npf = 0;
};
struct TileGemvHost {
  long long nt = 0;
  int nw = 0;
  std::vector<int> trow, tcol, rfirst, rslot, rnp;
  std::vector<int> tid;  // empty: tiles stored in stream order
  std::vector<int> split_rows;
  int nslots = 1;
};
// E's off-diagonal pattern (CSR, host)
int coarse_pattern(const double* E, int d, int ld, std::vector<int>& ptr, std::vector<int>& col,
                   cudaStream_t s);
// a node of the dissection tree in the new order: subtree [t0, s1), separator [s0, s1)
// (descendants [t0, s0) are the children's subtrees, which E does not couple)
struct NDTreeNode {
  int t0, s0, s1;
  std::vector<int> kids;  // indices of the children (post-order: children come first)
};
// level-structure nested dissection of the pattern graph: perm[new] = old; the tree in
// post-order (root last) when tree != nullptr
void nd_order(int d, const std::vector<int>& ptr, const std::vector<int>& col,
              std::vector<int>& perm, std::vector<NDTreeNode>* tree = nullptr);
// 32 x 32 tiles of W's structural row profile under perm (upper bound of the stream)
long long nd_profile_tiles(int d, const std::vector<int>& ptr, const std::vector<int>& col,
                           const std::vector<int>& perm);
void launch_permute_sym(const double* E, int d, int ld, const int* perm, double* out,
                        cudaStream_t s);
void launch_unpermute_sym(const double* X, int d, int ld, const int* perm, double* out, int ldo,
                          cudaStream_t s);
// nonzero tiles of W (row profile fW) as the two streams t = W s~ and y~ = W^T t; the tiles
// are stored once (pass 1's order), pass 2 visits them by block column and applies them
// transposed
int profile_streams(const double* W, int d, int ld, const std::vector<int>& fW,
                    TileGemvHost& p1, TileGemvHost& p2, cudaStream_t s);
// metadata to the device; with pack, W's tiles packed into g.T (allocated by the caller,
// nt x 8 KB).  A transposed stream (h.tid set) shares the tiles of the packed one.
int upload_stream(const double* W, int d, int ld, bool pack, const TileGemvHost& h, TileGemv& g,
                  cudaStream_t s);
void free_stream(TileGemv& g, cudaStream_t s);
// y[scatter ? scatter[i] : i] = (sum over the stream's tiles) for rows i < d
void launch_tgemv(const TileGemv& g, const double* x, double* y, const int* scatter, int d,
                  const int* gate, cudaStream_t s);
// kernels one launch_tgemv issues (1: spinning finisher; 2: NOSPIN pass + k_tg_finish)
int tgemv_launches(const TileGemv& g);
// Pass 1 with the column sums s = Z^T w folded in (k_restrict_final's arithmetic, then a grid
// barrier, inside the cooperative spinning pass); otherwise k_restrict_final + launch_tgemv.
// s_out = s~ (rm.s_pos order), the pass's x.  Returns the kernels launched.
int launch_tgemv_restrict(const TileGemv& g, const RunMap& rm, double* s_out, double* y,
                          int d, const int* gate, cudaStream_t s);
int tgemv_restrict_launches(const TileGemv& g);
// f[r] = first nonzero column of row r (<= r) of a d x d matrix (device)
void launch_row_first_nz(const double* X, int d, int ld, int* f, cudaStream_t s);

}  // namespace dk
