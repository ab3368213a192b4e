// dk_dense.cu — dense fp64 set-up algebra for the coarse operator E (d x d, row-major).
//
//   * k_dgemm_mma: C = beta C + alpha op(A) op(B) on the fp64 tensor cores (DMMA, mma.sync
//     m16n8k4), 128 x 128 CTA tile, 8 warps of 64 x 32, K in steps of 16 through a 3-stage
//     cp.async ring.  Options used by the factorisations: operand transposition, lower / upper
//     tile triangle only, and a per-tile K start for a lower-triangular B (structural zeros
//     are skipped, not multiplied).
//   * spd_inverse: E^-1 of a symmetric positive definite E (the TPFA case: E = Z^T A Z with A
//     SPD) by blocked Cholesky E = L L^T (lower tiles only), W = L^-1 (forward substitution
//     exploiting W's triangle) and E^-1 = W^T W (upper tiles, K from the tile column): d^3/2
//     multiply-adds instead of the d^3 of LU + two triangular solves.  The reference
//     factorises E with partial-pivoting LU (sparse.py:121-145, deflation.py:86-87); the
//     inverse is the same matrix up to rounding, and any E that is not numerically SPD goes
//     through lu_and_inverse (dk_coarse.cu), which keeps the reference's pivoting and
//     singularity semantics exactly.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <mutex>
#include <vector>

#include "dk_launch.h"

namespace dk {

namespace {

constexpr int GM = 128, GK = 16, GSTAGES = 3;
constexpr int LDK = GK + 4;  // K-contiguous operand rows in shared memory (conflict-free)

// operand tile of extent EXT (M or N) x GK per stage: K-contiguous [EXT][LDK] or
// MN-contiguous [GK][EXT + 4] (both strides = 4 mod 16 doubles: conflict-free fragments)
template <int EXT>
__host__ __device__ constexpr int op_doubles() {
  return EXT * LDK > GK * (EXT + 4) ? EXT * LDK : GK * (EXT + 4);
}
template <int NT>
__host__ __device__ constexpr int gemm_smem() {
  return GSTAGES * (op_doubles<GM>() + op_doubles<32 * NT>()) * (int)sizeof(double);
}

__device__ __forceinline__ unsigned sm32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void cp16(double* dst, const double* src, int bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sm32(dst)), "l"(src),
               "r"(bytes));
}

// 8-byte variant for operands that are not 16-byte aligned (odd column offsets / strides)
__device__ __forceinline__ void cp8(double* dst, const double* src, int bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sm32(dst)), "l"(src),
               "r"(bytes));
}

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void dmma(double (&c)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, "
      "{%0,%1,%2,%3};\n"
      : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

// Stage one GK-deep slice of an operand tile of extent EXT.  KCONT: the global operand is
// stored with K contiguous (rows = the M or N index), else with M/N contiguous (rows = K).
// `mn_lim` bounds the M/N index, `k_lim` the K index; invalid halves are zero-filled.
template <bool KCONT, int EXT, bool A8>
__device__ __forceinline__ void stage_operand(double* s, const double* g, int ldg, int mn0,
                                              int mn_lim, int k0, int k_lim) {
  constexpr int LDM = EXT + 4;
#pragma unroll
  for (int i = 0; i < EXT / 32; ++i) {
    const int e = threadIdx.x + 256 * i;  // 8 * EXT chunks of 16 B per slice
    int mn, k, so;
    if (KCONT) {
      mn = e >> 3;
      k = (e & 7) * 2;
      so = mn * LDK + k;
    } else {
      k = e / (EXT / 2);
      mn = (e % (EXT / 2)) * 2;
      so = k * LDM + mn;
    }
    const int gmn = mn0 + mn, gk = k0 + k;
    int valid;
    const double* src;
    if (KCONT) {
      valid = (gmn < mn_lim) ? min(2, max(0, k_lim - gk)) : 0;
      src = g + (long long)gmn * ldg + gk;
    } else {
      valid = (gk < k_lim) ? min(2, max(0, mn_lim - gmn)) : 0;
      src = g + (long long)gk * ldg + gmn;
    }
    if (A8) {  // the pair's second element sits at +1 (K) or +1 (M/N) in both layouts
      cp8(s + so, valid >= 1 ? src : g, valid >= 1 ? 8 : 0);
      cp8(s + so + 1, valid >= 2 ? src + 1 : g, valid >= 2 ? 8 : 0);
    } else {
      cp16(s + so, valid ? src : g, valid * 8);
    }
  }
}

// C[M x N] = beta C + alpha op(A) op(B), alpha != 0 (C enters the accumulators as
// (beta / alpha) C).  TA: A is stored K x M (op = transpose); TB: B is stored N x K.
// CTA tile 128 x (32 NT), 8 warps of 64 x (8 NT).  tri: 0 all tiles, 1 tiles touching the
// lower triangle, 2 the upper.  With beta == 0, C may alias A (N <= tile width) or B
// (M <= 128): a CTA then reads only the rows / columns it writes, and every operand load
// completes before the epilogue.  kshift != INT_MIN: B is lower triangular in the sense
// B[k][j] == 0 for k < j + kshift, so tile column c0 starts its K loop at c0 + kshift
// (rounded down to GK).
template <bool TA, bool TB, int NT, bool A8>
__global__ void __launch_bounds__(256, NT == 2 ? 2 : 1)
    k_dgemm_mma(const double* A, int lda, const double* B, int ldb, double* C, int ldc, int M,
                int N, int K, double alpha, double beta, int tri, int kshift, int kstop,
                double* P) {
  constexpr int BN = 32 * NT, LDMA = GM + 4, LDMB = BN + 4;
  constexpr int OPA = op_doubles<GM>(), OPB = op_doubles<BN>();
  extern __shared__ __align__(128) double smem[];
  const int r0 = blockIdx.y * GM, c0 = blockIdx.x * BN;
  if (tri == 1 && c0 > r0 + GM - 1) return;
  if (tri == 2 && r0 > c0 + BN - 1) return;
  int kbeg = 0;
  if (kshift != INT_MIN) {
    kbeg = c0 + kshift;
    kbeg = kbeg < 0 ? 0 : (kbeg / GK) * GK;
  }
  int kend = K;
  if (kstop != INT_MIN) kend = min(K, c0 + BN + kstop);  // op(B)[k][j] == 0 for k >= j + kstop
  int nk = (kend > kbeg) ? (kend - kbeg + GK - 1) / GK : 0;
  if (P != nullptr) {  // split K: this CTA's share of the tile's K steps, raw partial sums
    const int chunk = (nk + gridDim.z - 1) / gridDim.z;
    const int it0 = min(nk, (int)blockIdx.z * chunk);
    nk = min(nk, it0 + chunk) - it0;
    kbeg += it0 * GK;
    beta = 0.0;
    alpha = 1.0;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp >> 2) * 64, wn = (warp & 3) * (8 * NT);
  double acc[4][NT][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[i][j][q] = 0.0;
  if (beta != 0.0) {  // C enters the accumulators (its loads overlap the operand prologue)
    const double sc = beta / alpha;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = r0 + wm + i * 16 + g + 8 * h;
        if (row >= M) continue;
        const double* crow = C + (long long)row * ldc;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const int col = c0 + wn + j * 8 + 2 * t;
          if (A8) {
            if (col < N) acc[i][j][2 * h] = sc * crow[col];
            if (col + 1 < N) acc[i][j][2 * h + 1] = sc * crow[col + 1];
          } else if (col + 1 < N) {
            const double2 cv = *reinterpret_cast<const double2*>(crow + col);
            acc[i][j][2 * h] = sc * cv.x;
            acc[i][j][2 * h + 1] = sc * cv.y;
          } else if (col < N) {
            acc[i][j][2 * h] = sc * crow[col];
          }
        }
      }
  }

  auto load = [&](int it) {
    double* sa = smem + (it % GSTAGES) * (OPA + OPB);
    double* sb = sa + OPA;
    const int k0 = kbeg + it * GK;
    stage_operand<!TA, GM, A8>(sa, A, lda, r0, M, k0, K);
    stage_operand<TB, BN, A8>(sb, B, ldb, c0, N, k0, K);
  };
#pragma unroll
  for (int it = 0; it < GSTAGES - 1; ++it) {
    if (it < nk) load(it);
    cp_commit();
  }
  for (int it = 0; it < nk; ++it) {
    cp_wait<GSTAGES - 2>();
    __syncthreads();
    if (it + GSTAGES - 1 < nk) load(it + GSTAGES - 1);
    cp_commit();
    const double* sa = smem + (it % GSTAGES) * (OPA + OPB);
    const double* sb = sa + OPA;
#pragma unroll
    for (int kk = 0; kk < GK; kk += 4) {
      double af[4][2], bf[NT];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int m = wm + i * 16 + g;
        if (!TA) {
          af[i][0] = sa[m * LDK + kk + t];
          af[i][1] = sa[(m + 8) * LDK + kk + t];
        } else {
          af[i][0] = sa[(kk + t) * LDMA + m];
          af[i][1] = sa[(kk + t) * LDMA + m + 8];
        }
      }
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int n = wn + j * 8 + g;
        bf[j] = TB ? sb[n * LDK + kk + t] : sb[(kk + t) * LDMB + n];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma(acc[i][j], af[i][0], af[i][1], bf[j]);
    }
  }
  cp_wait<0>();
  if (P != nullptr) {  // partials of split z: [z][M][N]
    double* Pz = P + (long long)blockIdx.z * M * N;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = r0 + wm + i * 16 + g + 8 * h;
        if (row >= M) continue;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          const int col = c0 + wn + j * 8 + 2 * t;
          if (col < N) Pz[(long long)row * N + col] = acc[i][j][2 * h];
          if (col + 1 < N) Pz[(long long)row * N + col + 1] = acc[i][j][2 * h + 1];
        }
      }
    return;
  }
  // epilogue: c0,c1 at (g, 2t..2t+1), c2,c3 at (g+8, 2t..2t+1) of each 16 x 8 tile
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int row = r0 + wm + i * 16 + g + 8 * h;
      if (row >= M) continue;
      double* crow = C + (long long)row * ldc;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        const int col = c0 + wn + j * 8 + 2 * t;
        if (A8) {
          if (col < N) crow[col] = alpha * acc[i][j][2 * h];
          if (col + 1 < N) crow[col + 1] = alpha * acc[i][j][2 * h + 1];
        } else if (col + 1 < N) {
          *reinterpret_cast<double2*>(crow + col) =
              make_double2(alpha * acc[i][j][2 * h], alpha * acc[i][j][2 * h + 1]);
        } else if (col < N) {
          crow[col] = alpha * acc[i][j][2 * h];
        }
      }
    }
  }
}

// split-K epilogue: C = alpha (beta/alpha C + sum_z P[z]) over the tiles the GEMM writes, the
// partials summed in split order (deterministic)
__global__ void k_splitk_reduce(const double* __restrict__ P, int S, int M, int N, double* C,
                                int ldc, double alpha, double beta, int tri, int BN) {
  const long long total = (long long)M * N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(e / N), col = (int)(e % N);
    const int r0 = (row / GM) * GM, c0 = (col / BN) * BN;
    if (tri == 1 && c0 > r0 + GM - 1) continue;
    if (tri == 2 && r0 > c0 + BN - 1) continue;
    double v = beta != 0.0 ? (beta / alpha) * C[(long long)row * ldc + col] : 0.0;
    for (int z = 0; z < S; ++z) v += P[z * total + e];
    C[(long long)row * ldc + col] = alpha * v;
  }
}

// K splits of a GEMM whose tile grid cannot fill the SMs (the nested-dissection tree's
// separator products: a few hundred rows, K up to d): enough CTAs for two per SM, at least
// 256 K per split (DK_NO_SPLITK: one CTA per tile)
int splitk_count(int M, int N, int K, int BN) {
  static const bool off = getenv("DK_NO_SPLITK") != nullptr;
  if (off) return 1;
  const long long tiles = (long long)((N + BN - 1) / BN) * ((M + GM - 1) / GM);
  const long long want = 2ll * num_sms();
  if (tiles >= want || K < 512) return 1;
  long long S = (want + tiles - 1) / tiles;
  S = std::min<long long>(S, K / 256);
  S = std::min<long long>(S, 32);
  return S < 2 ? 1 : (int)S;
}

template <bool TA, bool TB, int NT, bool A8>
void launch_mma_a(const double* A, int lda, const double* B, int ldb, double* C, int ldc, int M,
                  int N, int K, double alpha, double beta, int tri, int kshift, int kstop,
                  cudaStream_t s) {
  smem_optin((const void*)k_dgemm_mma<TA, TB, NT, A8>, gemm_smem<NT>());
  const int S = splitk_count(M, N, K, 32 * NT);
  double* P = nullptr;
  if (S > 1 && cudaMallocAsync(&P, (size_t)S * M * N * sizeof(double), s) != cudaSuccess) {
    cudaGetLastError();
    P = nullptr;
  }
  dim3 grid((N + 32 * NT - 1) / (32 * NT), (M + GM - 1) / GM, P ? S : 1);
  k_dgemm_mma<TA, TB, NT, A8><<<grid, 256, gemm_smem<NT>(), s>>>(A, lda, B, ldb, C, ldc, M, N,
                                                                K, alpha, beta, tri, kshift,
                                                                kstop, P);
  if (P) {
    const long long total = (long long)M * N;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 8ll * num_sms());
    k_splitk_reduce<<<blocks, 256, 0, s>>>(P, S, M, N, C, ldc, alpha, beta, tri, 32 * NT);
    cudaFreeAsync(P, s);
  }
}

// operands at odd column offsets or with odd strides take the 8-byte copy path
template <bool TA, bool TB, int NT>
void launch_mma(const double* A, int lda, const double* B, int ldb, double* C, int ldc, int M,
                int N, int K, double alpha, double beta, int tri, int kshift, int kstop,
                cudaStream_t s) {
  const bool a8 = (((uintptr_t)A | (uintptr_t)B | (uintptr_t)C) & 15) != 0 ||
                  ((lda | ldb | ldc) & 1) != 0;
  if (a8)
    launch_mma_a<TA, TB, NT, true>(A, lda, B, ldb, C, ldc, M, N, K, alpha, beta, tri, kshift,
                                   kstop, s);
  else
    launch_mma_a<TA, TB, NT, false>(A, lda, B, ldb, C, ldc, M, N, K, alpha, beta, tri, kshift,
                                    kstop, s);
}

template <bool TA, bool TB>
void launch_mma_nt(int nt, const double* A, int lda, const double* B, int ldb, double* C,
                   int ldc, int M, int N, int K, double alpha, double beta, int tri, int kshift,
                   int kstop, cudaStream_t s) {
  if (nt == 2)
    launch_mma<TA, TB, 2>(A, lda, B, ldb, C, ldc, M, N, K, alpha, beta, tri, kshift, kstop, s);
  else
    launch_mma<TA, TB, 4>(A, lda, B, ldb, C, ldc, M, N, K, alpha, beta, tri, kshift, kstop, s);
}

// ---- Cholesky pieces ---------------------------------------------------------------------
constexpr int DB = 64;    // diagonal block (one CTA factorises and inverts it)
constexpr int DNW = 8;    // warps of the diagonal-block kernel
constexpr int GB = 256;   // blocks are grouped for the trailing updates (rank GB)
constexpr int kDiagSmem = (DB * (DB + 1) + 5 * DB + 2) * (int)sizeof(double);

// 1/v from the hardware approximation refined by two Newton steps (error ~1 ulp); on the
// critical path of every elimination step, where a correctly rounded division costs several
// times more
__device__ __forceinline__ double fast_rcp(double v) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(v));
  double e = fma(-v, r, 1.0);
  r = fma(r, e, r);
  e = fma(-v, r, 1.0);
  return fma(r, e, r);
}

template <int N>
__device__ __forceinline__ double sel(const double (&v)[N], int k) {
  double r = v[0];
#pragma unroll
  for (int i = 1; i < N; ++i) r = (k == i) ? v[i] : r;
  return r;
}

// One CTA of 32 DNW threads: the nb x nb (nb <= DB) diagonal block at (k0, k0) of A (lower
// triangle, already updated by the previous blocks) -> L11 = chol(block) -> L11^-1, written
// to W[k0.., k0..] (full block, zeros above the diagonal).  L11 itself is not needed later:
// the block column below becomes A21 L11^-T and W is built from L11^-1.
// Warp w keeps rows RPW w .. RPW w + RPW - 1, lane l the columns l + 32 j, in registers.  The
// block is factorised as L~ D L~^T (unit L~, right-looking, one barrier per column: the
// owners of column c+1 publish it, and the owner of the next pivot its reciprocal, as soon as
// step c has updated them; warps whose rows are all done sit out), then X = L~^-1 by a
// right-looking sweep over rows, and L11^-1 = D^-1/2 X.  pmin[blk] = min pivot D_cc
// (= L_cc^2); NaN if a pivot is not positive.
// jobs != nullptr: a batch of independent blocks, CTA b takes (k0, nb) = jobs[b] and
// writes pmin[blk + b].
__global__ void __launch_bounds__(32 * DNW, 1) k_chol_diag(const double* __restrict__ A, int ld,
                                                          int k0, int nb, double* __restrict__ W,
                                                          double* __restrict__ pmin, int blk,
                                                          const int2* __restrict__ jobs) {
  constexpr int RPW = DB / DNW, CPL = DB / 32;
  if (jobs != nullptr) {
    k0 = jobs[blockIdx.x].x;
    nb = jobs[blockIdx.x].y;
    blk += blockIdx.x;
  }
  extern __shared__ __align__(16) double dsm[];
  double(*lt)[DB + 1] = reinterpret_cast<double(*)[DB + 1]>(dsm);  // L~ (unit lower)
  double* buf = dsm + DB * (DB + 1);                                // 2 x DB columns
  double* piv = buf + 2 * DB;                                       // D
  double* rbuf = piv + DB;                                          // 2 x DB rows
  double* ipb = rbuf + 2 * DB;                                      // 2 reciprocals
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31, rb = RPW * w;
  double a[RPW][CPL];
#pragma unroll
  for (int i = 0; i < RPW; ++i)
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int r = rb + i, c = lane + 32 * j;
      a[i][j] = (r < nb && c <= r) ? A[(long long)(k0 + r) * ld + k0 + c] : 0.0;
    }
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < RPW; ++i) buf[rb + i] = a[i][0];
  if (tid == 0) ipb[0] = fast_rcp(a[0][0]);
  __syncthreads();
  for (int c = 0; c < nb; ++c) {
    const int n1 = c + 1;
    if (rb + RPW - 1 > c) {  // warp-uniform: this warp still has rows below the pivot
      const double* col = buf + (c & 1) * DB;
      const double ip = ipb[c & 1];
      double lr[RPW], lc[CPL];
#pragma unroll
      for (int i = 0; i < RPW; ++i) lr[i] = col[rb + i] * ip;
#pragma unroll
      for (int j = 0; j < CPL; ++j) lc[j] = col[lane + 32 * j];
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        if (32 * j + 31 <= c) continue;  // warp-uniform
        const int cc = lane + 32 * j;
#pragma unroll
        for (int i = 0; i < RPW; ++i)
          if (cc > c && cc <= rb + i) a[i][j] = fma(-lr[i], lc[j], a[i][j]);
      }
      if (lane < RPW && rb + lane > c) lt[rb + lane][c] = sel(lr, lane);
      if (n1 < nb && lane == (n1 & 31)) {
        double* nxt = buf + (n1 & 1) * DB;
        const int q = n1 >> 5;
#pragma unroll
        for (int i = 0; i < RPW; ++i) {
          const double v = sel(a[i], q);
          nxt[rb + i] = v;
          if (rb + i == n1) ipb[n1 & 1] = fast_rcp(v);
        }
      }
    }
    if (tid == 0) piv[c] = buf[(c & 1) * DB + c];
    __syncthreads();
  }
  if (tid < 32) {
    double m = INFINITY;
    bool bad = false;
    for (int c = tid; c < nb; c += 32) {
      const double p = piv[c];
      if (!(p > 0.0)) bad = true;
      m = fmin(m, p);
    }
    bad = __any_sync(0xffffffffu, bad);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (tid == 0) pmin[blk] = bad ? __longlong_as_double(0x7ff8000000000000ll) : m;
  }
  // X = L~^-1: row i0 is final once rows < i0 are applied; its owners publish it
  double x[RPW][CPL];
#pragma unroll
  for (int i = 0; i < RPW; ++i)
#pragma unroll
    for (int j = 0; j < CPL; ++j) x[i][j] = (rb + i == lane + 32 * j) ? 1.0 : 0.0;
  if (w == 0)
#pragma unroll
    for (int j = 0; j < CPL; ++j) rbuf[lane + 32 * j] = x[0][j];
  __syncthreads();
  for (int i0 = 0; i0 < nb; ++i0) {
    const int n1 = i0 + 1;
    if (rb + RPW - 1 > i0) {
      const double* row = rbuf + (i0 & 1) * DB;
      double xr[CPL], lv[RPW];
#pragma unroll
      for (int j = 0; j < CPL; ++j) xr[j] = row[lane + 32 * j];
#pragma unroll
      for (int i = 0; i < RPW; ++i) lv[i] = (rb + i > i0) ? lt[rb + i][i0] : 0.0;
#pragma unroll
      for (int j = 0; j < CPL; ++j) {
        if (32 * j > i0) continue;  // X[i0][col] == 0 for col > i0 (warp-uniform)
#pragma unroll
        for (int i = 0; i < RPW; ++i) x[i][j] = fma(-lv[i], xr[j], x[i][j]);
      }
      if (n1 < nb && n1 / RPW == w) {
        double* nxt = rbuf + (n1 & 1) * DB;
        const int q = n1 % RPW;
#pragma unroll
        for (int j = 0; j < CPL; ++j) {
          double v = x[0][j];
#pragma unroll
          for (int i = 1; i < RPW; ++i) v = (q == i) ? x[i][j] : v;
          nxt[lane + 32 * j] = v;
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < RPW; ++i) {
    const int r = rb + i;
    if (r >= nb) continue;
    const double sc = 1.0 / sqrt(piv[r]);
#pragma unroll
    for (int j = 0; j < CPL; ++j) {
      const int c = lane + 32 * j;
      if (c < nb) W[(long long)(k0 + r) * ld + k0 + c] = (c <= r) ? x[i][j] * sc : 0.0;
    }
  }
}

// f[r] = first column with E[r][c] != 0 (c <= r; r when none): the row profile.  Cholesky
// keeps it (no fill left of the first nonzero), so panel products touch only the rows whose
// profile reaches the panel.  One warp per row, 32 columns per step.
__global__ void k_row_first_nz(const double* __restrict__ E, int d, int ld, int* __restrict__ f) {
  const int lane = threadIdx.x & 31;
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < d;
       r += gridDim.x * (blockDim.x >> 5)) {
    int first = r;
    for (int c0 = 0; c0 < r; c0 += 32) {
      const int c = c0 + lane;
      const unsigned nz = __ballot_sync(0xffffffffu, c < r && E[(long long)r * ld + c] != 0.0);
      if (nz) {
        first = c0 + __ffs(nz) - 1;
        break;
      }
    }
    if (lane == 0) f[r] = first;
  }
}

// X[j][i] = X[i][j] for i < j (copy the upper triangle onto the lower), 32 x 32 tiles.
__global__ void __launch_bounds__(256) k_mirror_upper(double* __restrict__ X, int d, int ld) {
  __shared__ double tile[32][33];
  const int bi = blockIdx.y, bj = blockIdx.x;
  if (bj < bi) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const int i = bi * 32 + r, j = bj * 32 + tx;
    tile[r][tx] = (i < d && j < d) ? X[(long long)i * ld + j] : 0.0;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int j = bj * 32 + r, i = bi * 32 + tx;  // destination (j, i), source (i, j)
    if (i < d && j < d && i < j) X[(long long)j * ld + i] = tile[tx][r];
  }
}

}  // namespace

void launch_row_first_nz(const double* X, int d, int ld, int* f, cudaStream_t s) {
  k_row_first_nz<<<num_sms() * 4, 256, 0, s>>>(X, d, ld, f);
}

// X = W^T W (full) for lower-triangular W
void lauum_into(const double* W, int d, int ld, double* X, cudaStream_t s) {
  gemm_mma(true, false, W, ld, W, ld, X, ld, d, d, d, 1.0, 0.0, 2, 0, s);
  const int nt = (d + 31) / 32;
  k_mirror_upper<<<dim3(nt, nt), 256, 0, s>>>(X, d, ld);
}

int g_gemm_nt = 2;  // n8 tiles per warp of the set-up GEMM (2: 128 x 64 CTA tiles, 2 per SM)

void gemm_mma(bool ta, bool tb, const double* A, int lda, const double* B, int ldb, double* C,
              int ldc, int M, int N, int K, double alpha, double beta, int tri, int kshift,
              cudaStream_t s, int kstop) {
  if (M <= 0 || N <= 0) return;
  // N <= tile width: one tile column (the in-place TRSM relies on it)
  const int nt = (N <= 64) ? 2 : (N <= 128) ? 4 : g_gemm_nt;
  if (ta) {
    if (tb) launch_mma_nt<true, true>(nt, A, lda, B, ldb, C, ldc, M, N, K, alpha, beta, tri, kshift, kstop, s);
    else launch_mma_nt<true, false>(nt, A, lda, B, ldb, C, ldc, M, N, K, alpha, beta, tri, kshift, kstop, s);
  } else {
    if (tb) launch_mma_nt<false, true>(nt, A, lda, B, ldb, C, ldc, M, N, K, alpha, beta, tri, kshift, kstop, s);
    else launch_mma_nt<false, false>(nt, A, lda, B, ldb, C, ldc, M, N, K, alpha, beta, tri, kshift, kstop, s);
  }
}

// high-priority stream of the device for the factorisation's look-ahead chain
static cudaStream_t side_stream() {
  static std::mutex mu;
  static cudaStream_t st[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (!st[dev & 63]) {
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    cudaStreamCreateWithPriority(&st[dev & 63], cudaStreamNonBlocking, greatest);
  }
  return st[dev & 63];
}

int spd_inverse(double* L, int d, int ld, double* W, double* min_diag_sq, float* ms_fac,
                float* ms_inv, cudaStream_t s, bool form_inverse, bool clear_w) {
  smem_optin((const void*)k_chol_diag, kDiagSmem);
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&e2);
  cudaEventRecord(e0, s);
  const int nblk = (d + DB - 1) / DB;
  auto at = [&](double* X, int r, int c) { return X + (long long)r * ld + c; };
  double* dpmin = nullptr;
  cudaMallocAsync(&dpmin, nblk * sizeof(double), s);
  if (clear_w) cudaMemsetAsync(W, 0, (size_t)d * ld * sizeof(double), s);
  // row profile -> reach(t) = 1 + the last row whose profile starts left of column t: the rows
  // of L that can be nonzero in columns < t lie in [t, reach(t))
  std::vector<int> reach(d + 1, 0);
  {
    int* df = nullptr;
    std::vector<int> f(d);
    cudaMallocAsync(&df, (size_t)d * sizeof(int), s);
    k_row_first_nz<<<num_sms() * 4, 256, 0, s>>>(L, d, ld, df);
    cudaMemcpyAsync(f.data(), df, (size_t)d * sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(df, s);
    cudaStreamSynchronize(s);
    std::vector<int> last(d, -1);  // last row whose profile starts at column c
    for (int r = 0; r < d; ++r) last[f[r]] = std::max(last[f[r]], r);
    int mx = -1;
    for (int t = 1; t <= d; ++t) {
      mx = std::max(mx, last[t - 1]);
      reach[t] = std::max(t, mx + 1);
    }
  }
  // 1. E = L L^T, right-looking by DB-wide blocks in groups of GB columns, with look-ahead.
  //    The panel chain of a group runs on a high-priority side stream: per block, the
  //    diagonal block is factorised and inverted by one CTA (L11^-1 lands on W's diagonal),
  //    the block column below becomes L21 = A21 L11^-T (in place: one tile column, each CTA
  //    owns its rows), and the group's remaining columns receive the block's rank-DB update.
  //    When a group completes, the side stream applies its rank-GB update to the NEXT group's
  //    columns only (a), so that group's chain can start at once, while the main stream
  //    updates the rest of the trailing lower triangle (b).  Every product is limited to the
  //    rows inside the profile (reach).
  cudaStream_t side = side_stream();
  const int ngroups = (d + GB - 1) / GB;
  std::vector<cudaEvent_t> ev_chain(ngroups), ev_b(ngroups);
  for (int g = 0; g < ngroups; ++g) {
    cudaEventCreateWithFlags(&ev_chain[g], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_b[g], cudaEventDisableTiming);
  }
  cudaEvent_t ev_start, ev_side_done;
  cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&ev_side_done, cudaEventDisableTiming);
  cudaEventRecord(ev_start, s);
  cudaStreamWaitEvent(side, ev_start, 0);
  for (int g = 0; g < ngroups; ++g) {
    const int G0 = g * GB, gend = (d - G0 < GB) ? d : G0 + GB;
    for (int K0 = G0; K0 < gend; K0 += DB) {  // chain(g), side stream
      const int nb = (d - K0 < DB) ? d - K0 : DB, Kend = K0 + nb;
      k_chol_diag<<<1, 32 * DNW, kDiagSmem, side>>>(L, ld, K0, nb, W, dpmin, K0 / DB, nullptr);
      const int rq = reach[Kend] - Kend;  // rows below the block inside the profile
      if (Kend >= d || rq <= 0) continue;
      gemm_mma(false, true, at(L, Kend, K0), ld, at(W, K0, K0), ld, at(L, Kend, K0), ld, rq, nb,
               nb, 1.0, 0.0, 0, INT_MIN, side);
      if (Kend < gend)
        gemm_mma(false, true, at(L, Kend, K0), ld, at(L, Kend, K0), ld, at(L, Kend, Kend), ld, rq,
                 gend - Kend, nb, -1.0, 1.0, 0, INT_MIN, side);
    }
    cudaEventRecord(ev_chain[g], side);
    if (gend >= d) break;
    const int R = reach[gend], na = (d - gend < GB) ? d - gend : GB, rb0 = gend + na;
    // (a) the next group's columns, after the previous trailing update (b) wrote them
    if (g > 0) cudaStreamWaitEvent(side, ev_b[g - 1], 0);
    if (R > gend)
      gemm_mma(false, true, at(L, gend, G0), ld, at(L, gend, G0), ld, at(L, gend, gend), ld,
               R - gend, std::min(na, R - gend), gend - G0, -1.0, 1.0, 0, INT_MIN, side);
    // (b) the rest of the trailing lower triangle, main stream, once the group's panel is final
    cudaStreamWaitEvent(s, ev_chain[g], 0);
    if (R > rb0)
      gemm_mma(false, true, at(L, rb0, G0), ld, at(L, rb0, G0), ld, at(L, rb0, rb0), ld, R - rb0,
               R - rb0, gend - G0, -1.0, 1.0, 1, INT_MIN, s);
    cudaEventRecord(ev_b[g], s);
  }
  cudaEventRecord(ev_side_done, side);
  cudaStreamWaitEvent(s, ev_side_done, 0);
  std::vector<double> pm(nblk);
  cudaMemcpyAsync(pm.data(), dpmin, nblk * sizeof(double), cudaMemcpyDeviceToHost, s);
  cudaEventRecord(e1, s);
  cudaStreamSynchronize(s);
  cudaFreeAsync(dpmin, s);
  for (int g = 0; g < ngroups; ++g) {
    cudaEventDestroy(ev_chain[g]);
    cudaEventDestroy(ev_b[g]);
  }
  cudaEventDestroy(ev_start);
  cudaEventDestroy(ev_side_done);
  double mn = INFINITY;
  for (double v : pm) mn = (v != v || mn != mn) ? NAN : fmin(mn, v);
  *min_diag_sq = mn;
  if (!(mn >= 1e-280)) {  // not numerically SPD: the caller takes the LU path
    cudaEventElapsedTime(ms_fac, e0, e1);
    *ms_inv = 0.f;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    return (int)cudaGetLastError();
  }
  // 2. W = L^-1, right-looking by block rows: W[q, 0:K0] = L_qq^-1 W[q, 0:K0] (in place: one
  //    tile row); inside a group, the group's remaining block rows receive q's contribution;
  //    when the group completes, W[gend:, 0:gend] -= L[gend:, group] W[group, 0:gend]
  //    (W[G0 + kk][j] == 0 for kk < j - G0: the K loop of tile column j starts there)
  for (int q = 0; q < nblk; ++q) {
    const int K0 = q * DB, nb = (d - K0 < DB) ? d - K0 : DB, Kend = K0 + nb, rest = d - Kend;
    const int G0 = (K0 / GB) * GB, gend = (d - G0 < GB) ? d : G0 + GB;
    if (K0 > 0)
      gemm_mma(false, false, at(W, K0, K0), ld, at(W, K0, 0), ld, at(W, K0, 0), ld, nb, K0, nb,
               1.0, 0.0, 0, INT_MIN, s);
    if (rest <= 0) break;
    // L's rows below the profile reach are zero in these columns: no contribution
    const int rq = std::min(reach[Kend], Kend < gend ? gend : d) - Kend;
    if (rq <= 0) continue;
    if (Kend < gend)
      gemm_mma(false, false, at(L, Kend, K0), ld, at(W, K0, 0), ld, at(W, Kend, 0), ld, rq, Kend,
               nb, -1.0, 1.0, 0, -K0, s);
    else
      gemm_mma(false, false, at(L, Kend, G0), ld, at(W, G0, 0), ld, at(W, Kend, 0), ld, rq, Kend,
               Kend - G0, -1.0, 1.0, 0, -G0, s);
  }
  // 3. E^-1 = W^T W: upper tiles into L's storage (A = W^T, B = W lower: K from the tile
  //    column), then the lower triangle mirrored
  if (form_inverse) lauum_into(W, d, ld, L, s);
  cudaEventRecord(e2, s);
  cudaStreamSynchronize(s);
  cudaEventElapsedTime(ms_fac, e0, e1);
  cudaEventElapsedTime(ms_inv, e1, e2);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  return (int)cudaGetLastError();
}


// ---- SPD inverse factor along a nested-dissection tree ------------------------------------
// E~ (nested-dissection order) has, for every tree node N with separator S and descendants D
// (the children's subtrees, which E~ does not couple), the block structure
//     E~_T = [[E_D, E_SD^T], [E_SD, E_S]],  E_D = blockdiag(E_C),
// so with W_C = L_C^-1 of every child already formed (post-order):
//     L_SD = E_SD W_D^T,  S = E_S - L_SD L_SD^T = L_S L_S^T,  W_S = L_S^-1,
//     W_SD = -W_S L_SD W_D,
// i.e. W = L^-1 is built node by node with GEMMs over the node's own rows only: O(sum |S|
// |D|^2) instead of the O(d^3) of the dense factorisation.  Leaves (no descendants) are
// factorised and inverted in one batched launch.  E~ is overwritten by the Schur complements
// on the separator diagonal blocks; W must be zero on entry.
// L_SD = E_SD W_D^T with E_SD sparse (the label graph: a few neighbours per separator row):
// X[r][jj] = sum over the row's descendant neighbours k (ascending) of E~[s0 + r][k] W[t0 + jj][k]
// (W is zero right of its diagonal and across children).  One block per row of W_D (read
// once, L1-resident), fixed order per output.
__global__ void __launch_bounds__(128) k_lsd_sparse(const double* __restrict__ E,
                                                    const double* __restrict__ W, int ld, int s0,
                                                    int ns, int t0, int nd,
                                                    const int* __restrict__ rp,
                                                    const int* __restrict__ ck,
                                                    double* __restrict__ X, int ldx) {
  for (int jj = blockIdx.x; jj < nd; jj += gridDim.x) {
    const double* Wr = W + (long long)(t0 + jj) * ld;
    for (int r = threadIdx.x; r < ns; r += blockDim.x) {
      const double* Er = E + (long long)(s0 + r) * ld;
      double acc = 0.0;
      for (int i = rp[r]; i < rp[r + 1]; ++i) {
        const int k = ck[i];
        acc = fma(__ldg(Er + k), __ldg(Wr + k), acc);
      }
      X[(long long)r * ldx + jj] = acc;
    }
  }
}

int nd_tree_inverse(double* E, int d, int ld, const std::vector<NDTreeNode>& tree, double* W,
                    double* min_diag_sq, cudaStream_t s, const std::vector<int>* gptr,
                    const std::vector<int>* gcol, const std::vector<int>* iperm) {
  smem_optin((const void*)k_chol_diag, kDiagSmem);
  auto at = [&](double* X, int r, int c) { return X + (long long)r * ld + c; };
  // leaves: batched diagonal factorisation + inversion
  std::vector<int2> jobs;
  long long xmax = 0;
  int nbig = 0;
  for (const auto& n : tree) {
    const int ns = n.s1 - n.s0, nd = n.s0 - n.t0;
    if (ns <= 0) continue;
    if (nd == 0 && ns <= DB) jobs.push_back(make_int2(n.s0, ns));
    else if (ns > DB) ++nbig;
    if (nd > 0) xmax = std::max(xmax, (long long)ns * nd);
  }
  const int nslots = (int)jobs.size() + (int)tree.size() + 1;
  double* dpmin = nullptr;
  int2* djobs = nullptr;
  double *X = nullptr, *T = nullptr;
  cudaMallocAsync(&dpmin, (size_t)nslots * sizeof(double), s);
  cudaMemsetAsync(dpmin, 0x7f, (size_t)nslots * sizeof(double), s);  // large positive
  if (!jobs.empty()) {
    cudaMallocAsync(&djobs, jobs.size() * sizeof(int2), s);
    cudaMemcpyAsync(djobs, jobs.data(), jobs.size() * sizeof(int2), cudaMemcpyHostToDevice, s);
    k_chol_diag<<<(unsigned)jobs.size(), 32 * DNW, kDiagSmem, s>>>(E, ld, 0, 0, W, dpmin, 0,
                                                                     djobs);
  }
  if (xmax > 0) {
    cudaMallocAsync(&X, (size_t)xmax * sizeof(double), s);
    cudaMallocAsync(&T, (size_t)xmax * sizeof(double), s);
  }
  // separator-to-descendant couplings of every node (permuted columns, ascending), from E's
  // pattern: L_SD by the sparse product instead of a dense GEMM (DK_DENSE_LSD: the GEMM)
  std::vector<int> node_rp_off(tree.size(), -1), all_rp, all_ck;
  if (gptr && gcol && iperm && !getenv("DK_DENSE_LSD")) {
    std::vector<int> inv_perm(d);  // position -> label
    for (int L = 0; L < d; ++L) inv_perm[(*iperm)[L]] = L;
    for (size_t t = 0; t < tree.size(); ++t) {
      const auto& n = tree[t];
      const int ns = n.s1 - n.s0, nd = n.s0 - n.t0;
      if (ns <= 0 || nd <= 0) continue;
      node_rp_off[t] = (int)all_rp.size();
      const int base = (int)all_ck.size();
      std::vector<int> row;
      for (int r = 0; r < ns; ++r) {
        all_rp.push_back((int)all_ck.size() - base);
        const int L = inv_perm[n.s0 + r];
        row.clear();
        for (int e = (*gptr)[L]; e < (*gptr)[L + 1]; ++e) {
          const int p = (*iperm)[(*gcol)[e]];
          if (p >= n.t0 && p < n.s0) row.push_back(p);
        }
        std::sort(row.begin(), row.end());
        all_ck.insert(all_ck.end(), row.begin(), row.end());
      }
      all_rp.push_back((int)all_ck.size() - base);
    }
  }
  // rp entries are relative to each node's first column index: keep per node (rp offset,
  // ck offset) pairs
  std::vector<int2> node_off(tree.size(), make_int2(-1, -1));
  {
    size_t rpo = 0, cko = 0;
    for (size_t t = 0; t < tree.size(); ++t) {
      if (node_rp_off[t] < 0) continue;
      const auto& n = tree[t];
      const int ns = n.s1 - n.s0;
      node_off[t] = make_int2((int)rpo, (int)cko);
      cko += (size_t)all_rp[rpo + ns];
      rpo += (size_t)ns + 1;
    }
  }
  int *d_rp = nullptr, *d_ck = nullptr;
  if (!all_rp.empty()) {
    cudaMallocAsync(&d_rp, all_rp.size() * sizeof(int), s);
    cudaMemcpyAsync(d_rp, all_rp.data(), all_rp.size() * sizeof(int), cudaMemcpyHostToDevice, s);
    cudaMallocAsync(&d_ck, std::max<size_t>(all_ck.size(), 1) * sizeof(int), s);
    if (!all_ck.empty())
      cudaMemcpyAsync(d_ck, all_ck.data(), all_ck.size() * sizeof(int), cudaMemcpyHostToDevice,
                      s);
  }
  double host_min = INFINITY;
  int slot = (int)jobs.size();
  const bool trace = getenv("DK_TRACE_TREE") != nullptr;
  cudaEvent_t tev[3];
  if (trace) {
    for (auto& e : tev) cudaEventCreate(&e);
    cudaEventRecord(tev[0], s);
    cudaEventSynchronize(tev[0]);
  }
  auto t_start = std::chrono::steady_clock::now();
  for (size_t t = 0; t < tree.size(); ++t) {
    const auto& n = tree[t];
    const int ns = n.s1 - n.s0, nd = n.s0 - n.t0;
    if (ns <= 0 || (nd == 0 && ns <= DB)) continue;
    if (trace) cudaEventRecord(tev[1], s);
    if (nd > 0) {
      const int ldx = nd;
      if (node_off[t].x >= 0) {
        // L_SD = E_SD W_D^T, E_SD sparse
        k_lsd_sparse<<<(unsigned)std::min(nd, 16 * num_sms()), 128, 0, s>>>(
            E, W, ld, n.s0, ns, n.t0, nd, d_rp + node_off[t].x, d_ck + node_off[t].y, X, ldx);
      } else {
        // L_SD = E_SD W_D^T, child by child (W_C lower: op(B)[k][j] = 0 for k > j)
        for (int k : n.kids) {
          const int a = tree[k].t0, nc = tree[k].s1 - tree[k].t0;
          gemm_mma(false, true, at(E, n.s0, a), ld, at(W, a, a), ld, X + (a - n.t0), ldx, ns,
                   nc, nc, 1.0, 0.0, 0, INT_MIN, s, 0);
        }
      }
      // S = E_S - L_SD L_SD^T (lower tiles)
      gemm_mma(false, true, X, ldx, X, ldx, at(E, n.s0, n.s0), ld, ns, ns, nd, -1.0, 1.0, 1,
               INT_MIN, s);
      // T = L_SD W_D, child by child (W_C lower: B[k][j] = 0 for k < j)
      for (int k : n.kids) {
        const int a = tree[k].t0, nc = tree[k].s1 - tree[k].t0;
        gemm_mma(false, false, X + (a - n.t0), ldx, at(W, a, a), ld, T + (a - n.t0), ldx, ns,
                 nc, nc, 1.0, 0.0, 0, 0, s);
      }
    }
    // W_S = chol(S)^-1
    if (ns <= DB) {
      k_chol_diag<<<1, 32 * DNW, kDiagSmem, s>>>(E, ld, n.s0, ns, W, dpmin, slot++, nullptr);
    } else {
      double mn = 0.0;
      float f0 = 0.f, f1 = 0.f;
      const int err = spd_inverse(at(E, n.s0, n.s0), ns, ld, at(W, n.s0, n.s0), &mn, &f0, &f1,
                                  s, false, false);
      if (err) return err;
      host_min = (mn != mn || host_min != host_min) ? NAN : fmin(host_min, mn);
      if (!(mn >= 1e-280)) break;  // not SPD: the caller falls back
    }
    // W_SD = -W_S T
    if (nd > 0)
      gemm_mma(false, false, at(W, n.s0, n.s0), ld, T, nd, at(W, n.s0, n.t0), ld, ns, nd, ns,
               -1.0, 0.0, 0, INT_MIN, s);
    if (trace) {
      cudaEventRecord(tev[2], s);
      cudaEventSynchronize(tev[2]);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, tev[1], tev[2]);
      fprintf(stderr, "[tree] node sep %d desc %d kids %zu: %.3f ms\n", ns, nd, n.kids.size(),
              ms);
    }
  }
  if (trace) {
    cudaEventRecord(tev[2], s);
    cudaEventSynchronize(tev[2]);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, tev[0], tev[2]);
    fprintf(stderr, "[tree] leaves %zu; nodes total %.3f ms device, %.3f ms host\n", jobs.size(),
            ms, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() -
                                                          t_start).count());
  }
  std::vector<double> pm(slot > 0 ? slot : 1, INFINITY);
  if (slot > 0)
    cudaMemcpyAsync(pm.data(), dpmin, (size_t)slot * sizeof(double), cudaMemcpyDeviceToHost, s);
  const cudaError_t e = cudaStreamSynchronize(s);
  cudaFreeAsync(dpmin, s);
  if (djobs) cudaFreeAsync(djobs, s);
  if (d_rp) cudaFreeAsync(d_rp, s);
  if (d_ck) cudaFreeAsync(d_ck, s);
  if (X) cudaFreeAsync(X, s);
  if (T) cudaFreeAsync(T, s);
  double mn = host_min;
  for (int i = 0; i < slot; ++i) mn = (pm[i] != pm[i] || mn != mn) ? NAN : fmin(mn, pm[i]);
  *min_diag_sq = mn;
  return e != cudaSuccess ? (int)e : (int)cudaGetLastError();
}

}  // namespace dk
