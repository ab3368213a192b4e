// dk_coarse.cu — the coarse operator E = Z^T A_p Z on the device: deterministic assembly,
// dense fp64 LU with partial pivoting, explicit inverse, and the per-iteration GEMV
// y = E^-1 s.  Replaces build_context's AZ / E / dense_lu (deflation.py:84-88,
// sparse.py:121-137) and lu_solve (sparse.py:140-145).
//
// Why an explicit inverse: every GMRES iteration needs one coarse solve.  Forward and
// backward substitution with the LU factors is a d-long dependency chain; y = E^-1 s is a
// fully parallel GEMV that streams the same 8 d^2 bytes at HBM rate (and from L2 when
// 8 d^2 fits in the 126 MB L2).  The inverse is formed once from the LU factors.
#include <cuda_runtime.h>

#include <climits>

#include <cub/cub.cuh>
#include <vector>

#include "dk_launch.h"

namespace dk {

// ======================================================================================
// GEMV y = M x (one warp per row, x staged in shared memory, fixed summation order).
// ======================================================================================
// One CTA per contiguous block of rows (balanced over the 148 SMs); inside a CTA 4 rows are
// processed at a time, each by 8 warps that own contiguous eighths of the columns and keep
// 4 x 16 B loads in flight per lane.  The row sum is the fixed-order sum of the 8 warp
// partials (deterministic).
constexpr int kGemvThreads = 1024, kGemvRowsAtOnce = 4, kGemvSplit = 8;

template <bool SMEM_X>
__global__ void __launch_bounds__(kGemvThreads) k_gemv(const double* __restrict__ M, int d, int ld,
                                                       const double* __restrict__ x,
                                                       double* __restrict__ y, int rows_per_cta,
                                                       const int* __restrict__ gate) {
  pdl_wait();
  if (gate != nullptr && *gate == 0) return;
  extern __shared__ double sx[];
  __shared__ double red[kGemvRowsAtOnce][kGemvSplit];
  const double* xs = x;
  if (SMEM_X) {
    for (int i = threadIdx.x; i < ld; i += blockDim.x) sx[i] = i < d ? x[i] : 0.0;
    __syncthreads();
    xs = sx;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rsub = warp / kGemvSplit, part = warp % kGemvSplit;
  int seg = (ld + kGemvSplit - 1) / kGemvSplit;
  seg = (seg + 1) & ~1;
  const int c0 = part * seg;
  const int c1 = min(ld, c0 + seg);
  const int r0 = blockIdx.x * rows_per_cta;
  const int r1 = min(d, r0 + rows_per_cta);
  for (int rb = r0; rb < r1; rb += kGemvRowsAtOnce) {
    const int r = rb + rsub;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    if (r < r1) {
      const double* row = M + (long long)r * ld;
      int c = c0 + 2 * lane;
      for (; c + 192 < c1; c += 256) {
        const double2 p0 = ld2(row + c);
        const double2 p1 = ld2(row + c + 64);
        const double2 p2 = ld2(row + c + 128);
        const double2 p3 = ld2(row + c + 192);
        a0 = fma(p0.x, xs[c], a0);
        a1 = fma(p0.y, xs[c + 1], a1);
        a2 = fma(p1.x, xs[c + 64], a2);
        a3 = fma(p1.y, xs[c + 65], a3);
        a0 = fma(p2.x, xs[c + 128], a0);
        a1 = fma(p2.y, xs[c + 129], a1);
        a2 = fma(p3.x, xs[c + 192], a2);
        a3 = fma(p3.y, xs[c + 193], a3);
      }
      for (; c < c1; c += 64) {
        const double2 p0 = ld2(row + c);
        a0 = fma(p0.x, xs[c], a0);
        a1 = fma(p0.y, xs[c + 1], a1);
      }
    }
    const double s = warp_sum((a0 + a1) + (a2 + a3));
    if (lane == 0) red[rsub][part] = s;
    __syncthreads();
    if (threadIdx.x < kGemvRowsAtOnce && rb + threadIdx.x < r1) {
      double t = 0.0;
      for (int p = 0; p < kGemvSplit; ++p) t += red[threadIdx.x][p];
      y[rb + threadIdx.x] = t;
    }
    __syncthreads();
  }
}

void launch_gemv(const double* M, int d, int ld, const double* x, double* y, const int* gate,
                 cudaStream_t s) {
  const size_t smem = (size_t)ld * sizeof(double);
  const int ctas_max = num_sms();
  int rows_per_cta = (d + ctas_max - 1) / ctas_max;
  const unsigned grid = (unsigned)((d + rows_per_cta - 1) / rows_per_cta);
  if (smem <= 200 * 1024) {
    smem_optin((const void*)k_gemv<true>, 200 * 1024);
    launch_pdl(k_gemv<true>, dim3(grid), dim3(kGemvThreads), smem, s, M, d, ld, x, y,
               rows_per_cta, gate);
  } else {
    launch_pdl(k_gemv<false>, dim3(grid), dim3(kGemvThreads), 0, s, M, d, ld, x, y,
               rows_per_cta, gate);
  }
}

// ======================================================================================
// Symmetric coarse solve y = E^-1 s streaming only the upper tile triangle of E^-1.
//
// With A symmetric and A_p = A, E = Z^T A Z and E^-1 are symmetric: the tiles (I, J), I <= J,
// of 32 x 32 hold every entry once, halving the 8 d^2 bytes per iteration.  Tile (I, J)
// contributes y_I += T s_J (row part) and, off the diagonal, y_J += T^T s_I (column part).
// One warp streams a contiguous range of tiles (row-major over the triangle; balanced to
// +-1 tile): lane r owns tile row r, so the row part accumulates in a register across the
// warp's tiles of one tile row and the column part is a 32-way butterfly reduce-scatter
// (lane c ends with column c).  Partials go to fixed slots and k_symv_reduce sums them in
// a fixed order: deterministic.
// Tile storage: [16 column pairs][32 rows][2] (one coalesced 512 B double2 load per pair).
// ======================================================================================
constexpr int kST = 32;                 // tile edge

__host__ __device__ inline long long tri_start(long long I, long long nb) {
  return I * nb - I * (I - 1) / 2;      // index of tile (I, I)
}

__global__ void k_symv_pack(const double* __restrict__ Einv, int d, int ld, int nb,
                            double* __restrict__ P) {
  const long long ntiles = (long long)nb * (nb + 1) / 2;
  const long long tot = ntiles * kST * kST;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const long long t = e / (kST * kST);
    const int w = (int)(e % (kST * kST));
    const int pair = w / (2 * kST), r = (w / 2) % kST, c = 2 * pair + (w & 1);
    // tile row I: largest I with tri_start(I) <= t
    long long lo = 0, hi = nb - 1;
    while (lo < hi) {
      const long long mid = (lo + hi + 1) / 2;
      if (tri_start(mid, nb) <= t) lo = mid; else hi = mid - 1;
    }
    const long long I = lo, J = I + (t - tri_start(I, nb));
    const long long gr = I * kST + r, gc = J * kST + c;
    double v = 0.0;
    if (gr < d && gc < d) v = 0.5 * (Einv[gr * ld + gc] + Einv[gc * ld + gr]);
    P[e] = v;
  }
}

// Per-warp TMA pipeline: each warp owns kSymvStages shared-memory tile buffers filled by
// one-lane cp.async.bulk copies (8 KB each, completion on an mbarrier), so kSymvStages - 1
// tiles stream in while the warp reduces the current one.
constexpr int kSymvWarps = 16, kSymvStages = 1;
constexpr int kTileBytes = kST * kST * 8;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void tma_tile(void* dst, const void* src, unsigned long long* bar,
                                         unsigned long long pol) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"((unsigned)kTileBytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"((unsigned)kTileBytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, "
        "p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  }
}

__global__ void __launch_bounds__(kSymvWarps * 32) k_symv(const double* __restrict__ P, int d,
                                                          int nb, const double* __restrict__ x,
                                                          double* __restrict__ rowpart,
                                                          double* __restrict__ colpart,
                                                          const int* __restrict__ gate) {
  pdl_wait();
  if (gate != nullptr && *gate == 0) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long bars[kSymvWarps][kSymvStages];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  double* buf = reinterpret_cast<double*>(smem_raw) + (size_t)wl * kSymvStages * (kST * kST);
  double* sx = reinterpret_cast<double*>(smem_raw) + (size_t)kSymvWarps * kSymvStages * kST * kST;
  for (int i = threadIdx.x; i < nb * kST; i += blockDim.x) sx[i] = i < d ? x[i] : 0.0;
  __syncthreads();
  const long long W = (long long)gridDim.x * kSymvWarps;
  const long long w = (long long)blockIdx.x * kSymvWarps + wl;
  const long long ntiles = (long long)nb * (nb + 1) / 2;
  const long long t0 = w * ntiles / W, t1 = (w + 1) * ntiles / W;
  const unsigned long long pol = l2_evict_first();
  if (lane == 0)
    for (int s = 0; s < kSymvStages; ++s) mbar_init(&bars[wl][s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  if (t0 >= t1) return;
  if (lane == 0)
    for (int s = 0; s < kSymvStages && t0 + s < t1; ++s)
      tma_tile(buf + s * (kST * kST), P + (t0 + s) * (kST * kST), &bars[wl][s], pol);
  long long lo = 0, hi = nb - 1;
  while (lo < hi) {
    const long long mid = (lo + hi + 1) / 2;
    if (tri_start(mid, nb) <= t0) lo = mid; else hi = mid - 1;
  }
  long long I = lo, J = I + (t0 - tri_start(I, nb));
  long long seg = t0;  // slot of the current row-part segment
  double racc = 0.0;
  for (long long t = t0; t < t1; ++t) {
    const int s = (int)((t - t0) % kSymvStages);
    const unsigned parity = (unsigned)(((t - t0) / kSymvStages) & 1);
    mbar_wait(&bars[wl][s], parity);
    const double2* T = reinterpret_cast<const double2*>(buf + s * (kST * kST));
    double cacc[32];
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      const double2 v = T[p * kST + lane];
      cacc[2 * p] = v.x;
      cacc[2 * p + 1] = v.y;
    }
    __syncwarp();
    if (lane == 0 && t + kSymvStages < t1)  // refill this stage
      tma_tile(buf + s * (kST * kST), P + (t + kSymvStages) * (kST * kST), &bars[wl][s], pol);
    const double* xJ = sx + J * kST;
    const double xr = sx[I * kST + lane];
#pragma unroll
    for (int c = 0; c < 32; ++c) racc = fma(cacc[c], xJ[c], racc);
#pragma unroll
    for (int c = 0; c < 32; ++c) cacc[c] *= xr;
    if (J != I) {
      // butterfly reduce-scatter: lane c ends with sum over lanes of cacc[c]
#pragma unroll
      for (int k = 16; k >= 1; k >>= 1) {
        const bool up = (lane & k) != 0;
#pragma unroll
        for (int i = 0; i < k; ++i) {
          const double send = up ? cacc[i] : cacc[i + k];
          const double keep = up ? cacc[i + k] : cacc[i];
          cacc[i] = keep + __shfl_xor_sync(0xffffffffu, send, k);
        }
      }
      colpart[t * kST + lane] = cacc[0];
    }
    // advance (I, J); flush the row part when the tile row changes or the range ends
    ++J;
    if (J == nb || t + 1 == t1) {
      rowpart[seg * kST + lane] = racc;
      racc = 0.0;
      seg = t + 1;
      if (J == nb) {
        ++I;
        J = I;
      }
    }
  }
}

// y_J = sum of row-part segments of tile row J (warps in order) + sum_{I<J} column parts
// of tiles (I, J) (I in order); 32 warps split the I range, combined in a fixed order.
constexpr int kRedWarps = 16;
__global__ void __launch_bounds__(kRedWarps * 32) k_symv_reduce(const double* __restrict__ rowpart,
                                                     const double* __restrict__ colpart, int d,
                                                     int nb, const int* __restrict__ seg_ptr,
                                                     const int* __restrict__ seg_slot,
                                                     double* __restrict__ y,
                                                     const int* __restrict__ gate) {
  pdl_wait();
  if (gate != nullptr && *gate == 0) return;
  __shared__ double red[kRedWarps][kST];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int Jt = blockIdx.x;
  double acc = 0.0;
#pragma unroll 8
  for (int I = warp; I < Jt; I += kRedWarps) {
    const int t = (int)tri_start(I, nb) + (Jt - I);
    acc += colpart[(size_t)t * kST + lane];
  }
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0) {
    double s = 0.0;
    // row-part segments of tile row Jt (host-precomputed slots, in warp order)
    for (int k = seg_ptr[Jt]; k < seg_ptr[Jt + 1]; ++k)
      s += rowpart[(size_t)seg_slot[k] * kST + lane];
    for (int w2 = 0; w2 < kRedWarps; ++w2) s += red[w2][lane];
    const int row = Jt * kST + lane;
    if (row < d) y[row] = s;
  }
}

// Row-part segment slots per tile row for the static warp partition of k_symv: the row's
// first tile plus every warp range start strictly inside the row.
void symv_segments(int d, std::vector<int>& ptr, std::vector<int>& slots) {
  const long long nb = (d + kST - 1) / kST;
  const long long ntiles = nb * (nb + 1) / 2;
  const long long W = (long long)num_sms() * kSymvWarps;
  std::vector<long long> starts;
  for (long long ww = 0; ww < W; ++ww) {
    const long long r0 = ww * ntiles / W, r1 = (ww + 1) * ntiles / W;
    if (r0 < r1) starts.push_back(r0);
  }
  ptr.assign(nb + 1, 0);
  slots.clear();
  size_t k = 0;
  for (long long J = 0; J < nb; ++J) {
    const long long a = tri_start(J, nb), b = a + (nb - J);
    ptr[J] = (int)slots.size();
    slots.push_back((int)a);
    while (k < starts.size() && starts[k] <= a) ++k;
    for (size_t q = k; q < starts.size() && starts[q] < b; ++q) slots.push_back((int)starts[q]);
  }
  ptr[nb] = (int)slots.size();
}

// flag <- 0 unless |E_ij - E_ji| <= 1e-12 (|E_ij| + |E_ji|) for all i, j (assembly rounding)
__global__ void k_check_sym(const double* __restrict__ E, int d, int ld, int* flag) {
  const long long tot = (long long)d * d;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / d, j = e % d;
    if (j <= i) continue;
    const double a = E[i * ld + j], b = E[j * ld + i];
    if (!(fabs(a - b) <= 1e-12 * (fabs(a) + fabs(b)))) atomicExch(flag, 0);
  }
}

int coarse_is_symmetric(const double* E, int d, int ld, cudaStream_t s) {
  int h = 1;
  int* f = nullptr;
  cudaMallocAsync(&f, sizeof(int), s);
  cudaMemcpyAsync(f, &h, sizeof(int), cudaMemcpyHostToDevice, s);
  k_check_sym<<<num_sms() * 8, 256, 0, s>>>(E, d, ld, f);
  cudaMemcpyAsync(&h, f, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  cudaFreeAsync(f, s);
  return h;
}

long long symv_tiles(int d) {
  const long long nb = (d + kST - 1) / kST;
  return nb * (nb + 1) / 2;
}

void launch_symv_pack(const double* Einv, int d, int ld, double* P, cudaStream_t s) {
  const int nb = (d + kST - 1) / kST;
  k_symv_pack<<<num_sms() * 8, 256, 0, s>>>(Einv, d, ld, nb, P);
}

void launch_symv(const double* P, int d, const double* x, double* rowpart, double* colpart,
                 double* y, const int* gate, cudaStream_t s) {
  const int nb = (d + kST - 1) / kST;
  const size_t smem =
      (size_t)kSymvWarps * kSymvStages * kTileBytes + (size_t)nb * kST * sizeof(double);
  smem_optin((const void*)k_symv, smem);
  const unsigned grid = (unsigned)num_sms();
  launch_pdl(k_symv, dim3(grid), dim3(kSymvWarps * 32), smem, s, P, d, nb, x, rowpart, colpart,
             gate);
}

void launch_symv_reduce(int d, const double* rowpart, const double* colpart,
                        const int* seg_ptr, const int* seg_slot, double* y, const int* gate,
                        cudaStream_t s) {
  const int nb = (d + kST - 1) / kST;
  launch_pdl(k_symv_reduce, dim3(nb), dim3(kRedWarps * 32), 0, s, rowpart, colpart, d, nb,
             seg_ptr, seg_slot, y, gate);
}

// ======================================================================================
// Assembly of E = Z^T A_p Z for an indicator Z given by labels.
//   E[L][L]  = sum over cells i of L (ascending) of q_i, q_i = sum of the row's coefficients
//              whose column is in L (ascending column) — sequential, deterministic;
//   E[L][L2] = sum over (i in L, k in L2, k = i + off) of a_ik — the boundary-face list is
//              sorted by key (L, L2) with a stable radix sort and summed per key in cell
//              order (deterministic).
// With A_p = A M^-1 the coefficient a_ik is scaled by inv_diag_k (deflation.py:84).
// ======================================================================================
template <bool AM>
__device__ __forceinline__ double coarse_coef(const Dia& A, int q, long long i) {
  double a = dia_coef(A, q, i);
  if (AM) a = __dmul_rn(a, A.inv[i + A.off[q]]);
  return a;
}

template <bool AM>
__global__ void k_coarse_scan(Dia A, const int* __restrict__ lab, long long n_pad,
                              double* __restrict__ qv, int* __restrict__ cnt) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_pad;
       i += (long long)gridDim.x * blockDim.x) {
    const int L = lab[i];
    double q = 0.0;
    int c = 0;
    if (L >= 0) {
      for (int k = 0; k < A.ndiag; ++k) {
        const int L2 = lab[i + A.off[k]];
        if (L2 == L) q = __dadd_rn(q, coarse_coef<AM>(A, k, i));
        else if (L2 >= 0) ++c;
      }
    }
    qv[i] = q;
    cnt[i] = c;
  }
}

template <bool AM>
__global__ void k_coarse_emit(Dia A, const int* __restrict__ lab, long long n_pad, int d,
                              const int* __restrict__ off, unsigned long long* __restrict__ keys,
                              double* __restrict__ vals) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_pad;
       i += (long long)gridDim.x * blockDim.x) {
    const int L = lab[i];
    if (L < 0) continue;
    int p = off[i];
    for (int k = 0; k < A.ndiag; ++k) {
      const int L2 = lab[i + A.off[k]];
      if (L2 >= 0 && L2 != L) {
        keys[p] = (unsigned long long)L * (unsigned long long)d + (unsigned long long)L2;
        vals[p] = coarse_coef<AM>(A, k, i);
        ++p;
      }
    }
  }
}

__global__ void k_coarse_reduce(const unsigned long long* __restrict__ keys,
                                const double* __restrict__ vals, long long nk, int d,
                                double* __restrict__ E, int ld) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < nk;
       k += (long long)gridDim.x * blockDim.x) {
    const unsigned long long key = keys[k];
    if (k > 0 && keys[k - 1] == key) continue;
    double s = 0.0;
    for (long long t = k; t < nk && keys[t] == key; ++t) s = __dadd_rn(s, vals[t]);
    const long long L = (long long)(key / (unsigned long long)d);
    const long long L2 = (long long)(key % (unsigned long long)d);
    E[L * ld + L2] = s;
  }
}

// Diagonal E[L][L] = sum over the cells of L in ascending order of q_i — a plain sequential
// sum per label (the oracle's np.bincount order; the in-label couplings nearly cancel, so
// the order is what fixes the last bits at a high coefficient contrast).  Cells are grouped
// by a stable sort of their labels (unlabelled cells sort last, as label d).
__global__ void k_label_keys(const int* __restrict__ lab, long long n_pad, int d,
                             int* __restrict__ key, int* __restrict__ cell) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_pad;
       i += (long long)gridDim.x * blockDim.x) {
    const int L = lab[i];
    key[i] = L >= 0 ? L : d;
    cell[i] = (int)i;
  }
}

// start[L] = first sorted position of label L (start[d] = end of the labelled cells)
__global__ void k_label_start(const int* __restrict__ skey, long long n, int d,
                              int* __restrict__ start) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int k = skey[i];
    const int prev = i > 0 ? skey[i - 1] : -1;
    for (int L = prev + 1; L <= k && L <= d; ++L) start[L] = (int)i;
    if (i == n - 1)
      for (int L = k + 1; L <= d; ++L) start[L] = (int)n;
  }
}

__global__ void k_diag_seq(const double* __restrict__ q, const int* __restrict__ cells,
                           const int* __restrict__ start, int d, double* __restrict__ E, int ld) {
  for (int L = blockIdx.x * blockDim.x + threadIdx.x; L < d; L += gridDim.x * blockDim.x) {
    const int p0 = start[L], p1 = start[L + 1];
    double s = 0.0;
    int p = p0;
    for (; p + 8 <= p1; p += 8) {  // eight loads in flight, then the in-order sum
      double v[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) v[k] = q[cells[p + k]];
#pragma unroll
      for (int k = 0; k < 8; ++k) s = __dadd_rn(s, v[k]);
    }
    for (; p < p1; ++p) s = __dadd_rn(s, q[cells[p]]);
    E[(long long)L * ld + L] = s;
  }
}

static int bits_for(unsigned long long v) {
  int b = 1;
  while (b < 64 && (1ull << b) <= v) ++b;
  return b;
}

int build_coarse(const Dia& A, bool am, const int* lab, long long n_pad, const RunMap& rm,
                 double* E, int ld, double* qv, cudaStream_t s) {
  const int d = rm.d;
  cudaError_t err;
  int* cnt = nullptr;
  int* off = nullptr;
  void* tmp = nullptr;
  unsigned long long *k_in = nullptr, *k_out = nullptr;
  double *v_in = nullptr, *v_out = nullptr, *sdiag = nullptr;
  int total = 0, last_cnt = 0;
  size_t tmp_bytes = 0, need = 0;
  const unsigned grid = (unsigned)num_sms() * 8;
  long long nk = 0;
#define DKC(x)                       \
  do {                               \
    err = (x);                       \
    if (err != cudaSuccess) goto fail; \
  } while (0)
  DKC(cudaMemsetAsync(E, 0, (size_t)d * ld * sizeof(double), s));
  DKC(cudaMallocAsync(&cnt, (size_t)n_pad * sizeof(int), s));
  DKC(cudaMallocAsync(&off, (size_t)n_pad * sizeof(int), s));
  DKC(cudaMallocAsync(&sdiag, (size_t)(d > 0 ? d : 1) * sizeof(double), s));
  if (am) k_coarse_scan<true><<<grid, kThreads, 0, s>>>(A, lab, n_pad, qv, cnt);
  else k_coarse_scan<false><<<grid, kThreads, 0, s>>>(A, lab, n_pad, qv, cnt);
  DKC(cudaGetLastError());
  // diagonal: per label, the sequential sum of q over its cells in ascending order
  (void)rm;
  {
    int *key_in = nullptr, *key_out = nullptr, *cell_in = nullptr, *cell_out = nullptr,
        *start = nullptr;
    void* stmp = nullptr;
    size_t sbytes = 0;
    const int kbits = bits_for((unsigned long long)d + 1);
    DKC(cudaMallocAsync(&key_in, (size_t)n_pad * sizeof(int), s));
    DKC(cudaMallocAsync(&key_out, (size_t)n_pad * sizeof(int), s));
    DKC(cudaMallocAsync(&cell_in, (size_t)n_pad * sizeof(int), s));
    DKC(cudaMallocAsync(&cell_out, (size_t)n_pad * sizeof(int), s));
    DKC(cudaMallocAsync(&start, (size_t)(d + 1) * sizeof(int), s));
    k_label_keys<<<grid, kThreads, 0, s>>>(lab, n_pad, d, key_in, cell_in);
    DKC(cub::DeviceRadixSort::SortPairs(nullptr, sbytes, key_in, key_out, cell_in, cell_out,
                                        (int)n_pad, 0, kbits, s));
    DKC(cudaMallocAsync(&stmp, sbytes, s));
    DKC(cub::DeviceRadixSort::SortPairs(stmp, sbytes, key_in, key_out, cell_in, cell_out,
                                        (int)n_pad, 0, kbits, s));
    k_label_start<<<grid, kThreads, 0, s>>>(key_out, n_pad, d, start);
    k_diag_seq<<<(d + 127) / 128, 128, 0, s>>>(qv, cell_out, start, d, E, ld);
    DKC(cudaGetLastError());
    cudaFreeAsync(key_in, s);
    cudaFreeAsync(key_out, s);
    cudaFreeAsync(cell_in, s);
    cudaFreeAsync(cell_out, s);
    cudaFreeAsync(start, s);
    cudaFreeAsync(stmp, s);
  }
  // off-diagonal: boundary faces
  DKC(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, off, (int)n_pad, s));
  DKC(cudaMallocAsync(&tmp, tmp_bytes, s));
  DKC(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, off, (int)n_pad, s));
  DKC(cudaMemcpyAsync(&total, off + n_pad - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  DKC(cudaMemcpyAsync(&last_cnt, cnt + n_pad - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  DKC(cudaStreamSynchronize(s));
  nk = (long long)total + last_cnt;
  if (nk > 0) {
    DKC(cudaMallocAsync(&k_in, nk * sizeof(unsigned long long), s));
    DKC(cudaMallocAsync(&k_out, nk * sizeof(unsigned long long), s));
    DKC(cudaMallocAsync(&v_in, nk * sizeof(double), s));
    DKC(cudaMallocAsync(&v_out, nk * sizeof(double), s));
    if (am) k_coarse_emit<true><<<grid, kThreads, 0, s>>>(A, lab, n_pad, d, off, k_in, v_in);
    else k_coarse_emit<false><<<grid, kThreads, 0, s>>>(A, lab, n_pad, d, off, k_in, v_in);
    DKC(cudaGetLastError());
    const int nbits = bits_for((unsigned long long)d * (unsigned long long)d);
    DKC(cub::DeviceRadixSort::SortPairs(nullptr, need, k_in, k_out, v_in, v_out, (int)nk, 0, nbits,
                                        s));
    if (need > tmp_bytes) {
      DKC(cudaFreeAsync(tmp, s));
      DKC(cudaMallocAsync(&tmp, need, s));
      tmp_bytes = need;
    }
    DKC(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, k_in, k_out, v_in, v_out, (int)nk, 0, nbits,
                                        s));
    k_coarse_reduce<<<grid, kThreads, 0, s>>>(k_out, v_out, nk, d, E, ld);
    DKC(cudaGetLastError());
  }
  DKC(cudaStreamSynchronize(s));
fail:
  cudaFreeAsync(cnt, s);
  cudaFreeAsync(off, s);
  cudaFreeAsync(sdiag, s);
  if (tmp) cudaFreeAsync(tmp, s);
  if (k_in) cudaFreeAsync(k_in, s);
  if (k_out) cudaFreeAsync(k_out, s);
  if (v_in) cudaFreeAsync(v_in, s);
  if (v_out) cudaFreeAsync(v_out, s);
  cudaStreamSynchronize(s);
  return (int)err;
#undef DKC
}

// ======================================================================================
// Dense LU with partial pivoting (right-looking, panel width kNB), row-major, then the
// explicit inverse Einv = U^-1 L^-1 P by two blocked triangular solves on P.
// ======================================================================================
constexpr int kNB = 32;

// Unblocked panel factorisation of columns [k, k+nb) over rows [k, d) by one block.
// Pivot = first row of maximal |a| (LAPACK idamax); zero pivot columns are left unscaled
// (LAPACK dgetf2 semantics; singularity is reported from min |U_kk| afterwards).
__global__ void __launch_bounds__(1024) k_panel(double* __restrict__ E, int d, int ld, int k,
                                                int nb, int* __restrict__ piv) {
  __shared__ double sv[32];
  __shared__ int si[32];
  __shared__ double prow[kNB];
  __shared__ int s_p;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  for (int c = k; c < k + nb; ++c) {
    double best = -1.0;
    int bi = d;
    for (int r = c + t; r < d; r += blockDim.x) {
      const double a = fabs(E[(long long)r * ld + c]);
      if (a > best) {
        best = a;
        bi = r;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if (lane == 0) {
      sv[warp] = best;
      si[warp] = bi;
    }
    __syncthreads();
    if (t == 0) {
      double b = -1.0;
      int i = d;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w)
        if (sv[w] > b || (sv[w] == b && si[w] < i)) {
          b = sv[w];
          i = si[w];
        }
      if (i >= d) i = c;
      piv[c] = i;
      s_p = i;
    }
    __syncthreads();
    const int p = s_p;
    if (p != c) {  // swap rows c and p inside the panel
      for (int cc = k + t; cc < k + nb; cc += blockDim.x) {
        const double a = E[(long long)c * ld + cc];
        E[(long long)c * ld + cc] = E[(long long)p * ld + cc];
        E[(long long)p * ld + cc] = a;
      }
    }
    __syncthreads();
    if (t < nb) prow[t] = E[(long long)c * ld + k + t];
    __syncthreads();
    const double pv = prow[c - k];
    if (pv != 0.0) {
      for (int r = c + 1 + t; r < d; r += blockDim.x) {
        double* row = E + (long long)r * ld;
        const double l = row[c] / pv;
        row[c] = l;
        for (int cc = c + 1; cc < k + nb; ++cc) row[cc] = fma(-l, prow[cc - k], row[cc]);
      }
    }
    __syncthreads();
  }
}

// Apply the row interchanges piv[k0 .. k1) in order to columns outside [skip0, skip1).
__global__ void k_laswp(double* __restrict__ E, int ncols, int ld, const int* __restrict__ piv,
                        int k0, int k1, int skip0, int skip1) {
  for (int col = blockIdx.x * blockDim.x + threadIdx.x; col < ncols;
       col += gridDim.x * blockDim.x) {
    if (col >= skip0 && col < skip1) continue;
    for (int c = k0; c < k1; ++c) {
      const int p = piv[c];
      if (p != c) {
        const double a = E[(long long)c * ld + col];
        E[(long long)c * ld + col] = E[(long long)p * ld + col];
        E[(long long)p * ld + col] = a;
      }
    }
  }
}

// X[k..k+nb, col] <- T^-1 X[k..k+nb, col] for columns [c0, c1), T = E[k..k+nb, k..k+nb]
// (UNIT lower, or upper with its diagonal).  One thread per column.
template <bool UPPER>
__global__ void __launch_bounds__(256) k_trsm_block(const double* __restrict__ T, int ldt, int k,
                                                    int nb, double* __restrict__ X, int ldx,
                                                    int c0, int c1) {
  __shared__ double sT[kNB * kNB];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x)
    sT[e] = T[(long long)(k + e / nb) * ldt + k + e % nb];
  __syncthreads();
  for (int col = c0 + blockIdx.x * blockDim.x + threadIdx.x; col < c1;
       col += gridDim.x * blockDim.x) {
    double x[kNB];
#pragma unroll
    for (int i = 0; i < kNB; ++i)
      if (i < nb) x[i] = X[(long long)(k + i) * ldx + col];
    if (!UPPER) {
#pragma unroll
      for (int i = 0; i < kNB; ++i) {
        if (i < nb) {
#pragma unroll
          for (int l = 0; l < i; ++l) x[i] = fma(-sT[i * nb + l], x[l], x[i]);
        }
      }
    } else {
#pragma unroll
      for (int i = kNB - 1; i >= 0; --i) {
        if (i < nb) {
#pragma unroll
          for (int l = i + 1; l < kNB; ++l)
            if (l < nb) x[i] = fma(-sT[i * nb + l], x[l], x[i]);
          x[i] = x[i] / sT[i * nb + i];
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kNB; ++i)
      if (i < nb) X[(long long)(k + i) * ldx + col] = x[i];
  }
}

// C[M x N] -= A[M x K] * B[K x N] (row-major, fp64 DFMA), 64x64 tiles, 4x4 per thread.
constexpr int kGT = 64, kGK = 16;
__global__ void __launch_bounds__(256) k_dgemm_sub(const double* __restrict__ Am, int lda,
                                                   const double* __restrict__ Bm, int ldb,
                                                   double* __restrict__ C, int ldc, int M, int N,
                                                   int K) {
  __shared__ double sA[kGK][kGT + 1];
  __shared__ double sB[kGK][kGT];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int r0 = blockIdx.y * kGT, c0 = blockIdx.x * kGT;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int kk = 0; kk < K; kk += kGK) {
    for (int e = threadIdx.x; e < kGK * kGT; e += 256) {
      const int r = e / kGK, c = e % kGK;  // A tile: 64 rows x 16 k
      const int gr = r0 + r, gk = kk + c;
      sA[c][r] = (gr < M && gk < K) ? Am[(long long)gr * lda + gk] : 0.0;
      const int br = e / kGT, bc = e % kGT;  // B tile: 16 k x 64 cols
      const int gbk = kk + br, gc = c0 + bc;
      sB[br][bc] = (gbk < K && gc < N) ? Bm[(long long)gbk * ldb + gc] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kGK; ++q) {
      double av[4], bv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = sA[q][ty * 4 + a];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = sB[q][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b] = fma(av[a], bv[b], acc[a][b]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int gr = r0 + ty * 4 + a;
    if (gr >= M) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int gc = c0 + tx + 16 * b;
      if (gc < N) C[(long long)gr * ldc + gc] -= acc[a][b];
    }
  }
}

constexpr int kNB2 = 256;  // outer panel width of the two-level LU / triangular solves

static void dgemm_sub(const double* A, int lda, const double* B, int ldb, double* C, int ldc,
                      int M, int N, int K, cudaStream_t s) {
  if (M <= 0 || N <= 0 || K <= 0) return;
  if (K >= 32 && (long long)M * N >= 256LL * 256) {  // fp64 tensor cores (dk_dense.cu)
    gemm_mma(false, false, A, lda, B, ldb, C, ldc, M, N, K, -1.0, 1.0, 0, INT_MIN, s);
    return;
  }
  dim3 grid((N + kGT - 1) / kGT, (M + kGT - 1) / kGT);
  k_dgemm_sub<<<grid, 256, 0, s>>>(A, lda, B, ldb, C, ldc, M, N, K);
}

__global__ void k_min_pivot(const double* __restrict__ E, int d, int ld, double* out) {
  __shared__ double red[32];
  double m = INFINITY;
  for (int i = threadIdx.x; i < d; i += blockDim.x) m = fmin(m, fabs(E[(long long)i * ld + i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmin(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = INFINITY;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmin(r, red[w]);
    *out = r;
  }
}

__global__ void k_identity(double* __restrict__ X, int d, int ld) {
  const long long tot = (long long)d * ld;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / ld, c = e % ld;
    X[e] = (r == c && c < d) ? 1.0 : 0.0;
  }
}

// Column diagonal dominance |E_cc| >= sum_{r != c} |E_rc| for every column: partial pivoting
// then never interchanges rows (the property survives elimination, Golub & Van Loan 3.4.3),
// so the pivot-free blocked LU below is exactly the partially pivoted factorisation.
// E = Z^T A Z of a TPFA operator is symmetric and diagonally dominant.
__global__ void __launch_bounds__(256) k_col_dominance(const double* __restrict__ E, int d, int ld,
                                                       int* flag) {
  __shared__ double part[8][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  double off = 0.0;
  if (c < d) {
    for (int r = warp; r < d; r += 8)
      if (r != c) off += fabs(E[(long long)r * ld + c]);
  }
  part[warp][lane] = off;
  __syncthreads();
  if (warp == 0 && c < d) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += part[w][lane];
    // E = Z^T A Z of a TPFA operator is only weakly dominant (equality for regions without a
    // Dirichlet face), so rounding in the assembled sums is tolerated
    if (!(fabs(E[(long long)c * ld + c]) >= t * (1.0 - 1e-10))) atomicExch(flag, 0);
  }
}

// Unpivoted LU of the nb x nb diagonal block at (k, k), in shared memory, one block.
__global__ void __launch_bounds__(256) k_diag_lu(double* __restrict__ E, int ld, int k, int nb,
                                                 int* __restrict__ piv) {
  __shared__ double a[kNB][kNB + 1];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x)
    a[e / nb][e % nb] = E[(long long)(k + e / nb) * ld + k + e % nb];
  __syncthreads();
  for (int c = 0; c < nb; ++c) {
    const double p = a[c][c];
    for (int e = threadIdx.x; e < (nb - c - 1) * (nb - c); e += blockDim.x) {
      const int r = c + 1 + e / (nb - c);
      const int cc = c + e % (nb - c);
      if (cc == c) continue;
      const double l = (p != 0.0) ? a[r][c] / p : a[r][c];
      a[r][cc] = fma(-l, a[c][cc], a[r][cc]);
    }
    __syncthreads();
    if (p != 0.0)
      for (int r = c + 1 + threadIdx.x; r < nb; r += blockDim.x) a[r][c] = a[r][c] / p;
    __syncthreads();
  }
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x)
    E[(long long)(k + e / nb) * ld + k + e % nb] = a[e / nb][e % nb];
  for (int c = threadIdx.x; c < nb; c += blockDim.x) piv[k + c] = k + c;
}

// L21 = A21 U11^-1 (rows [k+nb, d)), one thread per row.
__global__ void __launch_bounds__(256) k_trsm_rows(double* __restrict__ E, int d, int ld, int k,
                                                   int nb) {
  __shared__ double sU[kNB * kNB];
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x)
    sU[e] = E[(long long)(k + e / nb) * ld + k + e % nb];
  __syncthreads();
  for (int r = k + nb + blockIdx.x * blockDim.x + threadIdx.x; r < d;
       r += gridDim.x * blockDim.x) {
    double* row = E + (long long)r * ld + k;
    double x[kNB];
#pragma unroll
    for (int j = 0; j < kNB; ++j)
      if (j < nb) x[j] = row[j];
#pragma unroll
    for (int j = 0; j < kNB; ++j) {
      if (j < nb) {
#pragma unroll
        for (int l = 0; l < j; ++l) x[j] = fma(-x[l], sU[l * nb + j], x[j]);
        const double u = sU[j * nb + j];
        if (u != 0.0) x[j] = x[j] / u;
      }
    }
#pragma unroll
    for (int j = 0; j < kNB; ++j)
      if (j < nb) row[j] = x[j];
  }
}

// Column test for the pivot-free path (see k_col_dominance); `strict` drops the rounding
// allowance, so the pivots equal partial pivoting's exactly (the public dense_lu).
static int column_dominant(const double* E, int d, int ld, cudaStream_t s) {
  int* dflag = nullptr;
  int dominant = 1;
  cudaMallocAsync(&dflag, sizeof(int), s);
  cudaMemcpyAsync(dflag, &dominant, sizeof(int), cudaMemcpyHostToDevice, s);
  k_col_dominance<<<(d + 31) / 32, 256, 0, s>>>(E, d, ld, dflag);
  cudaMemcpyAsync(&dominant, dflag, sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  cudaFreeAsync(dflag, s);
  return dominant;
}

// P E = L U in place (row-major; unit L below the diagonal, U on and above it; piv[k] = the
// row interchanged with row k, 0-based — LAPACK getrf's layout, sparse.py:109-137).
// Two-level right-looking LU: outer panels of kNB2 columns are factorised by kNB-wide steps
// whose rank-kNB updates stay inside the panel; the trailing matrix then receives one
// rank-kNB2 GEMM update per outer panel (compute-bound instead of C-traffic-bound).
// `dominant`: the columns are diagonally dominant, so partial pivoting never interchanges
// and the pivot-free path (k_diag_lu + k_trsm_rows) is the same factorisation.
// Writes min |U_kk| to *min_pivot (host).
int lu_factor(double* E, int d, int ld, int* piv, bool dominant, double* min_pivot,
              cudaStream_t s) {
  const unsigned cgrid = (unsigned)((d + 255) / 256);
  auto at = [&](int r, int c) { return E + (long long)r * ld + c; };
  for (int K0 = 0; K0 < d; K0 += kNB2) {
    const int Kend = (d - K0 < kNB2) ? d : K0 + kNB2;
    for (int k = K0; k < Kend; k += kNB) {
      const int nb = (Kend - k < kNB) ? Kend - k : kNB;
      const int rest = d - k - nb;
      if (dominant) {
        k_diag_lu<<<1, 256, 0, s>>>(E, ld, k, nb, piv);
        if (rest > 0) k_trsm_rows<<<(rest + 255) / 256, 256, 0, s>>>(E, d, ld, k, nb);
      } else {
        k_panel<<<1, 1024, 0, s>>>(E, d, ld, k, nb, piv);
        k_laswp<<<cgrid, 256, 0, s>>>(E, d, ld, piv, k, k + nb, k, k + nb);
      }
      const int inpanel = Kend - k - nb;
      if (inpanel > 0) {
        k_trsm_block<false><<<(inpanel + 255) / 256, 256, 0, s>>>(E, ld, k, nb, E, ld, k + nb,
                                                                   Kend);
        dgemm_sub(at(k + nb, k), ld, at(k, k + nb), ld, at(k + nb, k + nb), ld, rest, inpanel,
                  nb, s);
      }
    }
    const int right = d - Kend;
    if (right > 0) {
      // U12 = L11^-1 A12 for the columns right of the outer panel
      for (int k = K0; k < Kend; k += kNB) {
        const int nb = (Kend - k < kNB) ? Kend - k : kNB;
        k_trsm_block<false><<<(right + 255) / 256, 256, 0, s>>>(E, ld, k, nb, E, ld, Kend, d);
        if (k + nb < Kend)
          dgemm_sub(at(k + nb, k), ld, at(k, Kend), ld, at(k + nb, Kend), ld, Kend - k - nb,
                    right, nb, s);
      }
      dgemm_sub(at(Kend, K0), ld, at(K0, Kend), ld, at(Kend, Kend), ld, right, right,
                Kend - K0, s);
    }
  }
  double* dmin = nullptr;
  cudaMallocAsync(&dmin, sizeof(double), s);
  k_min_pivot<<<1, 1024, 0, s>>>(E, d, ld, dmin);
  cudaMemcpyAsync(min_pivot, dmin, sizeof(double), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  cudaFreeAsync(dmin, s);
  return (int)cudaGetLastError();
}

// X <- U^-1 L^-1 P X for the d x ncols block X (row-major, ldx): the row interchanges, then
// the unit-lower and the upper triangular solves, each two-level (kNB-wide substitution
// blocks, rank-kNB2 GEMM updates) — LAPACK getrs (sparse.py:140-145).  `lower_fill`: X = P
// with no interchanges, so L^-1 X stays lower triangular and the forward sweep of row block
// [K0, Kend) only touches columns [0, Kend).
void lu_solve_rows(const double* E, int d, int ld, const int* piv, double* X, int ldx,
                   int ncols, bool lower_fill, cudaStream_t s) {
  const unsigned xgrid = (unsigned)((ncols + 255) / 256);
  auto at = [&](int r, int c) { return E + (long long)r * ld + c; };
  auto xt = [&](int r, int c) { return X + (long long)r * ldx + c; };
  k_laswp<<<xgrid, 256, 0, s>>>(X, ncols, ldx, piv, 0, d, 0, 0);
  for (int K0 = 0; K0 < d; K0 += kNB2) {  // L Y = P X
    const int Kend = (d - K0 < kNB2) ? d : K0 + kNB2;
    const int nc = lower_fill && Kend < ncols ? Kend : ncols;
    for (int k = K0; k < Kend; k += kNB) {
      const int nb = (Kend - k < kNB) ? Kend - k : kNB;
      k_trsm_block<false><<<(nc + 255) / 256, 256, 0, s>>>(E, ld, k, nb, X, ldx, 0, nc);
      if (k + nb < Kend)
        dgemm_sub(at(k + nb, k), ld, xt(k, 0), ldx, xt(k + nb, 0), ldx, Kend - k - nb, nc, nb,
                  s);
    }
    if (Kend < d)
      dgemm_sub(at(Kend, K0), ld, xt(K0, 0), ldx, xt(Kend, 0), ldx, d - Kend, nc, Kend - K0, s);
  }
  const int lastK0 = ((d - 1) / kNB2) * kNB2;
  for (int K0 = lastK0; K0 >= 0; K0 -= kNB2) {  // U X = Y, from the bottom
    const int Kend = (d - K0 < kNB2) ? d : K0 + kNB2;
    const int lastk = K0 + ((Kend - K0 - 1) / kNB) * kNB;
    for (int k = lastk; k >= K0; k -= kNB) {
      const int nb = (Kend - k < kNB) ? Kend - k : kNB;
      k_trsm_block<true><<<xgrid, 256, 0, s>>>(E, ld, k, nb, X, ldx, 0, ncols);
      if (k > K0) dgemm_sub(at(K0, k), ld, xt(k, 0), ldx, xt(K0, 0), ldx, k - K0, ncols, nb, s);
    }
    if (K0 > 0)
      dgemm_sub(at(0, K0), ld, xt(K0, 0), ldx, xt(0, 0), ldx, K0, ncols, Kend - K0, s);
  }
}

int lu_and_inverse(double* E, int d, int ld, double* Einv, int* piv, double* min_pivot,
                   float* ms_lu, float* ms_inv, cudaStream_t s) {
  cudaEvent_t e0, e1, e2;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventCreate(&e2);
  cudaEventRecord(e0, s);
  const bool dominant = column_dominant(E, d, ld, s) != 0;
  int err = lu_factor(E, d, ld, piv, dominant, min_pivot, s);
  cudaEventRecord(e1, s);
  if (err || !(*min_pivot >= 1e-300)) {  // singular (or NaN): no inverse
    cudaStreamSynchronize(s);
    cudaEventElapsedTime(ms_lu, e0, e1);
    *ms_inv = 0.f;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    return err ? err : (int)cudaGetLastError();
  }
  // Einv = U^-1 L^-1 P I
  k_identity<<<num_sms() * 8, 256, 0, s>>>(Einv, d, ld);
  lu_solve_rows(E, d, ld, piv, Einv, ld, d, dominant, s);
  cudaEventRecord(e2, s);
  cudaStreamSynchronize(s);
  cudaEventElapsedTime(ms_lu, e0, e1);
  cudaEventElapsedTime(ms_inv, e1, e2);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  return (int)cudaGetLastError();
}

}  // namespace dk
