// dk_profile.cu — the coarse solve of a symmetric positive definite E through its inverse
// Cholesky factor in a nested-dissection order of the labels.
//
// E = Z^T A Z couples two labels only when their cells touch, so E is the (weighted) adjacency
// matrix of the label graph: ~6 neighbours per label at config 3.  Ordered by nested
// dissection, E~ = P E P^T has a Cholesky factor L whose inverse W = L^-1 is nonzero only where
// row i's separator lies above column j's in the dissection tree — 14 % of the lower 32 x 32
// tile triangle at config 3 instead of the 100 % of E^-1.  y = E^-1 s becomes
//     s~ = P s,  t = W s~,  y~ = W^T t,  y = P^T y~
// two streaming passes over the nonzero tiles of W (k_tgemv), 0.28x the bytes of the packed
// symmetric E^-1 (reference semantics unchanged: deflation.py:50-62 applies E^-1 exactly; the
// factor differs from the reference's LU solve only by rounding).
//
// Set-up pieces: E's pattern (k_row_nnz / k_row_cols), a level-structure nested dissection
// of the label graph on the host (nd_order), the symmetric permutation (k_permute_sym), the
// nonzero-tile lists of W and the packed tile streams (k_tile_nz, k_tile_pack).
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "dk_launch.h"

namespace dk {

namespace {

constexpr int kPT = 32;                    // tile edge
constexpr int kPTileBytes = kPT * kPT * 8;  // 8 KB
constexpr int kPSegBytes = kPT * 8;         // x segment of a tile, 256 B

// ---- E's off-diagonal pattern, one warp per row ----------------------------------------
__global__ void k_row_nnz(const double* __restrict__ E, int d, int ld, int* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < d;
       r += gridDim.x * (blockDim.x >> 5)) {
    int k = 0;
    for (int c0 = 0; c0 < d; c0 += 32) {
      const int c = c0 + lane;
      k += __popc(__ballot_sync(0xffffffffu, c < d && c != r && E[(long long)r * ld + c] != 0.0));
    }
    if (lane == 0) cnt[r] = k;
  }
}

__global__ void k_row_cols(const double* __restrict__ E, int d, int ld,
                           const int* __restrict__ ptr, int* __restrict__ col) {
  const int lane = threadIdx.x & 31;
  for (int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < d;
       r += gridDim.x * (blockDim.x >> 5)) {
    int k = ptr[r];
    for (int c0 = 0; c0 < d; c0 += 32) {
      const int c = c0 + lane;
      const bool nz = c < d && c != r && E[(long long)r * ld + c] != 0.0;
      const unsigned m = __ballot_sync(0xffffffffu, nz);
      if (nz) col[k + __popc(m & ((1u << lane) - 1u))] = c;
      k += __popc(m);
    }
  }
}

// out[i][j] = E[perm[i]][perm[j]] (full matrix), one warp per row
__global__ void k_permute_sym(const double* __restrict__ E, int d, int ld,
                              const int* __restrict__ perm, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < d;
       i += gridDim.x * (blockDim.x >> 5)) {
    const double* src = E + (long long)perm[i] * ld;
    double* dst = out + (long long)i * ld;
    for (int j = lane; j < d; j += 32) dst[j] = src[perm[j]];
  }
}

// out[perm[i]][perm[j]] = X[i][j]: back to the label order
__global__ void k_unpermute_sym(const double* __restrict__ X, int d, int ld,
                                const int* __restrict__ perm, double* __restrict__ out,
                                int ldo) {
  const int lane = threadIdx.x & 31;
  for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < d;
       i += gridDim.x * (blockDim.x >> 5)) {
    const double* src = X + (long long)i * ld;
    double* dst = out + (long long)perm[i] * ldo;
    for (int j = lane; j < d; j += 32) dst[perm[j]] = src[j];
  }
}

// flag[t] = 1 when tile (ti[t], tj[t]) of X holds a nonzero; one warp per tile
__global__ void k_tile_nz(const double* __restrict__ X, int d, int ld, const int* __restrict__ ti,
                          const int* __restrict__ tj, long long nt, int* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  for (long long t = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); t < nt;
       t += (long long)gridDim.x * (blockDim.x >> 5)) {
    const int r0 = ti[t] * kPT, c = tj[t] * kPT + lane;
    bool nz = false;
    for (int r = r0; r < r0 + kPT && r < d; ++r)
      nz |= c < d && X[(long long)r * ld + c] != 0.0;
    nz = __any_sync(0xffffffffu, nz);
    if (lane == 0) flag[t] = nz ? 1 : 0;
  }
}

// Tile t of a stream: element (r, c) of block (ti[t], tj[t]) of X, or of X^T when trans,
// stored [16 column pairs][32 rows][2] (one coalesced 512 B double2 load per pair).
__global__ void k_tile_pack(const double* __restrict__ X, int d, int ld, const int* __restrict__ ti,
                            const int* __restrict__ tj, long long nt, int trans,
                            double* __restrict__ out) {
  const long long tot = nt * kPT * kPT;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const long long t = e / (kPT * kPT);
    const int w = (int)(e % (kPT * kPT));
    const int pair = w / (2 * kPT), r = (w / 2) % kPT, c = 2 * pair + (w & 1);
    // output block R = ti, input block C = tj: element (R*32 + r, C*32 + c) of X, or of X^T
    // (= X[C*32 + c][R*32 + r])
    const long long gr = (long long)ti[t] * kPT + r, gc = (long long)tj[t] * kPT + c;
    double v = 0.0;
    if (gr < d && gc < d) v = trans ? X[gc * ld + gr] : X[gr * ld + gc];
    out[e] = v;
  }
}

// ---- the tile-sparse GEMV ------------------------------------------------------------
// y_R = sum over the tiles t of output block R (in stream order) of T_t x_{col(t)}.
// Each warp streams a contiguous, balanced range of tiles: one-lane TMA copies of the 8 KB
// tile and its 256 B x segment complete on the stage's mbarrier; lane r owns row r, so the
// row sum accumulates in a register across the warp's tiles of one output block.  A block
// whose tiles span several warps is finished by the last of them to arrive (row ticket),
// summing the pieces in warp order: deterministic.  With scatter, output row i goes to
// y[scatter[i]] (back to the label order).
constexpr int kTgStages = 2;
constexpr int kTgStageBytes = kPTileBytes + kPSegBytes;

// bulk copy on an mbarrier whose expect_tx the caller already posted; the tile streams are
// read once per pass (evict-first), the x segments are reused (default policy)
__device__ __forceinline__ void tma_copy_nx(void* dst, const void* src, unsigned bytes,
                                            unsigned long long* bar, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_copy_x(void* dst, const void* src, unsigned bytes,
                                           unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
// post the stage's byte count, then its tile and x segment
__device__ __forceinline__ void tg_issue(unsigned char* b, const double* T, const double* xseg,
                                         unsigned long long* bar, unsigned long long pol) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"((unsigned)kTgStageBytes)
               : "memory");
  tma_copy_nx(b, T, kPTileBytes, bar, pol);
  tma_copy_x(b + kPTileBytes, xseg, kPSegBytes, bar);
}

__global__ void __launch_bounds__(kTgWarps * 32, 1) k_tgemv(TileGemv g, const double* __restrict__ x,
                                                            double* __restrict__ y,
                                                            const int* __restrict__ scatter, int d,
                                                            const int* __restrict__ gate) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long bars[kTgWarps][kTgStages];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  unsigned char* wbuf = smem_raw + (size_t)wl * kTgStages * kTgStageBytes;
  // g.nw <= nt warps hold the tiles, every one of them at least one
  const long long Wn = g.nw;
  const long long w = (long long)blockIdx.x * kTgWarps + wl;
  const long long t0 = w < Wn ? w * g.nt / Wn : g.nt, t1 = w < Wn ? (w + 1) * g.nt / Wn : g.nt;
  const unsigned long long pol = l2_evict_first();
  if (lane == 0)
    for (int s = 0; s < kTgStages; ++s) mbar_init1(&bars[wl][s]);
  mbar_init_fence();
  __syncwarp();
  // The tiles and their metadata are set-up constants: fetched before the dependency wait,
  // so they stream in while the producer of x drains.  Lane k holds tile t0 + k's blocks.
  const int nfirst = t1 - t0 < kTgStages ? (int)(t1 - t0) : kTgStages;
  const int my_row = (t0 + lane < t1) ? g.trow[t0 + lane] : -1;
  const int my_col = (t0 + lane < t1) ? g.tcol[t0 + lane] : 0;
  if (lane == 0)
    for (int s = 0; s < nfirst; ++s) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       smem_addr(&bars[wl][s])),
                   "r"((unsigned)kTgStageBytes)
                   : "memory");
      tma_copy_nx(wbuf + s * kTgStageBytes, g.T + (t0 + s) * (kPT * kPT), kPTileBytes,
                  &bars[wl][s], pol);
    }
  pdl_wait();
  const bool off = gate != nullptr && *gate == 0;
  for (int s = 0; s < nfirst; ++s) {
    const int c = __shfl_sync(0xffffffffu, my_col, s);
    if (lane == 0)
      tma_copy_x(wbuf + s * kTgStageBytes + kPTileBytes, x + (long long)c * kPT, kPSegBytes,
                 &bars[wl][s]);
  }
  if (off) {  // drain the copies already in flight, then leave
    for (int s = 0; s < nfirst; ++s) mbar_wait_parity(&bars[wl][s], 0);
    return;
  }
  if (t0 >= t1) return;
  int R = __shfl_sync(0xffffffffu, my_row, 0);
  double racc = 0.0;
  for (long long t = t0; t < t1; ++t) {
    const int k = (int)(t - t0);
    const int s = k % kTgStages;
    const unsigned parity = (unsigned)((k / kTgStages) & 1);
    // metadata of tile t + kTgStages (refill) and t + 1 (block change)
    const int kr = k + kTgStages, kn = k + 1;
    const int col_r = kr < 32 ? __shfl_sync(0xffffffffu, my_col, kr & 31)
                              : (t + kTgStages < t1 ? g.tcol[t + kTgStages] : 0);
    const int row_n = kn < 32 ? __shfl_sync(0xffffffffu, my_row, kn & 31)
                              : (t + 1 < t1 ? g.trow[t + 1] : -1);
    mbar_wait_parity(&bars[wl][s], parity);
    const unsigned char* b = wbuf + s * kTgStageBytes;
    const double2* T = reinterpret_cast<const double2*>(b);
    const double2* xs = reinterpret_cast<const double2*>(b + kPTileBytes);
#pragma unroll
    for (int p = 0; p < 16; ++p) {
      const double2 a = T[p * kPT + lane], xx = xs[p];
      racc = fma(a.x, xx.x, racc);
      racc = fma(a.y, xx.y, racc);
    }
    __syncwarp();
    if (lane == 0 && t + kTgStages < t1)  // refill this stage
      tg_issue(wbuf + s * kTgStageBytes, g.T + (t + kTgStages) * (kPT * kPT),
               x + (long long)col_r * kPT, &bars[wl][s], pol);
    const int Rn = (t + 1 < t1) ? row_n : -1;
    if (Rn == R) continue;
    // output block R ends in this warp's range
    const int np = g.rnp[R];
    double out = racc;
    bool write = true;
    if (np > 1) {
      const int q0 = g.rslot[R] + (int)(w - g.rfirst[R]);
      g.part[(long long)q0 * kPT + lane] = racc;
      __threadfence();
      __syncwarp();
      unsigned old = 0;
      if (lane == 0) old = atomicAdd(g.cnt + R, 1u);
      old = __shfl_sync(0xffffffffu, old, 0);
      write = old == (unsigned)(np - 1);
      if (write) {
        __threadfence();
        out = 0.0;
        const double* p0 = g.part + (long long)g.rslot[R] * kPT;
        for (int q = 0; q < np; ++q) out += __ldcg(p0 + (long long)q * kPT + lane);
        if (lane == 0) g.cnt[R] = 0u;
      }
    }
    if (write) {
      const int row = R * kPT + lane;
      if (row < d) y[scatter ? scatter[row] : row] = out;
    }
    racc = 0.0;
    R = Rn;
  }
}

// ---- host: level-structure nested dissection -----------------------------------------
struct NestedDissection {
  const std::vector<int>& ptr;
  const std::vector<int>& col;
  std::vector<int> part, level, order, seen;
  int next_id = 2;
  int leaf;

  NestedDissection(int d, const std::vector<int>& p, const std::vector<int>& c, int lf)
      : ptr(p), col(c), part(d, 1), level(d, -1), leaf(lf) {
    order.reserve(d);
  }

  int deg(int v) const { return ptr[v + 1] - ptr[v]; }

  // BFS from src inside part pid; levels set, visit order in `seen`
  void bfs(int src, int pid) {
    seen.clear();
    level[src] = 0;
    seen.push_back(src);
    for (size_t h = 0; h < seen.size(); ++h) {
      const int u = seen[h];
      for (int k = ptr[u]; k < ptr[u + 1]; ++k) {
        const int v = col[k];
        if (part[v] == pid && level[v] < 0) {
          level[v] = level[u] + 1;
          seen.push_back(v);
        }
      }
    }
  }

  void emit_sorted(std::vector<int>& nodes) {
    std::sort(nodes.begin(), nodes.end());
    for (int v : nodes) {
      part[v] = 0;
      order.push_back(v);
    }
  }

  void rec(std::vector<int> nodes, int pid) {
    if ((int)nodes.size() <= leaf) {
      emit_sorted(nodes);
      return;
    }
    std::sort(nodes.begin(), nodes.end());
    for (int v : nodes) level[v] = -1;
    std::vector<std::vector<int>> comps;
    for (int v : nodes)
      if (level[v] < 0) {
        bfs(v, pid);
        comps.push_back(seen);
      }
    if (comps.size() > 1) {
      std::vector<int> ids;
      for (auto& c : comps) {
        const int id = next_id++;
        ids.push_back(id);
        for (int v : c) part[v] = id;
      }
      for (size_t i = 0; i < comps.size(); ++i) rec(std::move(comps[i]), ids[i]);
      return;
    }
    std::vector<int>& comp = comps[0];
    // pseudo-peripheral start: repeated BFS from a minimum-degree node of the last level
    int src = comp[0];
    for (int v : comp)
      if (deg(v) < deg(src)) src = v;
    int ecc = -1;
    for (;;) {
      for (int v : comp) level[v] = -1;
      bfs(src, pid);
      const int e = level[seen.back()];
      if (e <= ecc) break;
      ecc = e;
      int best = -1;
      for (int i = (int)seen.size() - 1; i >= 0 && level[seen[i]] == e; --i)
        if (best < 0 || deg(seen[i]) < deg(best)) best = seen[i];
      src = best;
    }
    const int nl = level[seen.back()] + 1;
    const long long n = (long long)seen.size();
    std::vector<long long> cnt(nl, 0), cum(nl, 0);
    for (int v : seen) ++cnt[level[v]];
    for (int l = 0; l < nl; ++l) cum[l] = cnt[l] + (l ? cum[l - 1] : 0);
    // the separator level: smallest level with 25-75 % of the nodes on either side
    int L = -1;
    for (int l = 1; l + 1 < nl; ++l)
      if (4 * cum[l - 1] >= n && 4 * cum[l] <= 3 * n && (L < 0 || cnt[l] < cnt[L])) L = l;
    if (L < 0) {
      L = 0;
      while (L < nl - 1 && 2 * cum[L] < n) ++L;
    }
    std::vector<int> sep, A, B;
    for (int v : seen) {
      if (level[v] > L) {
        B.push_back(v);
      } else if (level[v] == L) {
        bool cut = false;
        for (int k = ptr[v]; k < ptr[v + 1] && !cut; ++k)
          cut = part[col[k]] == pid && level[col[k]] == L + 1;
        (cut ? sep : A).push_back(v);
      } else {
        A.push_back(v);
      }
    }
    if (A.empty() || B.empty()) {
      emit_sorted(comp);
      return;
    }
    const int ida = next_id++, idb = next_id++;
    for (int v : A) part[v] = ida;
    for (int v : B) part[v] = idb;
    for (int v : sep) part[v] = 0;
    rec(std::move(A), ida);
    rec(std::move(B), idb);
    for (int v : sep) order.push_back(v);
  }
};

}  // namespace

void nd_order(int d, const std::vector<int>& ptr, const std::vector<int>& col,
              std::vector<int>& perm) {
  NestedDissection nd(d, ptr, col, 64);
  std::vector<int> all(d);
  for (int i = 0; i < d; ++i) all[i] = i;
  nd.rec(std::move(all), 1);
  perm.swap(nd.order);
}

long long nd_profile_tiles(int d, const std::vector<int>& ptr, const std::vector<int>& col,
                           const std::vector<int>& perm) {
  // the row profile f of E~, closed under W = L^-1: g(i) = min(f(i), min_{f(i)<=k<i} g(k)),
  // evaluated with a sparse-table-free sweep (g is checked over the range once per row)
  std::vector<int> inv(d), f(d), g(d);
  for (int i = 0; i < d; ++i) inv[perm[i]] = i;
  for (int i = 0; i < d; ++i) f[i] = i;
  for (int v = 0; v < d; ++v)
    for (int k = ptr[v]; k < ptr[v + 1]; ++k) f[inv[v]] = std::min(f[inv[v]], inv[col[k]]);
  // block-level closure is enough for a tile count: gb(I) = min over I's rows
  const int nb = (d + kPT - 1) / kPT;
  std::vector<int> fb(nb, 1 << 30), gb(nb);
  for (int i = 0; i < d; ++i) fb[i / kPT] = std::min(fb[i / kPT], f[i] / kPT);
  long long tiles = 0;
  for (int I = 0; I < nb; ++I) {
    int m = fb[I];
    for (int K = fb[I]; K < I; ++K) m = std::min(m, gb[K]);
    gb[I] = m;
    tiles += I - m + 1;
  }
  return tiles;
}

int coarse_pattern(const double* E, int d, int ld, std::vector<int>& ptr, std::vector<int>& col,
                   cudaStream_t s) {
  int* dcnt = nullptr;
  int* dptr = nullptr;
  int* dcol = nullptr;
  cudaMallocAsync(&dcnt, (size_t)d * sizeof(int), s);
  k_row_nnz<<<148 * 4, 256, 0, s>>>(E, d, ld, dcnt);
  std::vector<int> cnt(d);
  cudaMemcpyAsync(cnt.data(), dcnt, (size_t)d * sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return (int)e;
  ptr.assign(d + 1, 0);
  for (int i = 0; i < d; ++i) ptr[i + 1] = ptr[i] + cnt[i];
  col.resize(ptr[d]);
  cudaMallocAsync(&dptr, (size_t)(d + 1) * sizeof(int), s);
  cudaMallocAsync(&dcol, (size_t)std::max(ptr[d], 1) * sizeof(int), s);
  cudaMemcpyAsync(dptr, ptr.data(), (size_t)(d + 1) * sizeof(int), cudaMemcpyHostToDevice, s);
  k_row_cols<<<148 * 4, 256, 0, s>>>(E, d, ld, dptr, dcol);
  if (ptr[d] > 0)
    cudaMemcpyAsync(col.data(), dcol, (size_t)ptr[d] * sizeof(int), cudaMemcpyDeviceToHost, s);
  e = cudaStreamSynchronize(s);
  cudaFreeAsync(dcnt, s);
  cudaFreeAsync(dptr, s);
  cudaFreeAsync(dcol, s);
  return e != cudaSuccess ? (int)e : (int)cudaGetLastError();
}

void launch_permute_sym(const double* E, int d, int ld, const int* perm, double* out,
                        cudaStream_t s) {
  k_permute_sym<<<148 * 8, 256, 0, s>>>(E, d, ld, perm, out);
}

void launch_unpermute_sym(const double* X, int d, int ld, const int* perm, double* out, int ldo,
                          cudaStream_t s) {
  k_unpermute_sym<<<148 * 8, 256, 0, s>>>(X, d, ld, perm, out, ldo);
}

// Nonzero tiles of W (lower triangle, row profile fW from k_row_first_nz) as two streams:
// pass 1 by block rows of W (t = W s~), pass 2 by block columns of W, tiles transposed
// (y~ = W^T t).  Host metadata for the row tickets of k_tgemv.
static int build_stream(const std::vector<int>& ti, const std::vector<int>& tj, int nrows,
                        TileGemvHost& h) {
  const long long nt = (long long)ti.size();
  h.nt = nt;
  h.trow = ti;
  h.tcol = tj;
  h.rfirst.assign(nrows, 0);
  h.rslot.assign(nrows, 0);
  h.rnp.assign(nrows, 0);
  std::vector<long long> rs(nrows + 1, 0);
  for (long long t = 0; t < nt; ++t) ++rs[ti[t] + 1];
  for (int R = 0; R < nrows; ++R) rs[R + 1] += rs[R];
  const long long Wn = std::min<long long>((long long)kTgGrid * kTgWarps, nt);
  h.nw = (int)Wn;
  auto warp_of = [&](long long t) {  // the warp whose range [w nt / Wn, (w+1) nt / Wn) holds t
    long long w = (t * Wn) / nt;
    while (w > 0 && w * nt / Wn > t) --w;
    while ((w + 1) * nt / Wn <= t) ++w;
    return w;
  };
  int slots = 0;
  for (int R = 0; R < nrows; ++R) {
    if (rs[R + 1] == rs[R]) return -1;  // every output block holds its diagonal tile
    const long long wa = warp_of(rs[R]), wb = warp_of(rs[R + 1] - 1);
    h.rfirst[R] = (int)wa;
    h.rnp[R] = (int)(wb - wa + 1);
    h.rslot[R] = slots;
    if (wb > wa) slots += (int)(wb - wa + 1);
  }
  h.nslots = std::max(slots, 1);
  return 0;
}

int profile_streams(const double* W, int d, int ld, const std::vector<int>& fW,
                    TileGemvHost& p1, TileGemvHost& p2, cudaStream_t s) {
  const int nb = (d + kPT - 1) / kPT;
  std::vector<int> fb(nb, 1 << 30);
  for (int i = 0; i < d; ++i) fb[i / kPT] = std::min(fb[i / kPT], fW[i] / kPT);
  std::vector<int> ci, cj;
  for (int I = 0; I < nb; ++I)
    for (int J = fb[I]; J <= I; ++J) {
      ci.push_back(I);
      cj.push_back(J);
    }
  const long long nc = (long long)ci.size();
  int *dti = nullptr, *dtj = nullptr, *dfl = nullptr;
  cudaMallocAsync(&dti, nc * sizeof(int), s);
  cudaMallocAsync(&dtj, nc * sizeof(int), s);
  cudaMallocAsync(&dfl, nc * sizeof(int), s);
  cudaMemcpyAsync(dti, ci.data(), nc * sizeof(int), cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(dtj, cj.data(), nc * sizeof(int), cudaMemcpyHostToDevice, s);
  k_tile_nz<<<148 * 8, 256, 0, s>>>(W, d, ld, dti, dtj, nc, dfl);
  std::vector<int> fl(nc);
  cudaMemcpyAsync(fl.data(), dfl, nc * sizeof(int), cudaMemcpyDeviceToHost, s);
  cudaError_t e = cudaStreamSynchronize(s);
  cudaFreeAsync(dti, s);
  cudaFreeAsync(dtj, s);
  cudaFreeAsync(dfl, s);
  if (e != cudaSuccess) return (int)e;
  std::vector<int> ai, aj;  // pass 1: row-major
  for (long long t = 0; t < nc; ++t)
    if (fl[t] || ci[t] == cj[t]) {
      ai.push_back(ci[t]);
      aj.push_back(cj[t]);
    }
  // pass 2: grouped by W's block column J (output block of W^T), rows I ascending
  std::vector<long long> idx(ai.size());
  for (size_t k = 0; k < idx.size(); ++k) idx[k] = (long long)k;
  std::stable_sort(idx.begin(), idx.end(), [&](long long a, long long b) { return aj[a] < aj[b]; });
  std::vector<int> bi(ai.size()), bj(ai.size());
  for (size_t k = 0; k < idx.size(); ++k) {
    bi[k] = aj[idx[k]];  // output block of W^T
    bj[k] = ai[idx[k]];  // input block
  }
  if (build_stream(ai, aj, nb, p1) || build_stream(bi, bj, nb, p2)) return -1;
  return 0;
}

int upload_stream(const double* W, int d, int ld, bool trans, const TileGemvHost& h, TileGemv& g,
                  cudaStream_t s) {
  const int nrows = (int)h.rnp.size();
  g.nt = h.nt;
  g.nw = h.nw;
  g.nrows = nrows;
  cudaError_t e = cudaSuccess;
  auto up = [&](int** dst, const std::vector<int>& v) {
    if (e == cudaSuccess) e = cudaMallocAsync(dst, std::max<size_t>(v.size(), 1) * sizeof(int), s);
    if (e == cudaSuccess && !v.empty())
      e = cudaMemcpyAsync(*dst, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice, s);
  };
  int *trow = nullptr, *tcol = nullptr, *rfirst = nullptr, *rslot = nullptr, *rnp = nullptr;
  up(&trow, h.trow);
  up(&tcol, h.tcol);
  up(&rfirst, h.rfirst);
  up(&rslot, h.rslot);
  up(&rnp, h.rnp);
  g.trow = trow;
  g.tcol = tcol;
  g.rfirst = rfirst;
  g.rslot = rslot;
  g.rnp = rnp;
  if (e == cudaSuccess)
    e = cudaMallocAsync(&g.part, (size_t)h.nslots * kPT * sizeof(double), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&g.cnt, (size_t)nrows * sizeof(unsigned), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(g.cnt, 0, (size_t)nrows * sizeof(unsigned), s);
  if (e != cudaSuccess) return (int)e;
  // the tile stream itself (big_alloc'd by the caller into g.T)
  k_tile_pack<<<148 * 8, 256, 0, s>>>(W, d, ld, trow, tcol, h.nt, trans ? 1 : 0,
                                      const_cast<double*>(g.T));
  return (int)cudaGetLastError();
}

void free_stream(TileGemv& g, cudaStream_t s) {
  void* bufs[] = {(void*)g.trow, (void*)g.tcol, (void*)g.rfirst, (void*)g.rslot, (void*)g.rnp,
                  (void*)g.part, (void*)g.cnt};
  for (void* p : bufs)
    if (p) cudaFreeAsync(p, s);
  g.trow = g.tcol = g.rfirst = g.rslot = g.rnp = nullptr;
  g.part = nullptr;
  g.cnt = nullptr;
}

void launch_tgemv(const TileGemv& g, const double* x, double* y, const int* scatter, int d,
                  const int* gate, cudaStream_t s) {
  const size_t smem = (size_t)kTgWarps * kTgStages * kTgStageBytes;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_tgemv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  const unsigned grid = (unsigned)((g.nw + kTgWarps - 1) / kTgWarps);
  launch_pdl(k_tgemv, dim3(grid), dim3(kTgWarps * 32), smem, s, g, x, y, scatter, d, gate);
}

}  // namespace dk
