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
#include <cstdio>
#include <atomic>
#include <future>
#include <cstdlib>
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
// Each warp streams a contiguous, balanced range of tiles through KS shared-memory stages
// filled by one-lane TMA bulk copies (8 KB, completion on the stage's mbarrier); lane r owns
// row r, so the row sum accumulates in a register across the warp's tiles of one output
// block.  Lane c holds x_{col(t)}[c] (read after the dependency wait, the first kXPre tiles'
// segments prefetched at once) and broadcasts it by shuffle.  A block whose tiles span
// several warps is finished by the first of them, which reads the others' pieces from
// self-validating slots (sentinel until written; no fence, no ticket) and sums them in warp
// order: deterministic.  With scatter, output row i goes to y[scatter[i]].
constexpr int kXPre = 8;
constexpr int kTgLongBatch = 16;  // = k_restrict_final's kLongBatch (bitwise-equal sums)

// partial-row slots hold this bit pattern until written (a negative NaN with a full payload:
// never the result of arithmetic, which yields the canonical NaN)
__device__ __forceinline__ double sentinel_f64() { return __longlong_as_double(-1ll); }
__device__ __forceinline__ bool is_sentinel(double v) { return __double_as_longlong(v) == -1ll; }
__device__ __forceinline__ double ld_volatile_f64(const double* p) {
  return *reinterpret_cast<const volatile double*>(p);
}

// bulk copy of one tile on an mbarrier (evict-first: each tile is read once per pass)
__device__ __forceinline__ void tg_issue(unsigned char* b, const double* T,
                                         unsigned long long* bar, unsigned long long pol) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"((unsigned)kPTileBytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(b)),
      "l"(T), "r"((unsigned)kPTileBytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}

// Transposed tile product: lane r holds x_r of the tile's input block and accumulates
// acc[c] += T[r][c] x_r over every tile of the output block (no shuffles per tile); at the
// block's end a butterfly transpose-reduction (31 shuffles) leaves column `lane`'s sum in
// acc[0] of lane `lane`.  The pairing is fixed: deterministic.
__device__ __forceinline__ double butterfly_sum32(double (&v)[32], int lane) {
#pragma unroll
  for (int h = 16; h >= 1; h >>= 1) {
    const bool up = (lane & h) != 0;
#pragma unroll
    for (int k = 0; k < h; ++k) {
      const double send = up ? v[k] : v[k + h];
      const double keep = up ? v[k + h] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, h);
    }
  }
  return v[0];
}

// NOSPIN (DK_NO_SPIN, or a grid that cannot be co-resident): no warp waits for another —
// every piece of a split block goes to its slot and k_tg_finish sums them after the grid
// (same order, bitwise equal).
// grid barrier of the fused pass 1 (cooperative launch: all blocks resident): release-add
// arrival, relaxed polling of the generation, acquire; the last arriver resets the count
__device__ __forceinline__ void tg_grid_barrier(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned* count = bar;
    unsigned* gen = bar + 1;
    unsigned g0;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g0) : "l"(gen) : "memory");
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(count)
                 : "memory");
    if (old == gridDim.x - 1) {
      *reinterpret_cast<volatile unsigned*>(count) = 0u;
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g0 + 1u) : "memory");
    } else {
      while (*reinterpret_cast<volatile unsigned*>(gen) == g0) __nanosleep(20);
      unsigned t;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(t) : "l"(gen) : "memory");
    }
  }
  __syncthreads();
}

// s~ = the column sums of the stencil's run partials, each block a slice of the short
// columns (thread per column, all <= kShortRuns loads in flight, in-order sum) and every
// grid-th long column (warp per column, kLongBatch loads per lane, xor tree): exactly
// k_restrict_final's arithmetic
__device__ __forceinline__ void tg_restrict(const RunMap& rm, double* __restrict__ s_out) {
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int d = rm.d;
  const int per = (d + gridDim.x - 1) / gridDim.x;
  const int L0 = blockIdx.x * per, L1 = min(d, L0 + per);
  for (int L = L0 + threadIdx.x; L < L1; L += blockDim.x) {
    const int lo = rm.lab_run_ptr[L], len = rm.lab_run_ptr[L + 1] - lo;
    if (len > kShortRuns) continue;
    double v[kShortRuns];
#pragma unroll
    for (int k = 0; k < kShortRuns; ++k) v[k] = k < len ? __ldcg(rm.run_part + lo + k) : 0.0;
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < kShortRuns; ++k)
      if (k < len) acc += v[k];
    s_out[rm.s_pos ? rm.s_pos[L] : L] = acc;
  }
  for (int k = blockIdx.x * nwarp + wl; k < rm.nlong; k += gridDim.x * nwarp) {
    const int L = rm.long_ids[k];
    double acc = 0.0;
    const int lo = rm.lab_run_ptr[L], hi = rm.lab_run_ptr[L + 1];
    for (int k0 = lo + lane; k0 < hi; k0 += 32 * kTgLongBatch) {
      double v[kTgLongBatch];
#pragma unroll
      for (int i = 0; i < kTgLongBatch; ++i)
        v[i] = k0 + 32 * i < hi ? __ldcg(rm.run_part + k0 + 32 * i) : 0.0;
#pragma unroll
      for (int i = 0; i < kTgLongBatch; ++i)
        if (k0 + 32 * i < hi) acc += v[i];
    }
    acc = warp_sum(acc);
    if (lane == 0) s_out[rm.s_pos ? rm.s_pos[L] : L] = acc;
  }
}

template <int KW, int KS, bool TRANS, bool NOSPIN, bool FUSE_R = false>
__global__ void __launch_bounds__(KW * 32, 1) k_tgemv(TileGemv g, const double* __restrict__ x,
                                                      double* __restrict__ y,
                                                      const int* __restrict__ scatter, int d,
                                                      const int* __restrict__ gate,
                                                      RunMap rm, double* s_out) {
  DK_TL(TRANS ? TL_TG2 : TL_TG1, 0);
  DK_TLW(TRANS ? TL_TG2W : TL_TG1W, 0);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  __shared__ __align__(8) unsigned long long bars[KW][KS];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  unsigned char* wbuf = smem_raw + (size_t)wl * KS * kPTileBytes;
  // g.nw <= nt warps hold the tiles, every one of them at least one
  const long long Wn = g.nw;
  const long long w = (long long)blockIdx.x * KW + wl;
  const long long t0 = w < Wn ? w * g.nt / Wn : g.nt, t1 = w < Wn ? (w + 1) * g.nt / Wn : g.nt;
  // W is re-read by both passes of every iteration: kept L2-resident across the basis sweeps
  // (evict-first) in between by the persisting window of the launch, else by evict-last
  const unsigned long long pol = g.win_bytes ? l2_evict_unchanged() : l2_evict_last();
  auto tile_ptr = [&](long long t) {
    const long long q = TRANS ? (long long)__ldg(g.tid + t) : t;
    return g.T + q * (kPT * kPT);
  };
  if (lane == 0)
    for (int s = 0; s < KS; ++s) mbar_init1(&bars[wl][s]);
  mbar_init_fence();
  __syncwarp();
  // The tiles and their metadata are set-up constants: fetched before the dependency wait,
  // so they stream in while the producer of x drains.  Lane k holds tile t0 + k's blocks.
  const int nfirst = t1 - t0 < KS ? (int)(t1 - t0) : KS;
  const int my_row = (t0 + lane < t1) ? g.trow[t0 + lane] : -1;
  const int my_col = (t0 + lane < t1) ? g.tcol[t0 + lane] : 0;
  if (lane == 0)
    for (int s = 0; s < nfirst; ++s)
      tg_issue(wbuf + s * kPTileBytes, tile_ptr(t0 + s), &bars[wl][s], pol);
  // each warp prefetches its slice of the next kernel's constant streams into L2
  if (g.npf > 0 && lane < g.npf) {
    const unsigned long long nwarp = (unsigned long long)gridDim.x * KW;
    const unsigned long long tot = g.pf_bytes[lane];
    const unsigned long long slice = ((tot + nwarp - 1) / nwarp + 127ull) & ~127ull;
    const unsigned long long o = slice * (unsigned long long)(blockIdx.x * KW + wl);
    if (o < tot) l2_prefetch(g.pf[lane] + o, (unsigned)(o + slice < tot ? slice : tot - o));
  }
  // the next grid may launch now (its griddepcontrol.wait still waits for this one)
  pdl_trigger();
  pdl_wait();
  DK_TL(TRANS ? TL_TG2 : TL_TG1, 1);
  DK_TLW(TRANS ? TL_TG2W : TL_TG1W, 1);
  const bool off = gate != nullptr && *gate == 0;
  if (FUSE_R && !off) {  // s~ first (every block), then the pass reads it as x
    tg_restrict(rm, s_out);
    tg_grid_barrier(g.bar);
  }
  if (off || t0 >= t1) {  // drain the copies already in flight, then leave
    for (int s = 0; s < nfirst; ++s) mbar_wait_parity(&bars[wl][s], 0);
    return;
  }
  double xr[kXPre];
#pragma unroll
  for (int k = 0; k < kXPre; ++k) {
    const int c = __shfl_sync(0xffffffffu, my_col, k);
    xr[k] = (t0 + k < t1) ? __ldcg(x + (long long)c * kPT + lane) : 0.0;
  }
  int R = __shfl_sync(0xffffffffu, my_row, 0);
  double racc = 0.0;
  double acc[TRANS ? 32 : 1];
#pragma unroll
  for (int c = 0; c < (TRANS ? 32 : 1); ++c) acc[c] = 0.0;
  for (long long t = t0; t < t1; ++t) {
    const int k = (int)(t - t0);
    const int s = k % KS;
    const unsigned parity = (unsigned)((k / KS) & 1);
    const int kn = k + 1;
    const int row_n = kn < 32 ? __shfl_sync(0xffffffffu, my_row, kn & 31)
                              : (t + 1 < t1 ? g.trow[t + 1] : -1);
    double xv = 0.0;
#pragma unroll
    for (int q = 0; q < kXPre; ++q)
      if (q == k) xv = xr[q];
    if (k >= kXPre) {
      const int c = k < 32 ? __shfl_sync(0xffffffffu, my_col, k & 31) : g.tcol[t];
      xv = __ldcg(x + (long long)c * kPT + lane);
    }
    mbar_wait_parity(&bars[wl][s], parity);
    const double2* T = reinterpret_cast<const double2*>(wbuf + s * kPTileBytes);
    if constexpr (TRANS) {
#pragma unroll
      for (int p = 0; p < 16; ++p) {
        const double2 a = T[p * kPT + lane];
        acc[2 * p] = fma(a.x, xv, acc[2 * p]);
        acc[2 * p + 1] = fma(a.y, xv, acc[2 * p + 1]);
      }
    } else {
#pragma unroll
      for (int p = 0; p < 16; ++p) {
        const double2 a = T[p * kPT + lane];
        racc = fma(a.x, __shfl_sync(0xffffffffu, xv, 2 * p), racc);
        racc = fma(a.y, __shfl_sync(0xffffffffu, xv, 2 * p + 1), racc);
      }
    }
    __syncwarp();
    if (lane == 0 && t + KS < t1)  // refill this stage
      tg_issue(wbuf + s * kPTileBytes, tile_ptr(t + KS), &bars[wl][s], pol);
    const int Rn = (t + 1 < t1) ? row_n : -1;
    if (Rn == R) continue;
    // output block R ends in this warp's range
    if constexpr (TRANS) {
      racc = butterfly_sum32(acc, lane);
#pragma unroll
      for (int c = 0; c < 32; ++c) acc[c] = 0.0;
    }
    const int np = g.rnp[R];
    double out = racc;
    bool write = true;
    if (np > 1 && w == g.rfirst[R]) DK_TLW(TRANS ? TL_TG2W : TL_TG1W, 2 + (np > 32 ? 1 : 0));
    if (np > 1) {
      // A block split across warps is finished by its first warp (whose range ends with it,
      // so the others' pieces, at the starts of their ranges, are normally in by then).  The
      // pieces are self-validating: a slot holds the sentinel until its value lands, so no
      // fence or ticket is needed; the finisher re-arms the slots.  Sum in warp order.
      const int q = (int)(w - g.rfirst[R]);
      double* slots = g.part + (long long)g.rslot[R] * kPT + lane;
      if (NOSPIN) {
        slots[(long long)q * kPT] = racc;
        write = false;
      } else if (q != 0) {
        slots[(long long)q * kPT] = racc;
        write = false;
      } else {
        out = 0.0 + racc;
        // kFin slots in flight (the long block rows of the root separators are split over
        // tens of warps), then the in-order sum
        constexpr int kFin = TRANS ? 8 : 32;
        for (int k0 = 1; k0 < np; k0 += kFin) {
          double v[kFin];
#pragma unroll
          for (int i = 0; i < kFin; ++i)
            v[i] = k0 + i < np ? ld_volatile_f64(slots + (long long)(k0 + i) * kPT) : 0.0;
#pragma unroll
          for (int i = 0; i < kFin; ++i) {
            if (k0 + i >= np) break;
            double* sl = slots + (long long)(k0 + i) * kPT;
            while (is_sentinel(v[i])) {
              __nanosleep(32);
              v[i] = ld_volatile_f64(sl);
            }
            out += v[i];
            *sl = sentinel_f64();
          }
        }
      }
    }
    if (write) {
      const int row = R * kPT + lane;
      if (row < d) y[scatter ? scatter[row] : row] = out;
      if (np > 1) DK_TLW(TRANS ? TL_TG2W : TL_TG1W, 4 + (np > 32 ? 1 : 0));
    }
    racc = 0.0;
    R = Rn;
  }
  DK_TLW(TRANS ? TL_TG2W : TL_TG1W, 6);
  DK_TL(TRANS ? TL_TG2 : TL_TG1, 4);
}

}  // namespace

// ---- host: level-structure nested dissection -----------------------------------------
// George's automatic nested dissection: a BFS level structure from a pseudo-peripheral node
// (two sweeps), the separator = the vertices of the smallest level with 25-75 % of the nodes
// on either side that touch the next level, recursion on both sides (independent halves in
// parallel near the root), separator last.  Emits the order and the dissection tree.
namespace {

struct NDNode {
  int t0, s0, s1;       // subtree [t0, s1): descendants [t0, s0), separator [s0, s1)
  std::vector<int> kids;
};

struct NDPart {
  std::vector<int> order;
  std::vector<NDNode> nodes;  // post-order; the last is this part's root
};

struct NestedDissection {
  const std::vector<int>& ptr;
  const std::vector<int>& col;
  std::vector<int> part, level;
  std::atomic<int> next_id{2};
  int leaf;

  NestedDissection(int d, const std::vector<int>& p, const std::vector<int>& c, int lf)
      : ptr(p), col(c), part(d, 1), level(d, -1), leaf(lf) {}

  int deg(int v) const { return ptr[v + 1] - ptr[v]; }

  // BFS from src inside part pid (levels must be -1 on the part's nodes)
  void bfs(int src, int pid, std::vector<int>& seen) {
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

  // a leaf: every node in the separator, natural order
  static void leaf_node(std::vector<int>& nodes, int base, NDPart& out) {
    std::sort(nodes.begin(), nodes.end());
    out.order.insert(out.order.end(), nodes.begin(), nodes.end());
    out.nodes.push_back({base, base, base + (int)nodes.size(), {}});
  }

  // splice a child's nodes (renumbered) into out and register its root under `parent`
  static void append(NDPart& out, NDPart& sub, NDNode& parent) {
    const int off = (int)out.nodes.size();
    out.order.insert(out.order.end(), sub.order.begin(), sub.order.end());
    for (auto& nd : sub.nodes) {
      for (int& k : nd.kids) k += off;
      out.nodes.push_back(std::move(nd));
    }
    parent.kids.push_back((int)out.nodes.size() - 1);
  }

  // order `nodes` (all in part pid) into positions [base, base + n)
  NDPart rec(std::vector<int> nodes, int pid, int base, int depth) {
    NDPart out;
    const int n = (int)nodes.size();
    if (n <= leaf) {
      for (int v : nodes) part[v] = 0;
      leaf_node(nodes, base, out);
      return out;
    }
    for (int v : nodes) level[v] = -1;
    int src = nodes[0];
    for (int v : nodes)
      if (deg(v) < deg(src)) src = v;
    std::vector<int> seen;
    bfs(src, pid, seen);
    if ((int)seen.size() < n) {
      // several components: each is a child, no separator
      std::vector<std::vector<int>> comps;
      comps.push_back(seen);
      for (int v : nodes)
        if (level[v] < 0) {
          bfs(v, pid, seen);
          comps.push_back(seen);
        }
      std::vector<int> ids;
      for (auto& c : comps) {
        const int id = next_id++;
        ids.push_back(id);
        for (int v : c) part[v] = id;
      }
      NDNode root{base, base + n, base + n, {}};
      int b = base;
      for (size_t i = 0; i < comps.size(); ++i) {
        const int sz = (int)comps[i].size();
        NDPart sub = rec(std::move(comps[i]), ids[i], b, depth + 1);
        append(out, sub, root);
        b += sz;
      }
      out.nodes.push_back(std::move(root));
      return out;
    }
    // second sweep from a minimum-degree node of the last level
    {
      const int e = level[seen.back()];
      int best = -1;
      for (int i = (int)seen.size() - 1; i >= 0 && level[seen[i]] == e; --i)
        if (best < 0 || deg(seen[i]) < deg(best)) best = seen[i];
      for (int v : seen) level[v] = -1;
      bfs(best, pid, seen);
    }
    const int nl = level[seen.back()] + 1;
    std::vector<long long> cnt(nl, 0), cum(nl, 0);
    for (int v : seen) ++cnt[level[v]];
    for (int l = 0; l < nl; ++l) cum[l] = cnt[l] + (l ? cum[l - 1] : 0);
    int L = -1;
    for (int l = 1; l + 1 < nl; ++l)
      if (4 * cum[l - 1] >= n && 4 * cum[l] <= 3LL * n && (L < 0 || cnt[l] < cnt[L])) L = l;
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
    if (A.empty() || B.empty()) {  // no useful split: one dense node
      for (int v : nodes) part[v] = 0;
      leaf_node(nodes, base, out);
      return out;
    }
    const int ida = next_id++, idb = next_id++;
    for (int v : A) part[v] = ida;
    for (int v : B) part[v] = idb;
    for (int v : sep) part[v] = 0;
    const int na = (int)A.size(), nb = (int)B.size();
    NDPart pa, pb;
    if (depth < 4 && n > 2048) {  // independent halves, disjoint nodes: in parallel
      auto fa = std::async(std::launch::async,
                           [&] { return rec(std::move(A), ida, base, depth + 1); });
      pb = rec(std::move(B), idb, base + na, depth + 1);
      pa = fa.get();
    } else {
      pa = rec(std::move(A), ida, base, depth + 1);
      pb = rec(std::move(B), idb, base + na, depth + 1);
    }
    NDNode root{base, base + na + nb, base + n, {}};
    append(out, pa, root);
    append(out, pb, root);
    out.order.insert(out.order.end(), sep.begin(), sep.end());
    out.nodes.push_back(std::move(root));
    return out;
  }
};

}  // namespace

void nd_order(int d, const std::vector<int>& ptr, const std::vector<int>& col,
              std::vector<int>& perm, std::vector<NDTreeNode>* tree) {
  NestedDissection nd(d, ptr, col, 64);
  std::vector<int> all(d);
  for (int i = 0; i < d; ++i) all[i] = i;
  NDPart p = nd.rec(std::move(all), 1, 0, 0);
  perm.swap(p.order);
  if (tree) {
    tree->clear();
    for (auto& n : p.nodes) tree->push_back({n.t0, n.s0, n.s1, n.kids});
  }
}

long long nd_profile_tiles(int d, const std::vector<int>& ptr, const std::vector<int>& col,
                           const std::vector<int>& perm) {
  // the row profile f of E~ closed under W = L^-1: g(i) = min(f(i), min_{f(i)<=k<i} g(k))
  // (range minimum by a segment tree), counted in 32 x 32 tiles
  std::vector<int> inv(d), f(d);
  for (int i = 0; i < d; ++i) inv[perm[i]] = i;
  for (int i = 0; i < d; ++i) f[i] = i;
  for (int v = 0; v < d; ++v)
    for (int k = ptr[v]; k < ptr[v + 1]; ++k) f[inv[v]] = std::min(f[inv[v]], inv[col[k]]);
  int sz = 1;
  while (sz < d) sz <<= 1;
  std::vector<int> seg(2 * sz, 1 << 30);
  auto query = [&](int lo, int hi) {  // min over [lo, hi)
    int m = 1 << 30;
    for (lo += sz, hi += sz; lo < hi; lo >>= 1, hi >>= 1) {
      if (lo & 1) m = std::min(m, seg[lo++]);
      if (hi & 1) m = std::min(m, seg[--hi]);
    }
    return m;
  };
  const int nb = (d + kPT - 1) / kPT;
  std::vector<int> gb(nb, 1 << 30);
  for (int i = 0; i < d; ++i) {
    const int g = f[i] < i ? std::min(f[i], query(f[i], i)) : f[i];
    for (int p = i + sz; p >= 1; p >>= 1) seg[p] = std::min(seg[p], g);
    gb[i / kPT] = std::min(gb[i / kPT], g / kPT);
  }
  long long tiles = 0;
  for (int I = 0; I < nb; ++I) tiles += I - gb[I] + 1;
  return tiles;
}

int coarse_pattern(const double* E, int d, int ld, std::vector<int>& ptr, std::vector<int>& col,
                   cudaStream_t s) {
  int* dcnt = nullptr;
  int* dptr = nullptr;
  int* dcol = nullptr;
  cudaMallocAsync(&dcnt, (size_t)d * sizeof(int), s);
  k_row_nnz<<<num_sms() * 4, 256, 0, s>>>(E, d, ld, dcnt);
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
  k_row_cols<<<num_sms() * 4, 256, 0, s>>>(E, d, ld, dptr, dcol);
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
  k_permute_sym<<<num_sms() * 8, 256, 0, s>>>(E, d, ld, perm, out);
}

void launch_unpermute_sym(const double* X, int d, int ld, const int* perm, double* out, int ldo,
                          cudaStream_t s) {
  k_unpermute_sym<<<num_sms() * 8, 256, 0, s>>>(X, d, ld, perm, out, ldo);
}

int tgemv_warps_per_cta();
int tg_grid();

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
  const long long Wn = std::min<long long>((long long)tg_grid() * tgemv_warps_per_cta(), nt);
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
  h.split_rows.clear();
  for (int R = 0; R < nrows; ++R)
    if (h.rnp[R] > 1) h.split_rows.push_back(R);
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
  k_tile_nz<<<num_sms() * 8, 256, 0, s>>>(W, d, ld, dti, dtj, nc, dfl);
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
  std::vector<int> bi(ai.size()), bj(ai.size()), bt(ai.size());
  for (size_t k = 0; k < idx.size(); ++k) {
    bi[k] = aj[idx[k]];  // output block of W^T
    bj[k] = ai[idx[k]];  // input block
    bt[k] = (int)idx[k];  // the tile in pass 1's storage
  }
  if (build_stream(ai, aj, nb, p1) || build_stream(bi, bj, nb, p2)) return -1;
  p2.tid = std::move(bt);
  return 0;
}

int upload_stream(const double* W, int d, int ld, bool pack, const TileGemvHost& h, TileGemv& g,
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
  int* tid = nullptr;
  if (!h.tid.empty()) up(&tid, h.tid);
  g.tid = tid;
  g.trans = !h.tid.empty();
  int* srows = nullptr;
  if (!h.split_rows.empty()) up(&srows, h.split_rows);
  g.split_rows = srows;
  g.nsplit = (int)h.split_rows.size();
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
  if (e == cudaSuccess)  // every slot starts as the sentinel (all bits set)
    e = cudaMemsetAsync(g.part, 0xff, (size_t)h.nslots * kPT * sizeof(double), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&g.bar, 2 * sizeof(unsigned), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(g.bar, 0, 2 * sizeof(unsigned), s);
  if (e != cudaSuccess) return (int)e;
  // the tile stream itself (big_alloc'd by the caller into g.T)
  if (pack)
    k_tile_pack<<<num_sms() * 8, 256, 0, s>>>(W, d, ld, trow, tcol, h.nt, 0,
                                              const_cast<double*>(g.T));
  return (int)cudaGetLastError();
}

void free_stream(TileGemv& g, cudaStream_t s) {
  void* bufs[] = {(void*)g.trow, (void*)g.tcol, (void*)g.rfirst, (void*)g.rslot, (void*)g.rnp,
                  (void*)g.part, (void*)g.tid, (void*)g.split_rows, (void*)g.bar};
  for (void* p : bufs)
    if (p) cudaFreeAsync(p, s);
  g.trow = g.tcol = g.rfirst = g.rslot = g.rnp = g.tid = g.split_rows = nullptr;
  g.bar = nullptr;
  g.nsplit = 0;
  g.part = nullptr;
}

// (warps per CTA, stages per warp) of k_tgemv; DK_TG_CFG picks one (set-up and launch agree)
static const int kTgCfg[][2] = {{12, 2}, {16, 1}, {8, 3}, {4, 6}, {8, 2}, {6, 2}, {4, 3}, {4, 2}};
int tgemv_cfg() {
  static int c = -1;
  if (c < 0) {
    const char* e = getenv("DK_TG_CFG");
    c = e ? atoi(e) : 2;
    if (c < 0 || c > 7) c = 2;
  }
  return c;
}
int tgemv_warps_per_cta() { return kTgCfg[tgemv_cfg()][0]; }

// SMs of the current device (the tile streams are split over tg_grid() CTAs)
int tg_grid() { return num_sms(); }

// the split blocks of a NOSPIN pass: one warp per block, pieces summed in warp order (the
// finisher's arithmetic), slots re-armed
__global__ void __launch_bounds__(256) k_tg_finish(TileGemv g, double* __restrict__ y,
                                                   const int* __restrict__ scatter, int d,
                                                   const int* __restrict__ gate) {
  pdl_wait();
  if (gate != nullptr && *gate == 0) return;
  const int lane = threadIdx.x & 31;
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (k >= g.nsplit) return;
  const int R = g.split_rows[k];
  const int np = g.rnp[R];
  double* slots = g.part + (long long)g.rslot[R] * kPT + lane;
  double out = 0.0 + slots[0];
  slots[0] = sentinel_f64();
  for (int q = 1; q < np; ++q) {
    out += slots[(long long)q * kPT];
    slots[(long long)q * kPT] = sentinel_f64();
  }
  const int row = R * kPT + lane;
  if (row < d) y[scatter ? scatter[row] : row] = out;
}

// the whole grid (one CTA per SM at this shared-memory size) must be co-resident for the
// finisher warps' waits; otherwise, or with DK_NO_SPIN, the NOSPIN pass + k_tg_finish
template <int KW, int KS, bool TRANS>
static bool tg_spin_ok(unsigned grid, size_t smem) {
  static int per_sm[kMaxDevices];
  static bool init[kMaxDevices];
  static const bool env = getenv("DK_NO_SPIN") != nullptr;
  if (env) return false;
  const int dev = current_device();
  if (!init[dev]) {
    int b = 0;
    // the occupancy query needs the shared-memory opt-in first (0 blocks otherwise)
    if (smem_optin((const void*)k_tgemv<KW, KS, TRANS, false>, smem) != 0 ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_tgemv<KW, KS, TRANS, false>, KW * 32,
                                                      smem) != cudaSuccess) {
      cudaGetLastError();
      b = 0;
    }
    per_sm[dev] = b;
    init[dev] = true;
  }
  return (long long)per_sm[dev] * num_sms() >= (long long)grid;
}

template <int KW, int KS, bool TRANS>
static void launch_tg_t(const TileGemv& g, const double* x, double* y, const int* scatter, int d,
                        const int* gate, cudaStream_t s, unsigned grid, size_t smem,
                        const cudaAccessPolicyWindow* win) {
  const bool spin = tg_spin_ok<KW, KS, TRANS>(grid, smem);
  if (win) access_window_next() = win;
  if (spin) {
    smem_optin((const void*)k_tgemv<KW, KS, TRANS, false>, smem);
    if (!getenv("DK_NO_COOP")) coop_next() = true;  // finishers wait on other blocks
    launch_pdl(k_tgemv<KW, KS, TRANS, false>, dim3(grid), dim3(KW * 32), smem, s, g, x, y,
               scatter, d, gate, RunMap{}, (double*)nullptr);
    return;
  }
  smem_optin((const void*)k_tgemv<KW, KS, TRANS, true>, smem);
  launch_pdl(k_tgemv<KW, KS, TRANS, true>, dim3(grid), dim3(KW * 32), smem, s, g, x, y, scatter,
             d, gate, RunMap{}, (double*)nullptr);
  if (g.nsplit > 0)
    launch_pdl(k_tg_finish, dim3((unsigned)((g.nsplit * 32 + 255) / 256)), dim3(256), 0, s, g, y,
               scatter, d, gate);
}

template <int KW, int KS>
static void launch_tg(const TileGemv& g, const double* x, double* y, const int* scatter, int d,
                      const int* gate, cudaStream_t s) {
  const size_t smem = (size_t)KW * KS * kPTileBytes;
  const unsigned grid = (unsigned)((g.nw + KW - 1) / KW);
  cudaAccessPolicyWindow win{};
  if (g.win_bytes) {
    win.base_ptr = g.win_base;
    win.num_bytes = g.win_bytes;
    win.hitRatio = 1.0f;
    win.hitProp = cudaAccessPropertyPersisting;
    win.missProp = cudaAccessPropertyStreaming;
  }
  const cudaAccessPolicyWindow* wp = g.win_bytes ? &win : nullptr;
  if (g.trans)
    launch_tg_t<KW, KS, true>(g, x, y, scatter, d, gate, s, grid, smem, wp);
  else
    launch_tg_t<KW, KS, false>(g, x, y, scatter, d, gate, s, grid, smem, wp);
}

template <int KW, int KS>
static bool tg_fuse_ok(const TileGemv& g) {
  const size_t smem = (size_t)KW * KS * kPTileBytes;
  const unsigned grid = (unsigned)((g.nw + KW - 1) / KW);
  // opt-in (DK_FUSE_RESTRICT=1): measured 1.9 % slower at config 3 than the separate
  // column-sum kernel (148 blocks sum what 241 did, plus the barrier)
  static const bool no_fuse = getenv("DK_FUSE_RESTRICT") == nullptr;
  static const bool no_coop = getenv("DK_NO_COOP") != nullptr;
  return !(no_fuse || no_coop || g.bar == nullptr || g.trans || g.win_bytes ||
           !tg_spin_ok<KW, KS, false>(grid, smem));
}

template <int KW, int KS>
static int launch_tg_restrict(const TileGemv& g, const RunMap& rm, double* s_out, double* y,
                              int d, const int* gate, cudaStream_t s) {
  const size_t smem = (size_t)KW * KS * kPTileBytes;
  const unsigned grid = (unsigned)((g.nw + KW - 1) / KW);
  if (!tg_fuse_ok<KW, KS>(g)) {
    launch_restrict_final(rm, s_out, gate, s);
    launch_tgemv(g, s_out, y, nullptr, d, gate, s);
    return 1 + tgemv_launches(g);
  }
  smem_optin((const void*)k_tgemv<KW, KS, false, false, true>, smem);
  coop_next() = true;  // the in-kernel grid barrier and the finishers need every block resident
  launch_pdl(k_tgemv<KW, KS, false, false, true>, dim3(grid), dim3(KW * 32), smem, s, g,
             (const double*)s_out, y, (const int*)nullptr, d, gate, rm, s_out);
  return 1;
}

int tgemv_restrict_launches(const TileGemv& g) {
  bool f;
  switch (tgemv_cfg()) {
    case 0: f = tg_fuse_ok<12, 2>(g); break;
    case 1: f = tg_fuse_ok<16, 1>(g); break;
    case 3: f = tg_fuse_ok<4, 6>(g); break;
    case 4: f = tg_fuse_ok<8, 2>(g); break;
    case 5: f = tg_fuse_ok<6, 2>(g); break;
    case 6: f = tg_fuse_ok<4, 3>(g); break;
    case 7: f = tg_fuse_ok<4, 2>(g); break;
    default: f = tg_fuse_ok<8, 3>(g); break;
  }
  return f ? 1 : 1 + tgemv_launches(g);
}

int launch_tgemv_restrict(const TileGemv& g, const RunMap& rm, double* s_out, double* y,
                          int d, const int* gate, cudaStream_t s) {
  switch (tgemv_cfg()) {
    case 0: return launch_tg_restrict<12, 2>(g, rm, s_out, y, d, gate, s);
    case 1: return launch_tg_restrict<16, 1>(g, rm, s_out, y, d, gate, s);
    case 3: return launch_tg_restrict<4, 6>(g, rm, s_out, y, d, gate, s);
    case 4: return launch_tg_restrict<8, 2>(g, rm, s_out, y, d, gate, s);
    case 5: return launch_tg_restrict<6, 2>(g, rm, s_out, y, d, gate, s);
    case 6: return launch_tg_restrict<4, 3>(g, rm, s_out, y, d, gate, s);
    case 7: return launch_tg_restrict<4, 2>(g, rm, s_out, y, d, gate, s);
    default: return launch_tg_restrict<8, 3>(g, rm, s_out, y, d, gate, s);
  }
}

// kernels one launch_tgemv issues: 1 (spinning finisher) or 2 (NOSPIN pass + k_tg_finish)
template <int KW, int KS>
static int tg_launches_t(const TileGemv& g) {
  const size_t smem = (size_t)KW * KS * kPTileBytes;
  const unsigned grid = (unsigned)((g.nw + KW - 1) / KW);
  const bool spin = g.trans ? tg_spin_ok<KW, KS, true>(grid, smem)
                            : tg_spin_ok<KW, KS, false>(grid, smem);
  return spin || g.nsplit == 0 ? 1 : 2;
}
int tgemv_launches(const TileGemv& g) {
  switch (tgemv_cfg()) {
    case 0: return tg_launches_t<12, 2>(g);
    case 1: return tg_launches_t<16, 1>(g);
    case 3: return tg_launches_t<4, 6>(g);
    case 4: return tg_launches_t<8, 2>(g);
    case 5: return tg_launches_t<6, 2>(g);
    case 6: return tg_launches_t<4, 3>(g);
    case 7: return tg_launches_t<4, 2>(g);
    default: return tg_launches_t<8, 3>(g);
  }
}

void launch_tgemv(const TileGemv& g, const double* x, double* y, const int* scatter, int d,
                  const int* gate, cudaStream_t s) {
  switch (tgemv_cfg()) {
    case 1: launch_tg<16, 1>(g, x, y, scatter, d, gate, s); break;
    case 3: launch_tg<4, 6>(g, x, y, scatter, d, gate, s); break;
    case 4: launch_tg<8, 2>(g, x, y, scatter, d, gate, s); break;
    case 5: launch_tg<6, 2>(g, x, y, scatter, d, gate, s); break;
    case 6: launch_tg<4, 3>(g, x, y, scatter, d, gate, s); break;
    case 7: launch_tg<4, 2>(g, x, y, scatter, d, gate, s); break;
    case 0: launch_tg<12, 2>(g, x, y, scatter, d, gate, s); break;
    default: launch_tg<8, 3>(g, x, y, scatter, d, gate, s); break;
  }
}

DK_TL_SETTER(tl_set_profile)

}  // namespace dk
