// dk_kernels.cu — streaming sm_100a kernels of one deflated-GMRES iteration.
//
// Per inner iteration j (deflated), DESIGN.md §4:
//   K1 k_stencil        w = A M^-1 v_j (DIA, Jacobi fused) + per-run sums of w  (Z^T w, part 1)
//   K2 k_restrict_final s = Z^T w from the run partials, fixed order             (part 2)
//   K3 k_symv / k_gemv  y = E^-1 s (packed symmetric / dense)           (dk_coarse.cu)
//   K4 k_project        w -= A Z y (compact prolongation), h = V^T w, ||w||; last block: H
//                       column, re-orthogonalisation test corr = h - G h
//   K5 k_gs             u = w - V h, ||u||; last block: Givens update, convergence test
//   K6 k_project<REDOTS> + k_gs<reorth>: corr = V^T u, u -= V corr (only when the test fired)
//   dense bases (RDGMRES): k_zdots (s = Z^T w, y = E^-1 s) and k_project<DK_DENSE>
// Reference semantics: _run_cycles, krylov.py:107-236.
#include <cuda_runtime.h>

#include <climits>
#include <cstdlib>

#include "dk_launch.h"

namespace dk {

// ======================================================================================
// Segmented (run-wise) restriction of one kTile tile held in shared memory.
// A run is a maximal range of equal labels in linear cell order; every tile start is a
// run head.  Each run's sum is written to out[slot[run index within the tile]].  The summation
// order is fixed (serial within a thread, fixed Hillis-Steele tree across threads), so the
// result is bitwise deterministic.
// ======================================================================================
// shared-memory index of tile cell c: one pad slot per 8 cells, so the 8-contiguous-cell
// reads of the scan below are 2-way instead of 16-way bank conflicted
__device__ __forceinline__ int pidx(int c) { return c + (c >> 3); }
constexpr int kTilePad = kTile + kTile / 8;

// RING: called by one 256-thread compute group of a larger block (threads [256 g, 256 g + 256),
// named barrier 1 + g) with the tile's slot list in shared memory; otherwise by a whole
// 256-thread block, slots in global
template <bool RING>
__device__ __forceinline__ void tile_sync() {
  if (RING) asm volatile("bar.sync %0, 256;" ::"r"(1 + (int)(threadIdx.x >> 8)) : "memory");
  else __syncthreads();
}
// thread index within the tile's 256 threads, and the compute group
template <bool RING>
__device__ __forceinline__ int tile_tid() {
  return RING ? (int)(threadIdx.x & 255) : (int)threadIdx.x;
}
template <bool RING>
__device__ __forceinline__ int tile_grp() {
  return RING ? (int)(threadIdx.x >> 8) : 0;
}
constexpr int kRingGroupsMax = 2;

template <bool RING, class SlotFn>
__device__ __forceinline__ void tile_restrict(const double* sw, const int* sl, double* out,
                                              SlotFn slot) {
  __shared__ int wf_[(RING ? kRingGroupsMax : 1) * kWarps];
  __shared__ double ws_[(RING ? kRingGroupsMax : 1) * kWarps];
  __shared__ int wc_[(RING ? kRingGroupsMax : 1) * kWarps];
  int* wf = wf_ + tile_grp<RING>() * kWarps;
  double* ws = ws_ + tile_grp<RING>() * kWarps;
  int* wc = wc_ + tile_grp<RING>() * kWarps;
  const int t = tile_tid<RING>(), lane = t & 31, warp = t >> 5;
  const int c0 = 8 * t;
  double val[8];
  int lb[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    val[e] = sw[9 * t + e];
    lb[e] = sl[9 * t + e];
  }
  const int prev = (c0 == 0) ? INT_MIN : sl[pidx(c0 - 1)];
  const int next = (c0 + 8 < kTile) ? sl[pidx(c0 + 8)] : INT_MIN;
  unsigned heads = 0;
  int nh = 0;
  double tail = 0.0;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int p = e ? lb[e - 1] : prev;
    if (c0 + e == 0 || lb[e] != p) {
      heads |= 1u << e;
      ++nh;
      tail = 0.0;
    }
    tail = __dadd_rn(tail, val[e]);
  }
  // warp inclusive segmented scan of (flag, sum) and plain scan of head counts
  int f = nh > 0;
  double s = tail;
  int c = nh;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int fu = __shfl_up_sync(0xffffffffu, f, d);
    const double su = __shfl_up_sync(0xffffffffu, s, d);
    const int cu = __shfl_up_sync(0xffffffffu, c, d);
    if (lane >= d) {
      if (!f) s = __dadd_rn(su, s);
      f = f | fu;
      c += cu;
    }
  }
  if (lane == 31) {
    wf[warp] = f;
    ws[warp] = s;
    wc[warp] = c;
  }
  int fe = __shfl_up_sync(0xffffffffu, f, 1);
  double se = __shfl_up_sync(0xffffffffu, s, 1);
  int ce = __shfl_up_sync(0xffffffffu, c, 1);
  if (lane == 0) {
    fe = 0;
    se = 0.0;
    ce = 0;
  }
  tile_sync<RING>();
  double ps = 0.0;
  int pc = 0;
  for (int w = 0; w < warp; ++w) {
    ps = wf[w] ? ws[w] : __dadd_rn(ps, ws[w]);
    pc += wc[w];
  }
  double run = fe ? se : __dadd_rn(ps, se);
  int ridx = pc + ce - 1;
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    if (heads & (1u << e)) {
      run = 0.0;
      ++ridx;
    }
    run = __dadd_rn(run, val[e]);
    const bool is_tail = (e < 7) ? ((heads >> (e + 1)) & 1u) != 0
                                 : (c0 + 8 >= kTile || next != lb[7]);
    if (is_tail) out[slot(ridx)] = run;
  }
}

// Run sums of a stencil tile's outputs rr (8 per thread: cells 2t + 512k, +1) with labels lb.
// slot(r): the slot of the tile's r-th run
template <bool RING, class SlotFn>
__device__ __forceinline__ void restrict_tail_runs(const double (&rr)[8], const int2 (&lb)[4],
                                                   double* sw, int* sl, double* wsum, int nruns,
                                                   SlotFn slot,
                                                   double* __restrict__ run_part) {
  // a tile inside one region is a single run: plain block sum instead of the segmented scan
  const bool one_run = nruns == 1;
  const int tl = tile_tid<RING>();
  double tsum = 0.0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if (one_run) {
      tsum = __dadd_rn(tsum, __dadd_rn(rr[2 * k], rr[2 * k + 1]));
    } else {
      const int p = pidx(2 * tl + 512 * k);
      sw[p] = rr[2 * k];
      sw[p + 1] = rr[2 * k + 1];
      sl[p] = lb[k].x;
      sl[p + 1] = lb[k].y;
    }
  }
  if (one_run) {
    tsum = warp_sum(tsum);
    if ((tl & 31) == 0) wsum[tl >> 5] = tsum;
    tile_sync<RING>();
    if (tl == 0) {
      double s = 0.0;
      for (int w = 0; w < kWarps; ++w) s = __dadd_rn(s, wsum[w]);
      run_part[slot(0)] = s;
    }
  } else {
    tile_sync<RING>();
    tile_restrict<RING>(sw, sl, run_part, slot);
  }
}

__device__ __forceinline__ void stencil_restrict_tail(const double (&rr)[8], const int2 (&lb)[4],
                                                      double* sw, int* sl, double* wsum,
                                                      const int* __restrict__ tile_run_off,
                                                      const int* __restrict__ run_slot,
                                                      double* __restrict__ run_part,
                                                      int tile) {
  const int r0 = tile_run_off[tile];
  const int* rs = run_slot + r0;
  restrict_tail_runs<false>(rr, lb, sw, sl, wsum, tile_run_off[tile + 1] - r0,
                            [rs](int r) { return __ldg(rs + r); }, run_part);
}

// Early start of an iteration's stencil (wait != nullptr): the grid is launched while k_gs of
// the previous iteration finishes its reduction and Givens update.  It starts once all groups
// of k_gs's norm reduction are in (post counter == ng) and forms sigma itself from the group
// partials (the same arithmetic as k_gs's last block), instead of waiting for the whole grid;
// it waits for that completion (griddepcontrol.wait) only before it exits, so every later
// kernel still sees k_gs's control state.  A gate already closed means the previous k_gs did not run (it
// would have posted otherwise): skip.  Returns false when the block skips.
__device__ __forceinline__ bool early_start(const unsigned* wait, const int* gate,
                                            unsigned need) {
  __shared__ int s_go;
  if (threadIdx.x == 0) {
    int go = gate == nullptr || *reinterpret_cast<const volatile int*>(gate) != 0;
    if (go) {
      while (ld_flag(wait) < need) __nanosleep(64);
      __threadfence();
    }
    s_go = go;
  }
  __syncthreads();
  if (!s_go) pdl_wait();
  return s_go != 0;
}

// sigma = 1 / ||u|| from k_gs's group partials: one thread forms it (k_gs's last-block
// arithmetic), the block shares it
__device__ __forceinline__ double early_sigma(const double* gsig, int ng) {
  __shared__ double s_sig;
  if (threadIdx.x == 0) s_sig = 1.0 / sqrt(grouped_total(gsig, 0, ng));
  __syncthreads();
  return s_sig;
}

// ======================================================================================
// K1: DIA stencil with fused scale / Jacobi / residual, optional run restriction.
// Row sums are accumulated in ascending-offset (= CSR column) order with separately
// rounded multiply and add, i.e. exactly scipy's csr_matvec arithmetic (sparse.py:106).
// ======================================================================================
template <int MODE, bool PRE, bool RESTRICT, bool WRITE>
__global__ void __launch_bounds__(kThreads) k_stencil(Dia A, const double* __restrict__ v,
                                                      const double* __restrict__ scale,
                                                      const double* __restrict__ b,
                                                      double* __restrict__ out,
                                                      const int* __restrict__ lab,
                                                      const int* __restrict__ tile_run_off,
                                                      const int* __restrict__ run_slot,
                                                      double* __restrict__ run_part,
                                                      const int* __restrict__ gate,
                                                      const unsigned* wait, const double* gsig,
                                                      int ng) {
  if (wait != nullptr) {
    if (!early_start(wait, gate, (unsigned)ng)) return;
  } else {
    pdl_wait();
    if (gate != nullptr && *gate == 0) return;
  }
  __shared__ double sw[RESTRICT ? kTilePad : 2];
  __shared__ int sl[RESTRICT ? kTilePad : 2];
  __shared__ double wsum[kWarps];
  // ST_APPLY: the scaled, Jacobi-preconditioned input p = (sigma v) M^-1 of the tile and a
  // +-kHalo halo is staged in shared memory once; the in-plane neighbours (|offset| <= kHalo:
  // +-1, +-nx) read it there, the z-plane neighbours straight from L2
  constexpr int kHalo = 128;
  constexpr bool STAGE = (MODE == ST_APPLY);
  __shared__ __align__(16) double sp[STAGE ? kTile + 2 * kHalo : 2];
  const long long base = (long long)blockIdx.x * kTile;
  const bool has_scale = (MODE == ST_APPLY) && scale != nullptr;
  const double sc = !has_scale ? 1.0 : wait != nullptr ? early_sigma(gsig, ng) : __ldcg(scale);
  if (STAGE) {
    for (int e = threadIdx.x; e < (kTile + 2 * kHalo) / 2; e += kThreads) {
      const long long i = base - kHalo + 2 * e;
      double2 x = ld2(v + i);
      if (has_scale) {
        x.x = __dmul_rn(x.x, sc);
        x.y = __dmul_rn(x.y, sc);
      }
      if (PRE) {
        const double2 m = ld2(A.inv + i);
        x.x = __dmul_rn(x.x, m.x);
        x.y = __dmul_rn(x.y, m.y);
      }
      reinterpret_cast<double2*>(sp)[e] = x;
    }
    __syncthreads();
  }
  double rr[8];
  int2 lb[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int loc = 2 * threadIdx.x + 512 * k;
    const long long i = base + loc;
    double r0 = 0.0, r1 = 0.0;
    if (MODE == ST_IDENT) {
      const double2 x = ld2(v + i);
      r0 = x.x;
      r1 = x.y;
    } else {
#pragma unroll
      for (int q = 0; q < kMaxDiag; ++q) {
        if (q < A.ndiag) {
          const long long o = A.off[q];
          const double2 a = (A.csh[q] & 1)
                                ? make_double2(dia_coef(A, q, i), dia_coef(A, q, i + 1))
                                : ld2(A.co[q] + i + A.csh[q]);
          if (STAGE && o >= -kHalo && o <= kHalo) {
            const double* pp = sp + kHalo + loc + o;
            r0 = __dadd_rn(r0, __dmul_rn(a.x, pp[0]));
            r1 = __dadd_rn(r1, __dmul_rn(a.y, pp[1]));
            continue;
          }
          double x0, x1, m0 = 1.0, m1 = 1.0;
          if ((o & 1) == 0) {  // even offset: aligned 16 B loads of the neighbour pair
            const double2 xv = ld2(v + i + o);
            x0 = xv.x;
            x1 = xv.y;
            if (PRE) {
              const double2 mv = ld2(A.inv + i + o);
              m0 = mv.x;
              m1 = mv.y;
            }
          } else {
            x0 = __ldg(v + i + o);
            x1 = __ldg(v + i + o + 1);
            if (PRE) {
              m0 = __ldg(A.inv + i + o);
              m1 = __ldg(A.inv + i + o + 1);
            }
          }
          if (has_scale) {
            x0 = __dmul_rn(x0, sc);
            x1 = __dmul_rn(x1, sc);
          }
          if (PRE) {
            x0 = __dmul_rn(x0, m0);
            x1 = __dmul_rn(x1, m1);
          }
          r0 = __dadd_rn(r0, __dmul_rn(a.x, x0));
          r1 = __dadd_rn(r1, __dmul_rn(a.y, x1));
        }
      }
      if (MODE == ST_RESID) {
        const double2 bb = ld2(b + i);
        r0 = __dsub_rn(bb.x, r0);
        r1 = __dsub_rn(bb.y, r1);
      }
    }
    if (WRITE) st2(out + i, make_double2(r0, r1));
    rr[2 * k] = r0;
    rr[2 * k + 1] = r1;
    if (RESTRICT) lb[k] = *reinterpret_cast<const int2*>(lab + i);
  }
  if (RESTRICT) stencil_restrict_tail(rr, lb, sw, sl, wsum, tile_run_off, run_slot, run_part, blockIdx.x);
  if (wait != nullptr) pdl_wait();
}

// K1 for the symmetric 7-point operator (TPFA; DIA offsets -nxny, -nx, -1, 0, 1, nx, nxny,
// arrays c0, u1, ux, uz for the centre and the positive diagonals, nx and nxny even): the
// same arithmetic as k_stencil<ST_APPLY> (same products, same ascending-offset order), with
// every global load of a pair of cells known up front (no runtime offset branches): the
// tile's input p = (sigma v) M^-1 is staged in shared memory (halo H >= nx + 2), then each
// pair's eleven 16 B loads are issued together.  64 registers: four blocks per SM (measured
// against two pairs in flight at two blocks per SM: +0.8 %).
struct Sym7Pair {
  double2 c, u1, u1m, ux, uxm, uz, uzm, vm, vp, im, ip;
};

template <bool PRE>
__device__ __forceinline__ void sym7_load(Sym7Pair& q, const Dia& A, const double* __restrict__ v,
                                          long long i, long long nx, long long nz,
                                          unsigned long long pol) {
  q.c = ld2_stream(A.co[3] + i, pol);
  q.u1 = ld2_stream(A.co[4] + i, pol);
  q.u1m = ld2_stream(A.co[4] + i - 2, pol);
  q.ux = ld2_stream(A.co[5] + i, pol);
  q.uxm = ld2_stream(A.co[5] + i - nx, pol);
  q.uz = ld2_stream(A.co[6] + i, pol);
  q.uzm = ld2_stream(A.co[6] + i - nz, pol);
  q.vm = ld2_vec(v + i - nz);
  q.vp = ld2_vec(v + i + nz);
  if (PRE) {
    q.im = ld2_stream(A.inv + i - nz, pol);
    q.ip = ld2_stream(A.inv + i + nz, pol);
  }
}

__device__ __forceinline__ double sym7_x(double x, double sc, bool has_scale, bool pre, double m) {
  if (has_scale) x = __dmul_rn(x, sc);
  if (pre) x = __dmul_rn(x, m);
  return x;
}

template <bool PRE>
__device__ __forceinline__ double2 sym7_apply(const Sym7Pair& q, const double* pp, long long nx,
                                              double sc, bool has_scale) {
  // pp = staged p at cell i;  cell i: coefficients uzm.x uxm.x u1m.y c.x u1.x ux.x uz.x,
  // cell i+1: uzm.y uxm.y u1.x c.y u1.y ux.y uz.y
  const double zm0 = sym7_x(q.vm.x, sc, has_scale, PRE, PRE ? q.im.x : 1.0);
  const double zm1 = sym7_x(q.vm.y, sc, has_scale, PRE, PRE ? q.im.y : 1.0);
  const double zp0 = sym7_x(q.vp.x, sc, has_scale, PRE, PRE ? q.ip.x : 1.0);
  const double zp1 = sym7_x(q.vp.y, sc, has_scale, PRE, PRE ? q.ip.y : 1.0);
  double r0 = __dmul_rn(q.uzm.x, zm0);
  r0 = __dadd_rn(r0, __dmul_rn(q.uxm.x, pp[-nx]));
  r0 = __dadd_rn(r0, __dmul_rn(q.u1m.y, pp[-1]));
  r0 = __dadd_rn(r0, __dmul_rn(q.c.x, pp[0]));
  r0 = __dadd_rn(r0, __dmul_rn(q.u1.x, pp[1]));
  r0 = __dadd_rn(r0, __dmul_rn(q.ux.x, pp[nx]));
  r0 = __dadd_rn(r0, __dmul_rn(q.uz.x, zp0));
  double r1 = __dmul_rn(q.uzm.y, zm1);
  r1 = __dadd_rn(r1, __dmul_rn(q.uxm.y, pp[1 - nx]));
  r1 = __dadd_rn(r1, __dmul_rn(q.u1.x, pp[0]));
  r1 = __dadd_rn(r1, __dmul_rn(q.c.y, pp[1]));
  r1 = __dadd_rn(r1, __dmul_rn(q.u1.y, pp[2]));
  r1 = __dadd_rn(r1, __dmul_rn(q.ux.y, pp[1 + nx]));
  r1 = __dadd_rn(r1, __dmul_rn(q.uz.y, zp1));
  return make_double2(r0, r1);
}

template <bool PRE, bool RESTRICT, bool WRITE>
__global__ void __launch_bounds__(kThreads, 4) k_stencil_sym7(Dia A, const double* __restrict__ v,
                                                           const double* __restrict__ scale,
                                                           double* __restrict__ out,
                                                           const int* __restrict__ lab,
                                                           const int* __restrict__ tile_run_off,
                                                           const int* __restrict__ run_slot,
                                                           double* __restrict__ run_part,
                                                           const int* __restrict__ gate, int H,
                                                           const unsigned* wait,
                                                           const double* gsig, int ng) {
  DK_TL(TL_STENCIL, 0);
  if (wait != nullptr) {
    // the tile's operator diagonals, M^-1 and labels are final: into L2 while waiting
    const long long b0 = (long long)blockIdx.x * kTile;
    const int t = threadIdx.x;
    if (t < 4) l2_prefetch(A.co[3 + t] + b0, kTile * 8);
    if (PRE && t == 4) l2_prefetch(A.inv + b0, kTile * 8);
    if (RESTRICT && t == 5) l2_prefetch(lab + b0, kTile * 4);
    if (!early_start(wait, gate, (unsigned)ng)) return;
  } else {
    pdl_wait();
    if (gate != nullptr && *gate == 0) return;
  }
  DK_TL(TL_STENCIL, 1);
  pdl_trigger();  // the next grid launches while this one runs (it still waits for it)
  extern __shared__ __align__(16) double sp[];  // [H | kTile | H]
  __shared__ double sw[RESTRICT ? kTilePad : 2];
  __shared__ int sl[RESTRICT ? kTilePad : 2];
  __shared__ double wsum[kWarps];
  const long long base = (long long)blockIdx.x * kTile;
  const long long nx = A.off[5], nz = A.off[6];
  const bool has_scale = scale != nullptr;
  const double sc = !has_scale ? 1.0 : wait != nullptr ? early_sigma(gsig, ng) : __ldcg(scale);
  const unsigned long long pol = l2_evict_first();
  for (int e = threadIdx.x; e < (kTile + 2 * H) / 2; e += kThreads) {
    const long long i = base - H + 2 * e;
    double2 x = ld2_vec(v + i);
    if (has_scale) {
      x.x = __dmul_rn(x.x, sc);
      x.y = __dmul_rn(x.y, sc);
    }
    if (PRE) {
      const double2 m = ld2_stream(A.inv + i, pol);
      x.x = __dmul_rn(x.x, m.x);
      x.y = __dmul_rn(x.y, m.y);
    }
    reinterpret_cast<double2*>(sp)[e] = x;
  }
  int2 lb[4];
  if (RESTRICT)
#pragma unroll
    for (int k = 0; k < 4; ++k)
      lb[k] = ldi2_stream(lab + base + 2 * threadIdx.x + 512 * k, pol);
  __syncthreads();
  double rr[8];
  const double* pp = sp + H + 2 * threadIdx.x;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    Sym7Pair q;
    sym7_load<PRE>(q, A, v, base + 2 * threadIdx.x + 512 * k, nx, nz, pol);
    const double2 r = sym7_apply<PRE>(q, pp + 512 * k, nx, sc, has_scale);
    rr[2 * k] = r.x;
    rr[2 * k + 1] = r.y;
  }
  if (WRITE)
#pragma unroll
    for (int k = 0; k < 4; ++k)
      st2_vec(out + base + 2 * threadIdx.x + 512 * k, make_double2(rr[2 * k], rr[2 * k + 1]));
  if (RESTRICT)
    stencil_restrict_tail(rr, lb, sw, sl, wsum, tile_run_off, run_slot, run_part, blockIdx.x);
  DK_TL(TL_STENCIL, 3);
  if (wait != nullptr) pdl_wait();
  DK_TL(TL_STENCIL, 4);
}

// K1 as a persistent grid fed by a bulk-copy ring (one CTA per SM; opt-in, DK_RING=1): the same arithmetic and the same per-thread cell mapping as
// k_stencil_sym7 (bit-identical results), but every input of a 512-cell sub-tile — the four
// coefficient streams and their shifted re-reads, the z-planes of v and M^-1 above and below,
// the in-plane input with its halo — lands in one shared-memory stage through cp.async.bulk
// (one elected thread issues; an mbarrier per stage counts the bytes).  S stages keep
// S-1 sub-tiles (~47 KB each at nx <= 62) in flight per SM while the threads work on one and
// while a tile's restriction tail runs, so DRAM never waits for a dependent load round.
// Early start: the coefficient, M^-1 copies of the first stages are issued, and the later
// tiles' constants prefetched into L2, before the start flag; only v waits for it.
struct RingLayout {
  int c, u1, ux, uz, uzm, v, vm, vp, iv, im, ip, stage;  // offsets in doubles
};
constexpr int kSub = 512;       // cells per sub-tile (2 per thread)
constexpr int kRingMax = 8;     // stages (mbarriers)
__host__ __device__ inline RingLayout ring_layout(int H, bool pre) {
  RingLayout L;
  L.c = 0;
  L.u1 = L.c + kSub;
  L.ux = L.u1 + kSub + 2;
  L.uz = L.ux + kSub + H;
  L.uzm = L.uz + kSub;
  L.v = L.uzm + kSub;
  L.vm = L.v + kSub + 2 * H;
  L.vp = L.vm + kSub;
  L.iv = L.vp + kSub;
  L.im = L.iv + (pre ? kSub + 2 * H : 0);
  L.ip = L.im + (pre ? kSub : 0);
  L.stage = L.ip + (pre ? kSub : 0);
  return L;
}

constexpr int kSlotCap = kTile + 8;  // ints per slot-list buffer (aligned-down start + runs)
// NG compute groups of 8 warps (alternate tiles: one group's restriction tail overlaps the
// other's stencil phase) + the copy warp.  Each group has its own full / empty barrier per
// stage, so it sees every phase of the barriers it waits on (a group skipping the other
// group's phases could not follow a shared barrier's parity).
constexpr int ring_threads(int ng) { return ng * kThreads + 32; }
// dynamic shared memory ahead of the stages (bytes; a multiple of 16): the restriction's
// staging per group and NG + 1 tiles' slot lists
constexpr size_t ring_extra(int ng, bool restrict_) {
  return restrict_ ? (size_t)ng * kTilePad * 12 + (size_t)(ng + 1) * kSlotCap * 4 : 0;
}

__device__ __forceinline__ void mbar_init_n(unsigned long long* bar, unsigned n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(n));
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar))
               : "memory");
}

template <bool PRE, bool RESTRICT, bool WRITE, int NG>
__global__ void __launch_bounds__(ring_threads(NG), 1) k_stencil_sym7_ring(
    Dia A, const double* __restrict__ v, const double* __restrict__ scale,
    double* __restrict__ out, const int* __restrict__ lab, const int* __restrict__ tile_run_off,
    const int* __restrict__ run_slot, double* __restrict__ run_part,
    const int* __restrict__ gate, int H, int S, int ntiles, const unsigned* wait,
    const double* gsig, int ng, const char* __restrict__ pf, unsigned long long pf_bytes,
    int pf_early) {
  DK_TL(TL_STENCIL, 0);
  // dynamic shared memory: the restriction's staging (per group), NB tiles' slot lists,
  // then the S stages
  extern __shared__ __align__(16) double ring_smem[];
  __shared__ __align__(8) unsigned long long full[NG * kRingMax], empty[NG * kRingMax];
  constexpr int NB = NG + 1;  // slot-list buffers: tile j's is refilled for tile j + NB
  double* sw_ = ring_smem;
  int* sl_ = reinterpret_cast<int*>(sw_ + (RESTRICT ? NG * kTilePad : 0));
  int* sslot = sl_ + (RESTRICT ? NG * kTilePad : 0);
  double* ring = reinterpret_cast<double*>(sslot + (RESTRICT ? NB * kSlotCap : 0));
  __shared__ double wsum[NG * 2 * kWarps];  // by group and by the parity of its tile count
  __shared__ double s_sig;
  __shared__ int s_go;
  const int tid = threadIdx.x;
  const bool producer = tid >= NG * kThreads;
  const int grp = tid >> 8;  // compute group
  const int t = tid & 255;   // thread of the group (the cell mapping of k_stencil_sym7)
  double* sw = sw_ + (RESTRICT ? grp * kTilePad : 0);
  int* sl = sl_ + (RESTRICT ? grp * kTilePad : 0);
  const long long nx = A.off[5], nz = A.off[6];
  const RingLayout L = ring_layout(H, PRE);
  const int nmine = ((int)blockIdx.x < ntiles)
                        ? (ntiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x
                        : 0;
  const int nq = 4 * nmine;
  const int npro = nq < S ? nq : S;
  const bool has_scale = scale != nullptr;
  if (tid == 0) {
    for (int g = 0; g < NG; ++g)
      for (int s = 0; s < S; ++s) {
        mbar_init1(&full[g * kRingMax + s]);
        mbar_init_n(&empty[g * kRingMax + s], kWarps);
      }
    mbar_init_fence();
  }
  if (wait != nullptr) {
    if (tid == 0) s_go = gate == nullptr || *reinterpret_cast<const volatile int*>(gate) != 0;
    __syncthreads();
    if (!s_go) {  // the producer kernel did not run
      pdl_wait();
      return;
    }
  } else {
    pdl_wait();
    if (gate != nullptr && *gate == 0) return;
    __syncthreads();
  }
  if (producer) {
    // ---- copy warp: one lane issues every bulk copy of the block ----
    const int lane = tid - NG * kThreads;
    if (wait != nullptr && lane >= 1 && lane <= 6) {
      // later tiles' constants into L2 while the start flag is awaited
      for (int j = 1; j < nmine; ++j) {
        const long long b0 = ((long long)blockIdx.x + (long long)j * gridDim.x) * kTile;
        if (lane <= 4) l2_prefetch(A.co[2 + lane] + b0, kTile * 8);
        if (PRE && lane == 5) l2_prefetch(A.inv + b0, kTile * 8);
        if (RESTRICT && lane == 6) l2_prefetch(lab + b0, kTile * 4);
      }
    }
    if (lane != 0) return;
    const unsigned long long pol = l2_evict_first();
    const unsigned bytes_stage =
        8u * (unsigned)(kSub + (kSub + 2) + (kSub + nx) + 2 * kSub +
                        (PRE ? 3 * kSub + 2 * H : 0) + 3 * kSub + 2 * H);
    auto cell0 = [&](int q) {
      return ((long long)blockIdx.x + (long long)(q >> 2) * gridDim.x) * kTile + (q & 3) * kSub;
    };
    // run offsets of the tile whose first sub-tile is issued next (loaded one tile ahead)
    int r0 = 0, r1 = 0;
    if (RESTRICT && nmine > 0) {
      r0 = __ldg(tile_run_off + blockIdx.x);
      r1 = __ldg(tile_run_off + blockIdx.x + 1);
    }
    // final data (operator, M^-1, the tile's slot list): may precede the start flag
    auto issue_const = [&](int q) {
      const int s = q % S;
      double* st = ring + (size_t)s * L.stage;
      unsigned long long* bar = &full[((q >> 2) % NG) * kRingMax + s];
      const long long g = cell0(q);
      unsigned bytes = bytes_stage;
      unsigned sbytes = 0;
      int a0 = 0;
      if (RESTRICT && (q & 3) == 0) {
        a0 = r0 & ~3;
        sbytes = 4u * (unsigned)((r1 - a0 + 3) & ~3);
        bytes += sbytes;
      }
      mbar_arrive_expect(bar, bytes);
      if (RESTRICT && (q & 3) == 0) {
        bulk_g2s(sslot + ((q >> 2) % NB) * kSlotCap, run_slot + a0, sbytes, bar, pol);
        const int jn = (q >> 2) + 1;  // next tile's offsets for its own first sub-tile
        if (jn < nmine) {
          const long long tn = (long long)blockIdx.x + (long long)jn * gridDim.x;
          r0 = __ldg(tile_run_off + tn);
          r1 = __ldg(tile_run_off + tn + 1);
        }
      }
      bulk_g2s(st + L.c, A.co[3] + g, 8u * kSub, bar, pol);
      bulk_g2s(st + L.u1, A.co[4] + g - 2, 8u * (kSub + 2), bar, pol);
      bulk_g2s(st + L.ux, A.co[5] + g - nx, 8u * (unsigned)(kSub + nx), bar, pol);
      bulk_g2s(st + L.uz, A.co[6] + g, 8u * kSub, bar, pol);
      bulk_g2s(st + L.uzm, A.co[6] + g - nz, 8u * kSub, bar, pol);
      if (PRE) {
        bulk_g2s(st + L.iv, A.inv + g - H, 8u * (unsigned)(kSub + 2 * H), bar, pol);
        bulk_g2s(st + L.im, A.inv + g - nz, 8u * kSub, bar, pol);
        bulk_g2s(st + L.ip, A.inv + g + nz, 8u * kSub, bar, pol);
      }
    };
    // the iteration's input vector: after the start flag / the predecessor's completion
    auto issue_vec = [&](int q) {
      const int s = q % S;
      double* st = ring + (size_t)s * L.stage;
      unsigned long long* bar = &full[((q >> 2) % NG) * kRingMax + s];
      const long long g = cell0(q);
      bulk_g2s(st + L.v, v + g - H, 8u * (unsigned)(kSub + 2 * H), bar);
      bulk_g2s(st + L.vm, v + g - nz, 8u * kSub, bar);
      bulk_g2s(st + L.vp, v + g + nz, 8u * kSub, bar);
    };
    // L2 prefetch of the block's slice of the constant stream the coarse kernels read next
    // (the W tile store): the stencil leaves more than half of the DRAM bandwidth unused, so
    // one piece per issued stage rides along and the tile GEMV's first pass finds W in L2
    unsigned long long pf_off = 0, pf_end = 0;
    unsigned pf_piece = 0;
    if (pf != nullptr && nq > 0) {
      const unsigned long long slice =
          ((pf_bytes + gridDim.x - 1) / gridDim.x + 127ull) & ~127ull;
      pf_off = slice * blockIdx.x;
      pf_end = pf_off + slice < pf_bytes ? pf_off + slice : pf_bytes;
      pf_piece = (unsigned)(((slice + nq - 1) / nq + 127ull) & ~127ull);
    }
    auto issue_pf = [&]() {
      if (pf_off < pf_end) {
        const unsigned long long left = pf_end - pf_off;
        const unsigned len = left < pf_piece ? (unsigned)left : pf_piece;
        l2_prefetch(pf + pf_off, len);
        pf_off += len;
      }
    };
    unsigned epar[kRingGroupsMax] = {0u, 0u};  // per group: phase parity of each stage's empty
    for (int q = 0; q < npro; ++q) issue_const(q);
    for (int q = 0; q < pf_early && q < nq; ++q) issue_pf();
    if (wait != nullptr) {
      while (ld_flag(wait) < (unsigned)ng) __nanosleep(64);
      __threadfence();
      fence_async_global();
    }
    for (int q = 0; q < npro; ++q) issue_vec(q);
    for (int q = pf_early; q < npro; ++q) issue_pf();
    for (int q = npro; q < nq; ++q) {
      // stage q % S was last filled for sub-tile q - S: wait for its owner group's release
      // (the producer sees every phase of every empty barrier, in order)
      {
        const int s = q % S;
        const int go = ((q - S) >> 2) % NG;
        mbar_wait_parity(&empty[go * kRingMax + s], (epar[go] >> s) & 1u);
        epar[go] ^= 1u << s;
      }
      issue_const(q);
      issue_vec(q);
      if (q >= pf_early) issue_pf();
    }
    return;
  }
  // ---- compute warps ----
  double sc = 1.0;
  if (has_scale) {
    if (wait != nullptr) {
      // sigma from k_gs's group partials once they are all posted (early_sigma's arithmetic)
      if (tid == 0) {
        while (ld_flag(wait) < (unsigned)ng) __nanosleep(64);
        __threadfence();
        s_sig = 1.0 / sqrt(grouped_total(gsig, 0, ng));
      }
      asm volatile("bar.sync 3, %0;" ::"r"(NG * kThreads) : "memory");  // the compute threads
      sc = s_sig;
    } else {
      sc = __ldcg(scale);
    }
  }
  DK_TL(TL_STENCIL, 1);
  pdl_trigger();  // the next grid launches while this one runs (it still waits for it)
  const unsigned long long pol = l2_evict_first();
  const int lane = t & 31;
  unsigned fpar = 0u;  // phase parity of each stage's full barrier of this group
  for (int j = grp; j < nmine; j += NG) {
    const int tile = (int)blockIdx.x + j * (int)gridDim.x;
    const long long base = (long long)tile * kTile;
    int2 lb[4];
    int r0 = 0, r1 = 0;
    if (RESTRICT) {
#pragma unroll
      for (int k = 0; k < 4; ++k) lb[k] = ldi2_stream(lab + base + 2 * t + 512 * k, pol);
      r0 = __ldg(tile_run_off + tile);
      r1 = __ldg(tile_run_off + tile + 1);
    }
    double rr[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int q = 4 * j + k;
      const int s = q % S;
      double* st = ring + (size_t)s * L.stage;
      mbar_wait_parity(&full[grp * kRingMax + s], (fpar >> s) & 1u);
      fpar ^= 1u << s;
      // no block barrier inside a tile's four sub-tiles: p = (sigma v) M^-1 is formed on use
      // from the staged v and M^-1 (the same two roundings as the staged product)
      const double* sv = st + L.v + H + 2 * t;
      const double* si = st + L.iv + H + 2 * t;
      auto P2 = [&](int o) {  // p at cells i + o, i + o + 1 (o even)
        double2 x = *reinterpret_cast<const double2*>(sv + o);
        if (has_scale) {
          x.x = __dmul_rn(x.x, sc);
          x.y = __dmul_rn(x.y, sc);
        }
        if (PRE) {
          const double2 m = *reinterpret_cast<const double2*>(si + o);
          x.x = __dmul_rn(x.x, m.x);
          x.y = __dmul_rn(x.y, m.y);
        }
        return x;
      };
      const double2 pa = P2(-2), pb = P2(0), pc = P2(2), pd = P2(-(int)nx), pe = P2((int)nx);
      const double2 c = *reinterpret_cast<const double2*>(st + L.c + 2 * t);
      const double2 u1m = *reinterpret_cast<const double2*>(st + L.u1 + 2 * t);
      const double2 u1 = *reinterpret_cast<const double2*>(st + L.u1 + 2 * t + 2);
      const double2 uxm = *reinterpret_cast<const double2*>(st + L.ux + 2 * t);
      const double2 ux = *reinterpret_cast<const double2*>(st + L.ux + 2 * t + nx);
      const double2 uz = *reinterpret_cast<const double2*>(st + L.uz + 2 * t);
      const double2 uzm = *reinterpret_cast<const double2*>(st + L.uzm + 2 * t);
      double2 zm = *reinterpret_cast<const double2*>(st + L.vm + 2 * t);
      double2 zp = *reinterpret_cast<const double2*>(st + L.vp + 2 * t);
      if (has_scale) {
        zm.x = __dmul_rn(zm.x, sc);
        zm.y = __dmul_rn(zm.y, sc);
        zp.x = __dmul_rn(zp.x, sc);
        zp.y = __dmul_rn(zp.y, sc);
      }
      if (PRE) {
        const double2 im = *reinterpret_cast<const double2*>(st + L.im + 2 * t);
        const double2 ip = *reinterpret_cast<const double2*>(st + L.ip + 2 * t);
        zm.x = __dmul_rn(zm.x, im.x);
        zm.y = __dmul_rn(zm.y, im.y);
        zp.x = __dmul_rn(zp.x, ip.x);
        zp.y = __dmul_rn(zp.y, ip.y);
      }
      // sym7_apply's sums (ascending offsets): cell i, then cell i + 1
      double r0 = __dmul_rn(uzm.x, zm.x);
      r0 = __dadd_rn(r0, __dmul_rn(uxm.x, pd.x));
      r0 = __dadd_rn(r0, __dmul_rn(u1m.y, pa.y));
      r0 = __dadd_rn(r0, __dmul_rn(c.x, pb.x));
      r0 = __dadd_rn(r0, __dmul_rn(u1.x, pb.y));
      r0 = __dadd_rn(r0, __dmul_rn(ux.x, pe.x));
      r0 = __dadd_rn(r0, __dmul_rn(uz.x, zp.x));
      double r1 = __dmul_rn(uzm.y, zm.y);
      r1 = __dadd_rn(r1, __dmul_rn(uxm.y, pd.y));
      r1 = __dadd_rn(r1, __dmul_rn(u1.x, pb.x));
      r1 = __dadd_rn(r1, __dmul_rn(c.y, pb.y));
      r1 = __dadd_rn(r1, __dmul_rn(u1.y, pc.x));
      r1 = __dadd_rn(r1, __dmul_rn(ux.y, pe.y));
      r1 = __dadd_rn(r1, __dmul_rn(uz.y, zp.y));
      rr[2 * k] = r0;
      rr[2 * k + 1] = r1;
      // this warp is done with the stage: the copy warp may refill it once all eight are
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[grp * kRingMax + s]);
    }
    if (WRITE)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        st2_vec(out + base + 2 * t + 512 * k, make_double2(rr[2 * k], rr[2 * k + 1]));
    DK_TL(TL_STENCIL, 8);
    {
      const int* ss = sslot + (j % NB) * kSlotCap + (r0 & 3);
      if (RESTRICT)
        restrict_tail_runs<true>(rr, lb, sw, sl,
                                 wsum + (2 * grp + ((j / NG) & 1)) * kWarps, r1 - r0,
                                 [ss](int r) { return ss[r]; }, run_part);
    }
    DK_TL(TL_STENCIL, 9);
  }
  DK_TL(TL_STENCIL, 3);
  if (wait != nullptr) pdl_wait();
  DK_TL(TL_STENCIL, 4);
}

// The 7-point sums of a cell pair (i, i+1) in ascending-offset order (sym7_apply's), with the
// in-plane inputs from P(o) (o relative to cell i) and the z-plane inputs given.
template <class F>
__device__ __forceinline__ double2 sym7_pair(const Sym7Pair& q, F P, long long nx, double zm0,
                                             double zm1, double zp0, double zp1) {
  double r0 = __dmul_rn(q.uzm.x, zm0);
  r0 = __dadd_rn(r0, __dmul_rn(q.uxm.x, P(-nx)));
  r0 = __dadd_rn(r0, __dmul_rn(q.u1m.y, P(-1)));
  r0 = __dadd_rn(r0, __dmul_rn(q.c.x, P(0)));
  r0 = __dadd_rn(r0, __dmul_rn(q.u1.x, P(1)));
  r0 = __dadd_rn(r0, __dmul_rn(q.ux.x, P(nx)));
  r0 = __dadd_rn(r0, __dmul_rn(q.uz.x, zp0));
  double r1 = __dmul_rn(q.uzm.y, zm1);
  r1 = __dadd_rn(r1, __dmul_rn(q.uxm.y, P(1 - nx)));
  r1 = __dadd_rn(r1, __dmul_rn(q.u1.x, P(0)));
  r1 = __dadd_rn(r1, __dmul_rn(q.c.y, P(1)));
  r1 = __dadd_rn(r1, __dmul_rn(q.u1.y, P(2)));
  r1 = __dadd_rn(r1, __dmul_rn(q.ux.y, P(1 + nx)));
  r1 = __dadd_rn(r1, __dmul_rn(q.uz.y, zp1));
  return make_double2(r0, r1);
}

// Split-iteration stencil: w = A M^-1 (sigma v) exactly as k_stencil_sym7
// (same products, same order: bitwise equal), its run sums, and the run sums of
// a = A_p^T (sigma v) = A (sigma v) (times M^-1 for A_p = A M^-1; A symmetric), from which
// k_restrict_final forms the row c_j = Z^T A_p^T v_j of C.  sigma v and M^-1 are staged
// separately (the products are formed on use); the staging area is reused for the two
// segmented restrictions.
template <bool PRE>
__global__ void __launch_bounds__(kThreads, 4) k_stencil_sym7_split(
    Dia A, const double* __restrict__ v, const double* __restrict__ scale,
    double* __restrict__ out, const int* __restrict__ lab, const int* __restrict__ tile_run_off,
    const int* __restrict__ run_slot, double* __restrict__ run_part,
    double* __restrict__ run_part2, int am, const int* __restrict__ gate, int H,
    const unsigned* wait, const double* gsig, int ng) {
  DK_TL(TL_STENCIL, 0);
  if (wait != nullptr) {
    const long long b0 = (long long)blockIdx.x * kTile;
    const int t = threadIdx.x;
    if (t < 4) l2_prefetch(A.co[3 + t] + b0, kTile * 8);
    if (PRE && t == 4) l2_prefetch(A.inv + b0, kTile * 8);
    if (t == 5) l2_prefetch(lab + b0, kTile * 4);
    if (!early_start(wait, gate, (unsigned)ng)) return;
  } else {
    pdl_wait();
    if (gate != nullptr && *gate == 0) return;
  }
  DK_TL(TL_STENCIL, 1);
  pdl_trigger();
  extern __shared__ __align__(16) double sp[];  // [s1: sigma v | s2: M^-1], each H|kTile|H
  __shared__ double wsum[kWarps];
  const int L = kTile + 2 * H;
  double* s1 = sp;
  double* s2 = sp + L;
  const long long base = (long long)blockIdx.x * kTile;
  const long long nx = A.off[5], nz = A.off[6];
  const bool has_scale = scale != nullptr;
  const double sc = !has_scale ? 1.0 : wait != nullptr ? early_sigma(gsig, ng) : __ldcg(scale);
  const unsigned long long pol = l2_evict_first();
  for (int e = threadIdx.x; e < L / 2; e += kThreads) {
    const long long i = base - H + 2 * e;
    double2 x = ld2(v + i);
    if (has_scale) {
      x.x = __dmul_rn(x.x, sc);
      x.y = __dmul_rn(x.y, sc);
    }
    reinterpret_cast<double2*>(s1)[e] = x;
    if (PRE) reinterpret_cast<double2*>(s2)[e] = ld2_stream(A.inv + i, pol);
  }
  int2 lb[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) lb[k] = ldi2_stream(lab + base + 2 * threadIdx.x + 512 * k, pol);
  __syncthreads();
  double rr[8], aa[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int c = H + 2 * threadIdx.x + 512 * k;
    Sym7Pair q;
    sym7_load<PRE>(q, A, v, base + 2 * threadIdx.x + 512 * k, nx, nz, pol);
    const double vm0 = has_scale ? __dmul_rn(q.vm.x, sc) : q.vm.x;
    const double vm1 = has_scale ? __dmul_rn(q.vm.y, sc) : q.vm.y;
    const double vp0 = has_scale ? __dmul_rn(q.vp.x, sc) : q.vp.x;
    const double vp1 = has_scale ? __dmul_rn(q.vp.y, sc) : q.vp.y;
    const double2 r = sym7_pair(
        q, [&](long long o) { return PRE ? __dmul_rn(s1[c + o], s2[c + o]) : s1[c + o]; }, nx,
        PRE ? __dmul_rn(vm0, q.im.x) : vm0, PRE ? __dmul_rn(vm1, q.im.y) : vm1,
        PRE ? __dmul_rn(vp0, q.ip.x) : vp0, PRE ? __dmul_rn(vp1, q.ip.y) : vp1);
    double2 a = sym7_pair(q, [&](long long o) { return s1[c + o]; }, nx, vm0, vm1, vp0, vp1);
    if (PRE && am) {
      a.x = __dmul_rn(a.x, s2[c]);
      a.y = __dmul_rn(a.y, s2[c + 1]);
    }
    rr[2 * k] = r.x;
    rr[2 * k + 1] = r.y;
    aa[2 * k] = a.x;
    aa[2 * k + 1] = a.y;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
    st2(out + base + 2 * threadIdx.x + 512 * k, make_double2(rr[2 * k], rr[2 * k + 1]));
  __syncthreads();  // the staging area becomes the restriction scratch
  double* sw = sp;
  int* sl = reinterpret_cast<int*>(sp + kTilePad);
  stencil_restrict_tail(rr, lb, sw, sl, wsum, tile_run_off, run_slot, run_part, blockIdx.x);
  __syncthreads();
  stencil_restrict_tail(aa, lb, sw, sl, wsum, tile_run_off, run_slot, run_part2, blockIdx.x);
  DK_TL(TL_STENCIL, 3);
  if (wait != nullptr) pdl_wait();
  DK_TL(TL_STENCIL, 4);
}

// halo of k_stencil_sym7, or 0 when the operator is not the symmetric even 7-point stencil
static int sym7_halo(const Dia& A) {
  if (A.ndiag != 7 || A.center != 3 || A.off[3] != 0 || A.off[4] != 1) return 0;
  const long long nx = A.off[5], nz = A.off[6];
  if (A.off[2] != -1 || A.off[1] != -nx || A.off[0] != -nz) return 0;
  if ((nx & 1) || (nz & 1) || nx + 2 > 4096) return 0;
  if (A.co[0] != A.co[6] || A.co[1] != A.co[5] || A.co[2] != A.co[4]) return 0;
  if (A.csh[0] != -nz || A.csh[1] != -nx || A.csh[2] != -1) return 0;
  for (int q = 3; q < 7; ++q)
    if (A.csh[q] != 0) return 0;
  return (int)((nx + 2 + 31) / 32 * 32);
}

bool sym7_supported(const Dia& A) { return sym7_halo(A) > 0; }

void launch_stencil_split(bool pre, bool am, const Dia& A, long long n_pad, const double* v,
                          const double* scale, double* out, const RunMap& rm, double* run_part2,
                          const int* gate, cudaStream_t s, const unsigned* wait,
                          const double* gsig, int ng) {
  const int H = sym7_halo(A);
  const unsigned grid = (unsigned)(n_pad / kTile);
  size_t smem = (size_t)2 * (kTile + 2 * H) * sizeof(double);
  const size_t scratch = (size_t)kTilePad * (sizeof(double) + sizeof(int));
  if (smem < scratch) smem = scratch;
  if (pre) {
    smem_optin((const void*)k_stencil_sym7_split<true>, smem);
    launch_pdl(k_stencil_sym7_split<true>, dim3(grid), dim3(kThreads), smem, s, A, v, scale, out,
               rm.lab, rm.tile_run_off, rm.run_slot, rm.run_part, run_part2, am ? 1 : 0, gate,
               H, wait, gsig, ng);
  } else {
    smem_optin((const void*)k_stencil_sym7_split<false>, smem);
    launch_pdl(k_stencil_sym7_split<false>, dim3(grid), dim3(kThreads), smem, s, A, v, scale,
               out, rm.lab, rm.tile_run_off, rm.run_slot, rm.run_part, run_part2, am ? 1 : 0,
               gate, H, wait, gsig, ng);
  }
}

// stages of the bulk-copy ring that fit beside the kernel's static shared memory (0: use the
// register-load kernel, the default: the ring is opt-in with DK_RING=1 — at parity at config 3,
// 4 % / 11 % slower at configs 2 / 4, where its one 288-thread block per SM delays the early
// start against the previous kernel's draining blocks, profiles/r02f_ab_loop_ring.log)
template <bool PRE, bool R, bool W, int NG>
static int ring_stages(int H, size_t* stage_bytes) {
  static const bool on = getenv("DK_RING") != nullptr && getenv("DK_NO_RING") == nullptr;
  if (!on) return 0;
  static const int want = getenv("DK_RING_STAGES") ? atoi(getenv("DK_RING_STAGES")) : 4;
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, (const void*)k_stencil_sym7_ring<PRE, R, W, NG>) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, current_device());
  *stage_bytes = (size_t)ring_layout(H, PRE).stage * sizeof(double);
  const long long room = (long long)optin - (long long)fa.sharedSizeBytes - 256 -
                         (long long)ring_extra(NG, R);
  int S = (int)(room / (long long)*stage_bytes);
  if (S > want) S = want;
  if (S > 4) S = 4;  // a tile's slot list is refilled NG + 1 tiles later: needs S <= 4
  return S >= 2 ? S : 0;
}

// launches the ring kernel with NG compute groups when at least two stages fit
template <bool PRE, bool R, bool W, int NG>
static bool stencil7_ring(const Dia& A, int H, long long n_pad, const double* v,
                          const double* scale, double* out, const RunMap* rm, const int* gate,
                          cudaStream_t s, const unsigned* wait, const double* gsig, int ng) {
  const unsigned grid = (unsigned)(n_pad / kTile);
  size_t stage_bytes = 0;
  const int S = ring_stages<PRE, R, W, NG>(H, &stage_bytes);
  // pieces of the L2 prefetch issued before the early-start flag (DK_WPF_EARLY; default: the
  // ring's prologue stages)
  static const int pf_early = getenv("DK_WPF_EARLY") ? atoi(getenv("DK_WPF_EARLY")) : S;
  if (S <= 0 ||
      smem_optin((const void*)k_stencil_sym7_ring<PRE, R, W, NG>,
                 S * stage_bytes + ring_extra(NG, R)) != 0)
    return false;
  const unsigned sms = (unsigned)num_sms();
  launch_pdl(k_stencil_sym7_ring<PRE, R, W, NG>, dim3(grid < sms ? grid : sms),
             dim3(ring_threads(NG)), S * stage_bytes + ring_extra(NG, R), s, A, v, scale, out,
             rm ? rm->lab : nullptr, rm ? rm->tile_run_off : nullptr,
             rm ? rm->run_slot : nullptr, rm ? rm->run_part : nullptr, gate, H, S, (int)grid,
             wait, gsig, ng, rm ? (const char*)rm->pf_base : (const char*)nullptr,
             rm ? rm->pf_bytes : 0ull, pf_early);
  return true;
}

template <bool PRE, bool R, bool W>
static void stencil7_t(const Dia& A, int H, long long n_pad, const double* v, const double* scale,
                       double* out, const RunMap* rm, const int* gate, cudaStream_t s,
                       const unsigned* wait, const double* gsig, int ng) {
  const unsigned grid = (unsigned)(n_pad / kTile);
  // the opt-in ring (DK_RING=1): DK_RING_GROUPS=2 runs two compute groups per block
  static const int groups = getenv("DK_RING_GROUPS") ? atoi(getenv("DK_RING_GROUPS")) : 1;
  if (groups >= 2 &&
      stencil7_ring<PRE, R, W, 2>(A, H, n_pad, v, scale, out, rm, gate, s, wait, gsig, ng))
    return;
  if (stencil7_ring<PRE, R, W, 1>(A, H, n_pad, v, scale, out, rm, gate, s, wait, gsig, ng))
    return;
  const size_t smem = (size_t)(kTile + 2 * H) * sizeof(double);
  // static + dynamic above 48 KB needs the opt-in (wide grids: nx = 512)
  smem_optin((const void*)k_stencil_sym7<PRE, R, W>, smem);
  launch_pdl(k_stencil_sym7<PRE, R, W>, dim3(grid), dim3(kThreads), smem, s, A, v, scale, out,
             rm ? rm->lab : nullptr, rm ? rm->tile_run_off : nullptr,
             rm ? rm->run_slot : nullptr, rm ? rm->run_part : nullptr, gate, H, wait, gsig, ng);
}

template <int MODE, bool PRE, bool R, bool W>
static void stencil_t(const Dia& A, long long n_pad, const double* v, const double* scale,
                      const double* b, double* out, const RunMap* rm, const int* gate,
                      cudaStream_t s, const unsigned* wait = nullptr,
                      const double* gsig = nullptr, int ng = 0) {
  const unsigned grid = (unsigned)(n_pad / kTile);
  launch_pdl(k_stencil<MODE, PRE, R, W>, dim3(grid), dim3(kThreads), 0, s, A, v, scale, b, out,
             rm ? rm->lab : nullptr, rm ? rm->tile_run_off : nullptr,
             rm ? rm->run_slot : nullptr, rm ? rm->run_part : nullptr, gate, wait, gsig, ng);
}

template <int MODE, bool PRE>
static void stencil_rw(bool write, const Dia& A, long long n_pad, const double* v,
                       const double* scale, const double* b, double* out, const RunMap* rm,
                       const int* gate, cudaStream_t s, const unsigned* wait = nullptr,
                       const double* gsig = nullptr, int ng = 0) {
  if (rm) {
    if (write)
      stencil_t<MODE, PRE, true, true>(A, n_pad, v, scale, b, out, rm, gate, s, wait, gsig, ng);
    else stencil_t<MODE, PRE, true, false>(A, n_pad, v, scale, b, out, rm, gate, s, wait, gsig, ng);
  } else {
    stencil_t<MODE, PRE, false, true>(A, n_pad, v, scale, b, out, rm, gate, s, wait, gsig, ng);
  }
}

void launch_stencil(int mode, bool pre, bool write, const Dia& A, long long n_pad, const double* v,
                    const double* scale, const double* b, double* out, const RunMap* rm,
                    const int* gate, cudaStream_t s, const unsigned* wait, const double* gsig,
                    int ng) {
  if (mode != ST_APPLY) wait = nullptr;
  const int H = (mode == ST_APPLY && !getenv("DK_GENERIC_STENCIL")) ? sym7_halo(A) : 0;
  if (H > 0) {
    if (pre && rm && write)
      stencil7_t<true, true, true>(A, H, n_pad, v, scale, out, rm, gate, s, wait, gsig, ng);
    else if (pre && rm) stencil7_t<true, true, false>(A, H, n_pad, v, scale, out, rm, gate, s, wait, gsig, ng);
    else if (pre) stencil7_t<true, false, true>(A, H, n_pad, v, scale, out, rm, gate, s, wait, gsig, ng);
    else if (rm && write)
      stencil7_t<false, true, true>(A, H, n_pad, v, scale, out, rm, gate, s, wait, gsig, ng);
    else if (rm) stencil7_t<false, true, false>(A, H, n_pad, v, scale, out, rm, gate, s, wait, gsig, ng);
    else stencil7_t<false, false, true>(A, H, n_pad, v, scale, out, rm, gate, s, wait, gsig, ng);
    return;
  }
  if (mode == ST_IDENT) {
    stencil_rw<ST_IDENT, false>(write, A, n_pad, v, scale, b, out, rm, gate, s);
  } else if (mode == ST_RESID) {
    stencil_rw<ST_RESID, false>(write, A, n_pad, v, scale, b, out, rm, gate, s);
  } else if (pre) {
    stencil_rw<ST_APPLY, true>(write, A, n_pad, v, scale, b, out, rm, gate, s, wait, gsig, ng);
  } else {
    stencil_rw<ST_APPLY, false>(write, A, n_pad, v, scale, b, out, rm, gate, s, wait, gsig, ng);
  }
}

// ======================================================================================
// K2: per-column sum of run partials (label-major slots: one thread per column, a warp per
// column with more than kShortRuns runs; fixed order).
// ======================================================================================
#ifndef DK_LONG_BATCH
#define DK_LONG_BATCH 16
#endif
constexpr int kLongBatch = DK_LONG_BATCH;  // loads per lane in flight for a long column

__global__ void __launch_bounds__(kThreads) k_restrict_final(const double* __restrict__ run_part,
                                                             const int* __restrict__ ptr, int d,
                                                             const int* __restrict__ long_ids,
                                                             int nlong, int short_blocks,
                                                             double* __restrict__ s,
                                                             const int* __restrict__ s_pos,
                                                             const int* __restrict__ gate,
                                                             const double* __restrict__ rp2,
                                                             double* __restrict__ out2) {
  DK_TL(TL_RESTRICT, 0);
  pdl_trigger();  // the tile GEMV's prologue (tile prefetch) overlaps this grid
  pdl_wait();
  DK_TL(TL_RESTRICT, 1);
  if (gate != nullptr && *gate == 0) return;
  if ((int)blockIdx.x < short_blocks) {
    // one thread per column with at most kShortRuns runs, serial in run order
    const int L = blockIdx.x * blockDim.x + threadIdx.x;
    if (L >= d) return;
    const int lo = ptr[L], len = ptr[L + 1] - lo;
    if (len > kShortRuns) return;
    double v[kShortRuns];  // every load in flight, then the in-order sum
#pragma unroll
    for (int k = 0; k < kShortRuns; ++k) v[k] = k < len ? __ldcg(run_part + lo + k) : 0.0;
    double acc = 0.0;
#pragma unroll
    for (int k = 0; k < kShortRuns; ++k)
      if (k < len) acc += v[k];
    s[s_pos ? s_pos[L] : L] = acc;
    if (out2 != nullptr) {
#pragma unroll
      for (int k = 0; k < kShortRuns; ++k) v[k] = k < len ? __ldcg(rp2 + lo + k) : 0.0;
      double a2 = 0.0;
#pragma unroll
      for (int k = 0; k < kShortRuns; ++k)
        if (k < len) a2 += v[k];
      out2[L] = a2;
    }
    DK_TL(TL_RESTRICT, 4);
    return;
  }
  // one warp per long column (lane-strided, kLongBatch loads per lane in flight, fixed xor tree)
  const int wl = ((blockIdx.x - short_blocks) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wl >= nlong) return;
  const int L = long_ids[wl];
  double acc = 0.0, a2 = 0.0;
  const int lo = ptr[L], hi = ptr[L + 1];
  for (int k0 = lo + lane; k0 < hi; k0 += 32 * kLongBatch) {
    double v[kLongBatch];
#pragma unroll
    for (int i = 0; i < kLongBatch; ++i)
      v[i] = k0 + 32 * i < hi ? __ldcg(run_part + k0 + 32 * i) : 0.0;
#pragma unroll
    for (int i = 0; i < kLongBatch; ++i)
      if (k0 + 32 * i < hi) acc += v[i];
    if (out2 != nullptr) {
#pragma unroll
      for (int i = 0; i < kLongBatch; ++i)
        v[i] = k0 + 32 * i < hi ? __ldcg(rp2 + k0 + 32 * i) : 0.0;
#pragma unroll
      for (int i = 0; i < kLongBatch; ++i)
        if (k0 + 32 * i < hi) a2 += v[i];
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) s[s_pos ? s_pos[L] : L] = acc;
  if (out2 != nullptr) {
    a2 = warp_sum(a2);
    if (lane == 0) out2[L] = a2;
  }
  DK_TL(TL_RESTRICT, 4);
}

void launch_restrict_final(const RunMap& rm, double* s_out, const int* gate, cudaStream_t s,
                           const double* run_part2, double* out2) {
  if (rm.d <= 0) return;
  const int short_blocks = (rm.d + kThreads - 1) / kThreads;
  const unsigned grid =
      (unsigned)(short_blocks + ((long long)rm.nlong * 32 + kThreads - 1) / kThreads);
  launch_pdl(k_restrict_final, dim3(grid), dim3(kThreads), 0, s, rm.run_part, rm.lab_run_ptr,
             rm.d, rm.long_ids, rm.nlong, short_blocks, s_out, rm.s_pos, gate, run_part2, out2);
}

// ======================================================================================
// Control sections.  These restate _run_cycles' scalar logic (krylov.py:127-212) on the
// device so nothing round-trips to the host per iteration.  They run in the last block of a
// reduction kernel; all threads of that block call them (shared-memory staging), one
// thread makes the decisions.
// ======================================================================================
__device__ void restart_done_block(const Scal& sc, double norm2) {
  __shared__ int s_open;
  State* st = sc.st;
  if (threadIdx.x == 0) {
    const double beta = sqrt(norm2);
    st->beta = beta;
    st->xupdate = 0;
    st->cycle_open = 0;
    st->active = 0;
    st->reorth = 0;
    s_open = 0;
    if (!st->denom_set) {  // krylov.py:132-136
      st->denom = beta > 0.0 ? beta : 1.0;
      st->denom_set = 1;
      sc.hist[0] = beta;
      sc.restart_of[0] = 0;
    }
    if (beta == 0.0 || (beta <= st->tol * st->denom && st->iterations >= st->min_iters)) {
      st->converged = 1;  // krylov.py:137-139
      st->running = 0;
    } else if (st->has_prev && beta >= st->prev_beta * (1.0 - 1e-14) && st->warning) {
      st->running = 0;  // krylov.py:140-141: breakdown with no progress
    } else {
      st->prev_beta = beta;
      st->has_prev = 1;
      sc.sigma[0] = 1.0 / beta;  // V[0] = r / beta  (krylov.py:145)
      st->cols = 0;
      st->cycle_open = 1;
      st->active = (st->iterations < st->max_iters) ? 1 : 0;  // krylov.py:157-158
      s_open = 1;
    }
  }
  __syncthreads();
  if (s_open) {
    const int m = sc.m;
    const double beta = st->beta;
    for (int i = threadIdx.x; i <= m; i += blockDim.x) sc.g[i] = (i == 0) ? beta : 0.0;
    for (int i = threadIdx.x; i < (m + 1) * m; i += blockDim.x) {
      sc.H[i] = 0.0;
      sc.R[i] = 0.0;
    }
  }
}

// Hessenberg column j is final in H except H[j+1, j] = hj1: Givens update, residual
// estimate, convergence and breakdown tests (krylov.py:171-197).  sm: >= 3(m+1) doubles.
__device__ void finish_iteration_block(const Scal& sc, int j, double hj1, double* sm) {
  State* st = sc.st;
  const int m = sc.m;
  double* Hc = sc.H + (size_t)j * (m + 1);
  double* Rc = sc.R + (size_t)j * (m + 1);
  double* col = sm;
  double* cs = sm + (m + 1);
  double* sn = cs + (m + 1);
  for (int i = threadIdx.x; i <= j; i += blockDim.x) col[i] = Hc[i];
  for (int i = threadIdx.x; i < j; i += blockDim.x) {
    cs[i] = sc.cs[i];
    sn[i] = sc.sn[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    col[j + 1] = hj1;
    Hc[j + 1] = hj1;  // krylov.py:172
    double hn = 0.0;
    for (int i = 0; i <= j + 1; ++i) hn += col[i] * col[i];
    hn = sqrt(hn);
    // _givens_update, krylov.py:90-104 (separately rounded products, as Python floats)
    for (int i = 0; i < j; ++i) {
      const double t = __dadd_rn(__dmul_rn(cs[i], col[i]), __dmul_rn(sn[i], col[i + 1]));
      col[i + 1] = __dadd_rn(__dmul_rn(-sn[i], col[i]), __dmul_rn(cs[i], col[i + 1]));
      col[i] = t;
    }
    const double den = hypot(col[j], col[j + 1]);
    double c = 1.0, s = 0.0;
    if (den != 0.0) {
      c = col[j] / den;
      s = col[j + 1] / den;
    }
    sc.cs[j] = c;
    sc.sn[j] = s;
    col[j] = den;
    col[j + 1] = 0.0;
    const double gj = sc.g[j];
    sc.g[j + 1] = __dmul_rn(-s, gj);
    sc.g[j] = __dmul_rn(c, gj);
    st->cols = j + 1;
    const double resnorm = fabs(sc.g[j + 1]);
    st->iterations += 1;
    sc.hist[st->iterations] = resnorm;
    sc.restart_of[st->iterations] = st->cycle;
    st->reorth = 0;
    if (resnorm <= st->tol * st->denom && st->iterations >= st->min_iters) {  // :189-191
      st->converged = 1;
      st->active = 0;
      st->last_broke = 1;
    } else if (hj1 <= 1e-13 * fmax(1.0, hn)) {  // :192-194
      st->warning = DK_WARNING_BREAKDOWN;
      st->active = 0;
      st->last_broke = 1;
    } else {
      st->last_broke = 0;
      sc.sigma[j + 1] = 1.0 / hj1;  // V[j+1] = w / hj1 (:197)
      if (j + 1 >= m || st->iterations >= st->max_iters) st->active = 0;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i <= j + 1; i += blockDim.x) Rc[i] = col[i];
}

// ======================================================================================
// K4: prolongation + subtraction, multi-dot and norm.
//
// h_i = V_i . w (classical Gram-Schmidt coefficients) in one sweep over V.  With the basis
// Gram matrix G the reference's re-orthogonalisation test (krylov.py:167-168: max |V^T w'|
// > 1e-8 ||w0|| after the projection) is evaluated without another pass over V:
//     V^T (w - V h) = h - G h,
// and the same identity gives G's next column (iter_finish): the test and G are exact up to
// O(eps ||w||), several orders below the threshold.
// ======================================================================================
// Prolongation (A_p Z y)_i = sum over the row's coefficients of y[label of the column].
// Precomputed per cell (k_prolong_setup): own = sum of the coefficients whose column carries
// the cell's own label; the first two other labels met along the row (ascending diagonal)
// with their summed coefficients (95 % of the cells at config 3 have at most two); an 8-bit
// mask of the diagonals whose label is a third or later one.  Every per-cell input is one
// coalesced load at the cell's own index and the y gathers follow directly; only the masked
// remainder reads coefficients and neighbour labels.
template <bool AM>
__device__ __forceinline__ double prolong_cell(const Dia& A, const Prolong& P,
                                               const double* __restrict__ yc, long long c,
                                               int L, double own, int f1, int f2, double c1,
                                               double c2, unsigned msk) {
  const double y0 = L >= 0 ? __ldg(yc + L) : 0.0;
  const double y1 = f1 >= 0 ? __ldg(yc + f1) : 0.0;
  const double y2 = f2 >= 0 ? __ldg(yc + f2) : 0.0;
  double t = (L >= 0) ? __dmul_rn(own, y0) : 0.0;
  if (f1 >= 0) t = __dadd_rn(t, __dmul_rn(c1, y1));
  if (f2 >= 0) t = __dadd_rn(t, __dmul_rn(c2, y2));
  if (msk) {
    // all masked coefficients and neighbour labels first (independent loads in flight), then
    // the y gathers, then the sum in diagonal order
    double a[kMaxDiag];
    int nl[kMaxDiag];
#pragma unroll
    for (int q = 0; q < kMaxDiag; ++q) {
      const bool on = (msk >> q) & 1u;
      const long long o = A.off[q];
      a[q] = on ? dia_coef(A, q, c) : 0.0;
      if (AM) a[q] = on ? __dmul_rn(a[q], __ldg(A.inv + c + o)) : 0.0;
      nl[q] = on ? __ldg(P.lab + c + o) : 0;
    }
    double yv[kMaxDiag];
#pragma unroll
    for (int q = 0; q < kMaxDiag; ++q) yv[q] = ((msk >> q) & 1u) ? __ldg(yc + nl[q]) : 0.0;
#pragma unroll
    for (int q = 0; q < kMaxDiag; ++q)
      if ((msk >> q) & 1u) t = __dadd_rn(t, __dmul_rn(a[q], yv[q]));
  }
  return t;
}

template <bool AM>
__global__ void k_prolong_setup(Dia A, const int* __restrict__ lab, long long n_pad,
                                double* __restrict__ own, int2* __restrict__ flab,
                                double2* __restrict__ fco, unsigned char* __restrict__ mask,
                                unsigned long long* __restrict__ nmasked) {
  unsigned cnt = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_pad;
       i += (long long)gridDim.x * blockDim.x) {
    const int L = lab[i];
    double s = 0.0, c1 = 0.0, c2 = 0.0;
    int f1 = -1, f2 = -1;
    unsigned m = 0;
    for (int q = 0; q < A.ndiag; ++q) {
      const int L2 = lab[i + A.off[q]];
      if (L2 < 0) continue;
      double a = dia_coef(A, q, i);
      if (AM) a = __dmul_rn(a, A.inv[i + A.off[q]]);
      if (L2 == L) {
        s = __dadd_rn(s, a);
      } else if (f1 < 0 || L2 == f1) {
        f1 = L2;
        c1 = __dadd_rn(c1, a);
      } else if (f2 < 0 || L2 == f2) {
        f2 = L2;
        c2 = __dadd_rn(c2, a);
      } else {
        m |= 1u << q;
      }
    }
    own[i] = s;
    flab[i] = make_int2(f1, f2);
    fco[i] = make_double2(c1, c2);
    mask[i] = (unsigned char)m;
    cnt += __popc(m);
  }
  // number of foreign-label coefficients (the gathers the prolongation pays beyond `own`)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(nmasked, (unsigned long long)cnt);
}

void launch_prolong_setup(bool am, const Dia& A, const int* lab, long long n_pad, double* own,
                          int2* flab, double2* fco, unsigned char* mask,
                          unsigned long long* nmasked, cudaStream_t s) {
  if (am)
    k_prolong_setup<true><<<num_sms() * 8, kThreads, 0, s>>>(A, lab, n_pad, own, flab, fco, mask,
                                                         nmasked);
  else
    k_prolong_setup<false><<<num_sms() * 8, kThreads, 0, s>>>(A, lab, n_pad, own, flab, fco, mask,
                                                          nmasked);
}

__device__ __forceinline__ double gram_at(const double* Gm, int m, int i, int k) {
  return i <= k ? Gm[(size_t)k * (m + 1) + i] : Gm[(size_t)i * (m + 1) + k];
}

// Warp reduce-scatter of 8 per-lane values: returns, in lanes with (lane & 3) == 0, the warp
// sum of value (lane >> 2).  9 shuffles instead of 8 x 5; fixed order (deterministic).
__device__ __forceinline__ double reduce8(double (&v)[8], int lane) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const bool up = (lane & 16) != 0;
    const double send = up ? v[i] : v[i + 4];
    const double keep = up ? v[i + 4] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const bool up = (lane & 8) != 0;
    const double send = up ? v[i] : v[i + 2];
    const double keep = up ? v[i + 2] : v[i];
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  {
    const bool up = (lane & 4) != 0;
    const double send = up ? v[0] : v[1];
    const double keep = up ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
  }
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
  v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
  return v[0];
}

// Last block of an Arnoldi projection: red[0..2 nvec] holds the reduced V^T w, the reduced
// Gram column V^T v_j (measured in the same sweep: it carries the basis' actual loss of
// orthogonality, which the test exists to detect) and ||w||^2.  Writes the Hessenberg column,
// the update coefficients and the Gram column, and evaluates the re-orthogonalisation test
// (krylov.py:162-170): corr = V^T u = h - G h for u = w - V h; corr is also kept in gcol (the
// Gram row of the cycle's last vector, reported with the Arnoldi data).  Shared scratch after
// red[0..2 nvec]: h[nvec], |corr|[nvec] and, for nvec <= kStageGram, G[nvec][nvec] (larger
// cycles read G from global memory).
constexpr int kStageGram = 96;
// h_i of the split iteration: sigma_i (U^T w)_i - (C y)_i, the arithmetic k_gs's early start
// repeats bitwise
__device__ __forceinline__ double split_h(const Scal& sc, int i, double cy) {
  return __dsub_rn(__dmul_rn(__ldcg(sc.hraw + i), __ldcg(sc.sigma + i)), cy);
}

// SPLIT: red[0..nvec) = C y, red[nvec] = ||w||^2, U^T w and U^T u_j in sc.hraw
template <bool SPLIT = false>
__device__ void iter_finish(const Scal& sc, int j, int nvec, double* red) {
  State* st = sc.st;
  const int m = sc.m;
  double* Hc = sc.H + (size_t)j * (m + 1);
  const double sj = sc.sigma[nvec - 1];
  const bool stage = nvec <= kStageGram;
  double* sh_h = red + 2 * nvec + 1;
  double* sh_c = sh_h + nvec;
  double* sh_g = sh_c + nvec;
  for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
    // h_i = V_i . w  (krylov.py:164-165)
    const double h = SPLIT ? split_h(sc, v, red[v]) : red[v] * sc.sigma[v];
    Hc[v] = h;
    sh_h[v] = h;
    sc.coef[v] = h * sc.sigma[v];
    // V_i . V_j
    const double g = (SPLIT ? sc.hraw[sc.m + 1 + v] : red[nvec + v]) * sc.sigma[v] * sj;
    sc.Gm[(size_t)j * (m + 1) + v] = g;
    if (stage) {
      sh_g[v * nvec + (nvec - 1)] = g;
      sh_g[(nvec - 1) * nvec + v] = g;
    }
  }
  if (stage) {  // eight Gram loads per thread in flight (this section is latency-bound)
    const int ne = (nvec - 1) * (nvec - 1);
    for (int e0 = threadIdx.x; e0 < ne; e0 += 8 * blockDim.x) {
      double g8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * blockDim.x;
        g8[u] = e < ne ? gram_at(sc.Gm, m, e / (nvec - 1), e % (nvec - 1)) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + u * blockDim.x;
        if (e < ne) sh_g[(e / (nvec - 1)) * nvec + e % (nvec - 1)] = g8[u];
      }
    }
  }
  __syncthreads();
  // corr_i = h_i - sum_k G_ik h_k
  for (int i = threadIdx.x; i < nvec; i += blockDim.x) {
    double c = sh_h[i];
    for (int k = 0; k < nvec; ++k)
      c -= (stage ? sh_g[i * nvec + k] : gram_at(sc.Gm, m, i, k)) * sh_h[k];
    sh_c[i] = fabs(c);
    sc.gcol[i] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    st->wnorm0 = sqrt(red[SPLIT ? nvec : 2 * nvec]);  // krylov.py:162
    double mx = 0.0;
    for (int i = 0; i < nvec; ++i) mx = fmax(mx, sh_c[i]);
    if (mx > 1e-8 * fmax(st->wnorm0, 1e-300)) {  // krylov.py:168
      st->reorth = 1;
      st->reorths += 1;
    } else {
      st->reorth = 0;
    }
  }
}

template <int MODE, int DEFL, bool AM>
__global__ void __launch_bounds__(kThreads, 4) k_project(Dia A, Prolong P,
                                                      const double* __restrict__ yc,
                                                      const double* w_in, double* w_out,
                                                      const double* __restrict__ V,
                                                      long long vstride, int nvec, long long n_pad,
                                                      double* __restrict__ part, int G, Scal sc,
                                                      int j, const int* __restrict__ gate) {
  constexpr bool DOTS = MODE == PJ_ITER || MODE == PJ_REDOTS || MODE == PJ_DOTS;  // V sweep
  constexpr bool GRAM = MODE == PJ_ITER || MODE == PJ_DOTS;  // also V^T v_j
  constexpr bool NORM = MODE == PJ_ITER || MODE == PJ_RESTART || MODE == PJ_FIX;
  constexpr bool CTRL = MODE == PJ_ITER || MODE == PJ_FIX;  // the iteration's control block
  if (CTRL) DK_TL(TL_PROJECT, 0);
  if (MODE == PJ_DOTS) DK_TL(TL_DOTS, 0);
  pdl_wait();
  if (CTRL) DK_TL(TL_PROJECT, 1);
  if (MODE == PJ_DOTS) DK_TL(TL_DOTS, 1);
  // the stencil of this iteration has completed: re-arm its early-start flag
  if (CTRL && sc.post != nullptr && j >= 1 && blockIdx.x == 0 && threadIdx.x == 0) {
    sc.post[j - 1] = 0u;            // consumed by this iteration's stencil
    sc.post[sc.m + 1 + j - 1] = 0u;  // consumed by the previous k_gs (done: the stencil waited)
  }
  if (*gate == 0) return;
  extern __shared__ double red[];  // [nq][kWarps]
  __shared__ __align__(16) double s_w[DOTS ? kChunk : 2];
  __shared__ __align__(16) double s_vj[GRAM ? kChunk : 2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // quantities: ITER: h[nvec], g[nvec], |w|^2 ; RESTART: |w|^2 ; REDOTS: corr[nvec] ;
  // DOTS: h'[nvec], g[nvec] ; FIX: (C y)[nvec], |w|^2
  const int nq = (MODE == PJ_ITER) ? 2 * nvec + 1
                 : (MODE == PJ_DOTS) ? 2 * nvec
                 : (MODE == PJ_REDOTS) ? nvec
                 : (MODE == PJ_FIX) ? nvec + 1 : 1;
  const int nslot = (MODE == PJ_ITER) ? 2 * nvec : (MODE == PJ_FIX) ? nvec : 0;
  for (int q = threadIdx.x; q < nq * kWarps; q += blockDim.x) red[q] = 0.0;
  __syncthreads();
  const long long nchunks = n_pad / kChunk;
  const double* Vj = V + (long long)(nvec - 1) * vstride;
  for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const long long cb = ch * kChunk + 2 * threadIdx.x;
    double w[8];
    // every per-cell input of the chunk first (w is updated in place: no load may wait
    // behind a store), then the prolongation gathers, then the stores
    double2 xin[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const long long i = cb + 512 * k;
      xin[k] = (MODE == PJ_REDOTS) ? ld2cg(w_in + i) : ld2_vec(w_in + i);
    }
    if (DEFL == DK_LABELS) {
      const unsigned long long cpol = l2_evict_first();
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const long long i = cb + 512 * k;
        const int2 L = ldi2_stream(P.lab + i, cpol);
        const double2 ow = ld2_stream(P.own + i, cpol);
        const int4 fl = ldi4_stream(reinterpret_cast<const int*>(P.flab + i), cpol);
        const double2 fa = ld2_stream(reinterpret_cast<const double*>(P.fco + i), cpol);
        const double2 fb = ld2_stream(reinterpret_cast<const double*>(P.fco + i) + 2, cpol);
        const double4 fc = make_double4(fa.x, fa.y, fb.x, fb.y);
        const unsigned short mw = ldu16_stream(P.mask + i, cpol);
        const uchar2 mk = make_uchar2((unsigned char)(mw & 0xff), (unsigned char)(mw >> 8));
        xin[k].x = __dsub_rn(xin[k].x, prolong_cell<AM>(A, P, yc, i, L.x, ow.x, fl.x, fl.y,
                                                        fc.x, fc.y, mk.x));
        xin[k].y = __dsub_rn(xin[k].y, prolong_cell<AM>(A, P, yc, i + 1, L.y, ow.y, fl.z, fl.w,
                                                        fc.z, fc.w, mk.y));
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const long long i = cb + 512 * k;
      double2 x = xin[k];
      if (DEFL == DK_LABELS) {
      } else if (DEFL == DK_DENSE) {  // w -= (A_p Z) y   (deflation.py:61-62)
        double t0 = 0.0, t1 = 0.0;
        for (int q = 0; q < P.dz; ++q) {
          const double yq = __ldg(yc + q);
          const double2 a = ld2(P.az + (long long)q * P.azs + i);
          t0 = fma(yq, a.x, t0);
          t1 = fma(yq, a.y, t1);
        }
        x.x = __dsub_rn(x.x, t0);
        x.y = __dsub_rn(x.y, t1);
      }
      w[2 * k] = x.x;
      w[2 * k + 1] = x.y;
      if (MODE != PJ_REDOTS && (DEFL != DK_NONE || w_out != w_in)) st2_vec(w_out + i, x);
    }
    if (CTRL && ch == blockIdx.x) DK_TL(TL_PROJECT, 2);
    if (NORM) {
      double nrm = 0.0;
#pragma unroll
      for (int e = 0; e < 8; ++e) nrm = fma(w[e], w[e], nrm);
      nrm = warp_sum(nrm);
      if (lane == 0) red[nslot * kWarps + warp] += nrm;
    }
    if (DOTS) {
      // Stage w (and v_j) of the chunk in shared memory; the warps then stream the basis as
      // (vector, quarter-chunk) items: 8 x 16 B loads in flight per lane and one warp
      // reduction per 4 KB of V, instead of one per 128 B.  Item (v, q) goes to warp
      // (4v + q) % 8 and its partial to that warp's slot: fixed order, deterministic.  Each
      // V_i load serves both dots, V_i . w and the Gram entry V_i . v_j.  (Register-resident
      // quarters of w and v_j instead of the staging spill at 64 registers: measured slower.)
      double2* sw2 = reinterpret_cast<double2*>(s_w);
      double2* sv2 = reinterpret_cast<double2*>(s_vj);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        sw2[threadIdx.x + 256 * k] = make_double2(w[2 * k], w[2 * k + 1]);
        if (GRAM) sv2[threadIdx.x + 256 * k] = ld2_vec(Vj + cb + 512 * k);
      }
      __syncthreads();
      const long long c0 = ch * kChunk;
      const unsigned long long pol = l2_evict_first();
#ifndef DK_K4_SINGLE
      // two items per round (16 loads per lane in flight), each reduced as before
      for (int it = warp; it < 4 * nvec; it += 2 * kWarps) {
        const int it2 = it + kWarps;
        const bool two = it2 < 4 * nvec;
        const int v = it >> 2, qtr = it & 3, v2 = it2 >> 2;
        const double* Vr = V + (long long)v * vstride + c0 + 512 * qtr + 2 * lane;
        const double* Vr2 = V + (long long)(two ? v2 : v) * vstride + c0 + 512 * qtr + 2 * lane;
        double2 p[8], p2[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) p[i] = ld2_stream(Vr + 64 * i, pol);
#pragma unroll
        for (int i = 0; i < 8; ++i)
          p2[i] = two ? ld2_stream(Vr2 + 64 * i, pol) : make_double2(0.0, 0.0);
        double ah = 0.0, ag = 0.0, ah2 = 0.0, ag2 = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int e = 256 * qtr + lane + 32 * i;
          const double2 ww = sw2[e];
          ah = fma(p[i].x, ww.x, ah);
          ah = fma(p[i].y, ww.y, ah);
          ah2 = fma(p2[i].x, ww.x, ah2);
          ah2 = fma(p2[i].y, ww.y, ah2);
          if (GRAM) {
            const double2 gg = sv2[e];
            ag = fma(p[i].x, gg.x, ag);
            ag = fma(p[i].y, gg.y, ag);
            ag2 = fma(p2[i].x, gg.x, ag2);
            ag2 = fma(p2[i].y, gg.y, ag2);
          }
        }
        ah = warp_sum(ah);
        ah2 = warp_sum(ah2);
        if (GRAM) {
          ag = warp_sum(ag);
          ag2 = warp_sum(ag2);
        }
        if (lane == 0) {
          red[v * kWarps + warp] += ah;
          if (GRAM) red[(nvec + v) * kWarps + warp] += ag;
          if (two) {
            red[v2 * kWarps + warp] += ah2;
            if (GRAM) red[(nvec + v2) * kWarps + warp] += ag2;
          }
        }
      }
#else
      for (int it = warp; it < 4 * nvec; it += kWarps) {
        const int v = it >> 2, qtr = it & 3;
        const double* Vr = V + (long long)v * vstride + c0 + 512 * qtr + 2 * lane;
        double2 p[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) p[i] = ld2_stream(Vr + 64 * i, pol);
        double ah = 0.0, ag = 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int e = 256 * qtr + lane + 32 * i;
          const double2 ww = sw2[e];
          ah = fma(p[i].x, ww.x, ah);
          ah = fma(p[i].y, ww.y, ah);
          if (GRAM) {
            const double2 gg = sv2[e];
            ag = fma(p[i].x, gg.x, ag);
            ag = fma(p[i].y, gg.y, ag);
          }
        }
        ah = warp_sum(ah);
        if (GRAM) ag = warp_sum(ag);
        if (lane == 0) {
          red[v * kWarps + warp] += ah;
          if (GRAM) red[(nvec + v) * kWarps + warp] += ag;
        }
      }
#endif
      __syncthreads();  // the next chunk reuses s_w / s_vj
    }
  }
  if (MODE == PJ_FIX) {
    // this block's slice of the coarse columns: (C y)_i over [c0, c1), serial in k
    const long long c0 = (long long)blockIdx.x * sc.dco / gridDim.x;
    const long long c1 = (long long)(blockIdx.x + 1) * sc.dco / gridDim.x;
    if ((int)threadIdx.x < nvec) {
      const double* Cr = sc.cmat + (long long)threadIdx.x * sc.ldc;
      double acc = 0.0;
      for (long long k = c0; k < c1; ++k) acc = fma(__ldcg(Cr + k), __ldcg(yc + k), acc);
      red[threadIdx.x * kWarps] += acc;
    }
  }
  if (CTRL) DK_TL(TL_PROJECT, 3);
  if (MODE == PJ_DOTS) DK_TL(TL_DOTS, 3);
  pdl_trigger();
  if (MODE == PJ_PLAIN) return;
  __syncthreads();
  for (int q = threadIdx.x; q < nq; q += blockDim.x) {
    double s = 0.0;
    for (int w2 = 0; w2 < kWarps; ++w2) s += red[q * kWarps + w2];
    part[(size_t)q * G + blockIdx.x] = s;
  }
  if (!reduce_grouped(part, nq, G, sc.gticket, sc.gpart, red,
                      (CTRL && sc.post != nullptr) ? sc.post + (sc.m + 1) + j : nullptr)) {
    if (CTRL) DK_TL(TL_PROJECT, 4);
    if (MODE == PJ_DOTS) DK_TL(TL_DOTS, 4);
    return;
  }
  if (MODE == PJ_DOTS) {  // U^T w and U^T u_j for the split iteration's control block
    for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
      sc.hraw[v] = red[v];
      sc.hraw[sc.m + 1 + v] = red[nvec + v];
    }
    DK_TL(TL_DOTS, 5);
    return;
  }
  State* st = sc.st;
  const int m = sc.m;
  if (MODE == PJ_RESTART) {
    restart_done_block(sc, red[0]);
    return;
  }
  double* Hc = sc.H + (size_t)j * (m + 1);
  if (MODE == PJ_REDOTS) {  // second Gram-Schmidt pass coefficients (krylov.py:169-170)
    double* cr = red + nvec;
    for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
      cr[v] = red[v] * sc.sigma[v];
      Hc[v] += cr[v];
      sc.corr[v] = cr[v] * sc.sigma[v];
    }
    __syncthreads();
    // V^T u' for u' = u - V corr2: corr2 - G corr2 (the next Gram column, up to sigma)
    for (int i = threadIdx.x; i < nvec; i += blockDim.x) {
      double c = cr[i];
      for (int k = 0; k < nvec; ++k) c -= gram_at(sc.Gm, m, i, k) * cr[k];
      sc.gcol[i] = c;
    }
    return;
  }
  (void)st;
  iter_finish<MODE == PJ_FIX>(sc, j, nvec, red);
  if (CTRL) DK_TL(TL_PROJECT, 5);
}

template <int MODE, int DEFL, bool AM>
static void project_t(const Dia& A, const Prolong& lab, const double* yc, const double* w_in,
                      double* w_out, const double* V, long long vstride, int nvec,
                      long long n_pad, double* part, int G, const Scal& sc, int j,
                      const int* gate, cudaStream_t s, bool pdl = true) {
  const int nq = (MODE == PJ_ITER || MODE == PJ_DOTS) ? 2 * nvec + 1
                 : (MODE == PJ_REDOTS) ? nvec : (MODE == PJ_FIX) ? nvec + 1 : 1;
  int slots = nq * kWarps > 3 * (sc.m + 1) ? nq * kWarps : 3 * (sc.m + 1);
  // PJ_ITER / PJ_FIX re-orthogonalisation test scratch (iter_finish)
  const int tail = 4 * nvec + 1 + (nvec <= kStageGram ? nvec * nvec : 0);
  if ((MODE == PJ_ITER || MODE == PJ_FIX) && tail > slots) slots = tail;
  if (nq + 260 > slots) slots = nq + 260;  // reduce_grouped scratch
  const size_t smem = (size_t)slots * sizeof(double);
  // one per instantiation and device: dynamic + 32 KB static > 48 KB default
  smem_optin((const void*)k_project<MODE, DEFL, AM>, 160 * 1024);
  if (!pdl) pdl_skip_next() = true;
  launch_pdl(k_project<MODE, DEFL, AM>, dim3(G), dim3(kThreads), smem, s, A, lab, yc, w_in,
             w_out, V, vstride, nvec, n_pad, part, G, sc, j, gate);
}

template <int MODE>
static void project_m(int defl, bool am, const Dia& A, const Prolong& lab, const double* yc,
                      const double* w_in, double* w_out, const double* V, long long vstride,
                      int nvec, long long n_pad, double* part, int G, const Scal& sc, int j,
                      const int* gate, cudaStream_t s) {
  if (defl == DK_NONE)
    project_t<MODE, DK_NONE, false>(A, lab, yc, w_in, w_out, V, vstride, nvec, n_pad, part, G,
                                    sc, j, gate, s);
  else if (defl == DK_DENSE)
    project_t<MODE, DK_DENSE, false>(A, lab, yc, w_in, w_out, V, vstride, nvec, n_pad, part, G,
                                     sc, j, gate, s);
  else if (am)
    project_t<MODE, DK_LABELS, true>(A, lab, yc, w_in, w_out, V, vstride, nvec, n_pad, part, G,
                                     sc, j, gate, s);
  else
    project_t<MODE, DK_LABELS, false>(A, lab, yc, w_in, w_out, V, vstride, nvec, n_pad, part, G,
                                      sc, j, gate, s);
}

void launch_project(int mode, int defl, bool am, const Dia& A, const Prolong& lab, const double* yc,
                    const double* w_in, double* w_out, const double* V, long long vstride,
                    int nvec, long long n_pad, double* part, int G, const Scal& sc, int j,
                    const int* gate, cudaStream_t s, bool pdl) {
  if (mode == PJ_DOTS) {
    project_t<PJ_DOTS, DK_NONE, false>(A, lab, yc, w_in, w_out, V, vstride, nvec, n_pad, part, G,
                                       sc, j, gate, s, pdl);
    return;
  }
  if (mode == PJ_FIX) {
    if (am)
      project_t<PJ_FIX, DK_LABELS, true>(A, lab, yc, w_in, w_out, V, vstride, nvec, n_pad, part,
                                         G, sc, j, gate, s, pdl);
    else
      project_t<PJ_FIX, DK_LABELS, false>(A, lab, yc, w_in, w_out, V, vstride, nvec, n_pad, part,
                                          G, sc, j, gate, s, pdl);
    return;
  }
  if (mode == PJ_ITER)
    project_m<PJ_ITER>(defl, am, A, lab, yc, w_in, w_out, V, vstride, nvec, n_pad, part, G, sc, j,
                       gate, s);
  else if (mode == PJ_RESTART)
    project_m<PJ_RESTART>(defl, am, A, lab, yc, w_in, w_out, V, vstride, nvec, n_pad, part, G, sc,
                          j, gate, s);
  else if (mode == PJ_REDOTS)
    project_t<PJ_REDOTS, DK_NONE, false>(A, lab, yc, w_in, w_out, V, vstride, nvec, n_pad, part,
                                         G, sc, j, gate, s);
  else
    project_m<PJ_PLAIN>(defl, am, A, lab, yc, w_in, w_out, V, vstride, nvec, n_pad, part, G, sc,
                        j, gate, s);
}

// ======================================================================================
// Dense deflation basis (RDGMRES harmonic-Ritz vectors, harmonic.py:97-180, or any n x d
// basis with d <= kDenseMaxD): s = Z^T v by the same (row, quarter-chunk) item sweep as the
// Arnoldi dots, y = E^-1 s in the last block; fixed order, deterministic.
// ======================================================================================
__global__ void __launch_bounds__(kThreads) k_zdots(const double* __restrict__ v,
                                                    const double* __restrict__ Z, long long zs,
                                                    int nz, long long n_pad,
                                                    double* __restrict__ part, int G,
                                                    unsigned int* ticket,
                                                    const double* __restrict__ Einv, int ld,
                                                    double* __restrict__ y, long long ystride,
                                                    const int* __restrict__ gate) {
  pdl_wait();
  if (gate != nullptr && *gate == 0) return;
  extern __shared__ double red[];  // [nz][kWarps], later s[nz]
  __shared__ __align__(16) double s_v[kChunk];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = threadIdx.x; q < nz * kWarps; q += blockDim.x) red[q] = 0.0;
  __syncthreads();
  const long long nchunks = n_pad / kChunk;
  double2* sv2 = reinterpret_cast<double2*>(s_v);
  for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const long long c0 = ch * kChunk;
#pragma unroll
    for (int k = 0; k < 4; ++k) sv2[threadIdx.x + 256 * k] = ld2(v + c0 + 2 * threadIdx.x + 512 * k);
    __syncthreads();
    for (int it = warp; it < 4 * nz; it += kWarps) {
      const int r = it >> 2, qtr = it & 3;
      const double* Zr = Z + (long long)r * zs + c0 + 512 * qtr + 2 * lane;
      double2 p[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = ld2(Zr + 64 * i);
      double a = 0.0;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const double2 vv = sv2[256 * qtr + lane + 32 * i];
        a = fma(p[i].x, vv.x, a);
        a = fma(p[i].y, vv.y, a);
      }
      a = warp_sum(a);
      if (lane == 0) red[r * kWarps + warp] += a;
    }
    __syncthreads();
  }
  pdl_trigger();
  for (int q = threadIdx.x; q < nz; q += blockDim.x) {
    double t = 0.0;
    for (int w2 = 0; w2 < kWarps; ++w2) t += red[q * kWarps + w2];
    part[(size_t)q * G + blockIdx.x] = t;
  }
  if (!last_block(ticket)) return;
  reduce_partials(part, nz, G, red);
  for (int i = threadIdx.x; i < nz; i += blockDim.x) {
    double t = red[i];
    if (Einv != nullptr) {
      t = 0.0;
      for (int k = 0; k < nz; ++k) t = fma(Einv[(size_t)i * ld + k], red[k], t);
    }
    y[(long long)i * ystride] = t;
  }
}

void launch_zdots(const double* v, const double* Z, long long zs, int nz, long long n_pad,
                  double* part, int G, unsigned int* ticket, const double* Einv, int ld,
                  double* y, long long ystride, const int* gate, cudaStream_t s) {
  const size_t smem = (size_t)(nz * kWarps > 64 ? nz * kWarps : 64) * sizeof(double);
  launch_pdl(k_zdots, dim3(G), dim3(kThreads), smem, s, v, Z, zs, nz, n_pad, part, G, ticket,
             Einv, ld, y, ystride, gate);
}

__global__ void k_dense_recon(const double* __restrict__ Z, long long zs, int nz,
                              const double* __restrict__ y, const double* __restrict__ xs,
                              const double* __restrict__ xh, double* __restrict__ out,
                              long long n_pad, int mode) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_pad;
       i += (long long)gridDim.x * blockDim.x) {
    double zy = 0.0;
    for (int q = 0; q < nz; ++q) zy = fma(__ldg(y + q), Z[(long long)q * zs + i], zy);
    if (mode == 0) out[i] = __dadd_rn(xs[i], __dsub_rn(xh[i], zy));  // x* + (xh - Z y)
    else if (mode == 1) out[i] = zy;                                  // Z y
    else out[i] = __dsub_rn(xh[i], zy);                               // v - Z y
  }
}

void launch_dense_recon(const double* Z, long long zs, int nz, const double* y, const double* xs,
                        const double* xh, double* out, long long n_pad, int mode,
                        cudaStream_t s) {
  k_dense_recon<<<num_sms() * 8, kThreads, 0, s>>>(Z, zs, nz, y, xs, xh, out, n_pad, mode);
}

// out_j = sum_i Y[i + j nrows] sigma_i R_i, eight outputs per sweep over the rows
__global__ void __launch_bounds__(kThreads) k_combine_rows(const double* __restrict__ R,
                                                           long long rs,
                                                           const double* __restrict__ sigma,
                                                           int nrows,
                                                           const double* __restrict__ Y,
                                                           int nout, double* __restrict__ out,
                                                           long long os, long long n_pad) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_pad;
       i += (long long)gridDim.x * blockDim.x) {
    for (int j0 = 0; j0 < nout; j0 += 8) {
      double acc[8];
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) acc[jj] = 0.0;
      for (int r = 0; r < nrows; ++r) {
        const double v = __ldg(sigma + r) * R[(long long)r * rs + i];
#pragma unroll
        for (int jj = 0; jj < 8; ++jj)
          if (j0 + jj < nout) acc[jj] = fma(__ldg(Y + r + (long long)(j0 + jj) * nrows), v, acc[jj]);
      }
#pragma unroll
      for (int jj = 0; jj < 8; ++jj)
        if (j0 + jj < nout) out[(long long)(j0 + jj) * os + i] = acc[jj];
    }
  }
}

void launch_combine_rows(const double* R, long long rs, const double* sigma, int nrows,
                         const double* Y, int nout, double* out, long long os, long long n_pad,
                         cudaStream_t s) {
  k_combine_rows<<<num_sms() * 8, kThreads, 0, s>>>(R, rs, sigma, nrows, Y, nout, out, os, n_pad);
}

// ======================================================================================
// K5: classical Gram-Schmidt update u = w - sum_i h_i V_i with ||u||^2, one sweep over V.
// REORTH: the second pass u -= sum_i corr_i V_i (only when the test in K4 fired; corr is
// then recomputed from the stored u by a PJ_REDOTS sweep, as the reference does).
// ======================================================================================
// Grid-wide release of the fused second pass: every block arrives; the last one runs `lead`
// (all its threads), then releases the others, which spin on the generation counter.  Only
// used when the whole grid is co-resident (checked on the host) and no dependent launch was
// triggered, so nothing can hold the SMs the waiting blocks need.
template <class F>
__device__ __forceinline__ void grid_arrive_lead_release(unsigned int* count, unsigned int* gen,
                                                         F lead) {
  __shared__ int s_lead;
  __shared__ unsigned int s_gen;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    s_gen = *reinterpret_cast<volatile unsigned int*>(gen);
    __threadfence();
    s_lead = (atomicAdd(count, 1u) == gridDim.x - 1) ? 1 : 0;
  }
  __syncthreads();
  if (s_lead) {
    __threadfence();
    lead();
    __syncthreads();
    if (threadIdx.x == 0) {
      *count = 0u;
      __threadfence();
      atomicAdd(gen, 1u);
    }
  } else if (threadIdx.x == 0) {
    while (*reinterpret_cast<volatile unsigned int*>(gen) == s_gen) __nanosleep(64);
    __threadfence();
  }
  __syncthreads();
}

// K5 (FUSE): when the projection's test fired (rare), the reference's second Gram-Schmidt
// pass (krylov.py:169-170) runs inside the same launch — corr = V^T u over the stored u,
// the coefficients in the leading block, u -= V corr — instead of two extra launches that
// are otherwise issued gated-off every iteration.
#ifndef DK_EARLY_ROWS
#define DK_EARLY_ROWS 4
#endif
constexpr int kEarlyRows = DK_EARLY_ROWS;  // basis rows k_gs prefetches while it waits

template <bool REORTH>
__global__ void __launch_bounds__(kThreads) k_gs(const double* w_in, double* u_out,
                                                 const double* __restrict__ V, long long vstride,
                                                 int nvec, long long n_pad,
                                                 double* __restrict__ part, int G, Scal sc, int j,
                                                 const int* __restrict__ gate, int fuse,
                                                 const unsigned* wait) {
  if (!REORTH) DK_TL(TL_GS, 0);
  // early start (wait != nullptr): on the projection's published coefficients; its
  // re-orthogonalisation verdict is read after its completion (griddepcontrol.wait below)
  if (wait != nullptr) {
    // the basis rows are final: the first ones of this block's chunk into L2 while waiting
    if (gridDim.x * (long long)kChunk >= n_pad && threadIdx.x < kEarlyRows &&
        (int)threadIdx.x < nvec)
      l2_prefetch(V + (long long)threadIdx.x * vstride + (long long)blockIdx.x * kChunk,
                  kChunk * 8);
    if (!early_start(wait, gate, (unsigned)sc.ng)) return;
  } else {
    pdl_wait();
    if (*gate == 0) return;
  }
  if (!REORTH) DK_TL(TL_GS, 1);
  extern __shared__ double sh[];
  double* cf = sh;                                  // [nvec]
  double* red = sh + nvec;                          // [kWarps] (+ scratch)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (!REORTH && wait != nullptr) {
    // the projection's coefficients, as its last block forms them, from its group partials
    double* gp = red;  // nvec x ng staged (red is free until the sweep's partial sums)
    for (int e = threadIdx.x; e < nvec * sc.ng; e += blockDim.x) gp[e] = __ldcg(sc.gpart + e);
    __syncthreads();
    for (int q = threadIdx.x; q < nvec; q += blockDim.x) {
      const double sv = __ldcg(sc.sigma + q);
      const double t = grouped_total(gp, q, sc.ng, false);
      // iter_finish's h_i (split: sigma_i h'_i - (C y)_i), times sigma_i
      cf[q] = (sc.split ? split_h(sc, q, t) : t * sv) * sv;
    }
    __syncthreads();
  } else {
    for (int q = threadIdx.x; q < nvec; q += blockDim.x) cf[q] = REORTH ? sc.corr[q] : sc.coef[q];
  }
  for (int q = threadIdx.x; q < kWarps; q += blockDim.x) red[q] = 0.0;
  __syncthreads();
  const long long nchunks = n_pad / kChunk;
  const unsigned long long pol = l2_evict_first();
  for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const long long cb = ch * kChunk + 2 * threadIdx.x;
    double u[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double2 x = REORTH ? ld2cg(w_in + cb + 512 * k) : ld2_vec(w_in + cb + 512 * k);
      u[2 * k] = x.x;
      u[2 * k + 1] = x.y;
    }
#pragma unroll 8
    for (int v = 0; v < nvec; ++v) {
      const double* Vr = V + (long long)v * vstride + cb;
      const double c = cf[v];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double2 p = ld2_stream(Vr + 512 * k, pol);
        u[2 * k] = __dsub_rn(u[2 * k], __dmul_rn(c, p.x));
        u[2 * k + 1] = __dsub_rn(u[2 * k + 1], __dmul_rn(c, p.y));
      }
    }
    double nrm = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      st2_vec(u_out + cb + 512 * k, make_double2(u[2 * k], u[2 * k + 1]));
      nrm = fma(u[2 * k], u[2 * k], nrm);
      nrm = fma(u[2 * k + 1], u[2 * k + 1], nrm);
    }
    nrm = warp_sum(nrm);
    if (lane == 0) red[warp] += nrm;
  }
  if (!REORTH) DK_TL(TL_GS, 3);
  if (wait != nullptr) pdl_wait();
  const bool second =
      !REORTH && fuse && *reinterpret_cast<const volatile int*>(&sc.st->reorth) != 0;
  if (second) {
    // corr_v = V_v . u: block partials over this block's chunks (u re-read from its own writes)
    __syncthreads();
    for (int v = 0; v < nvec; ++v) {
      double a = 0.0;
      for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
        const long long cb = ch * kChunk + 2 * threadIdx.x;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double2 uu = ld2cg(u_out + cb + 512 * k);
          const double2 p = ld2_stream(V + (long long)v * vstride + cb + 512 * k, pol);
          a = fma(p.x, uu.x, a);
          a = fma(p.y, uu.y, a);
        }
      }
      a = warp_sum(a);
      if (lane == 0) red[warp] = a;
      __syncthreads();
      if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w2 = 0; w2 < kWarps; ++w2) t += red[w2];
        part[(size_t)v * G + blockIdx.x] = t;
      }
      __syncthreads();
    }
    grid_arrive_lead_release(sc.gticket + kGroupTickets - 2, sc.gticket + kGroupTickets - 3, [&] {
      // the PJ_REDOTS finish: H column += corr, coefficients, next Gram column corr - G corr
      const int m = sc.m;
      double* Hc = sc.H + (size_t)j * (m + 1);
      double* cr = red;
      for (int v = warp; v < nvec; v += kWarps) {
        double t = 0.0;
        for (int b = lane; b < G; b += 32) t += __ldcg(part + (size_t)v * G + b);
        t = warp_sum(t);
        if (lane == 0) cr[v] = t * sc.sigma[v];
      }
      __syncthreads();
      for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
        Hc[v] += cr[v];
        sc.corr[v] = cr[v] * sc.sigma[v];
      }
      for (int i = threadIdx.x; i < nvec; i += blockDim.x) {
        double c = cr[i];
        for (int k = 0; k < nvec; ++k) c -= gram_at(sc.Gm, m, i, k) * cr[k];
        sc.gcol[i] = c;
      }
    });
    // u -= V corr, new norm
    for (int q = threadIdx.x; q < nvec; q += blockDim.x) cf[q] = __ldcg(sc.corr + q);
    for (int q = threadIdx.x; q < kWarps; q += blockDim.x) red[q] = 0.0;
    __syncthreads();
    for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
      const long long cb = ch * kChunk + 2 * threadIdx.x;
      double u[8];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const double2 x = ld2cg(u_out + cb + 512 * k);
        u[2 * k] = x.x;
        u[2 * k + 1] = x.y;
      }
      for (int v = 0; v < nvec; ++v) {
        const double c = cf[v];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double2 p = ld2_stream(V + (long long)v * vstride + cb + 512 * k, pol);
          u[2 * k] = __dsub_rn(u[2 * k], __dmul_rn(c, p.x));
          u[2 * k + 1] = __dsub_rn(u[2 * k + 1], __dmul_rn(c, p.y));
        }
      }
      double nrm = 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        st2(u_out + cb + 512 * k, make_double2(u[2 * k], u[2 * k + 1]));
        nrm = fma(u[2 * k], u[2 * k], nrm);
        nrm = fma(u[2 * k + 1], u[2 * k + 1], nrm);
      }
      nrm = warp_sum(nrm);
      if (lane == 0) red[warp] += nrm;
    }
  } else {
    pdl_trigger();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w2 = 0; w2 < kWarps; ++w2) s += red[w2];
    part[blockIdx.x] = s;
  }
  const bool early = !REORTH && sc.post != nullptr;  // the next stencil forms sigma itself
  if (!reduce_grouped(part, 1, G, sc.gticket, early ? sc.gpart_gs : sc.gpart, red,
                      early ? sc.post + j : nullptr)) {
    if (!REORTH) DK_TL(TL_GS, 4);
    return;
  }
  const double hj1 = sqrt(red[0]);
  __syncthreads();
  if (!REORTH && !second && sc.st->reorth) return;  // the separate second pass finishes it
  finish_iteration_block(sc, j, hj1, red);
  if (!REORTH) DK_TL(TL_GS, 5);
}

// ======================================================================================
// Small problems (one 2048-cell chunk per block, the basis L2-resident: BASELINE config 1):
// the cycle's m Arnoldi steps run in ONE persistent, co-resident (cooperative) grid instead of
// 5 launches per step, each of which is pure latency at this size.  Per step j:
//   stencil w = A M^-1 (sigma_j u_j) of the block's chunk (kept in registers) + its run sums
//   | lead: s = Z^T w (warp per column, runs in order), y = E^-1 s (dense E^-1, d <= 64)
//   w -= A_p Z y (compact prolongation, y in shared memory); block partials of U^T w, the
//   Gram column U^T u_j and ||w||^2
//   | lead: reduction + iter_finish (H column, coefficients, re-orthogonalisation test)
//   u = w - U coef (+ the second pass through one more lead when the test fired), stored
//   as basis row j+1; block partial of ||u||^2
//   | lead: finish_iteration_block (Givens, convergence, breakdown, sigma_{j+1})
// "|" is grid_arrive_lead_release: the last block to arrive runs the control section (the
// same device functions as the multi-kernel path) before releasing the others.  Block-local
// sums run in fixed order; results agree with the multi-kernel path to rounding (parity
// against the reference is the bar; the path is chosen by shape, DK_NO_SMALL disables it).
// ======================================================================================
constexpr int kSmallMaxD = 64;
constexpr int kSmallRuns = 32;  // label runs per warp and cell slot (at most one per lane)

template <bool AM>
__device__ __forceinline__ double prolong_cell_smem(const Dia& A, const Prolong& P,
                                                    const double* ys, long long c) {
  const int L = P.lab[c];
  const double own = P.own[c];
  const int2 fl = P.flab[c];
  const double2 fc = P.fco[c];
  const unsigned msk = P.mask[c];
  double t = (L >= 0) ? __dmul_rn(own, ys[L]) : 0.0;
  if (fl.x >= 0) t = __dadd_rn(t, __dmul_rn(fc.x, ys[fl.x]));
  if (fl.y >= 0) t = __dadd_rn(t, __dmul_rn(fc.y, ys[fl.y]));
  if (msk) {
#pragma unroll
    for (int q = 0; q < kMaxDiag; ++q) {
      if (!((msk >> q) & 1u)) continue;
      const long long o = A.off[q];
      double a = dia_coef(A, q, c);
      if (AM) a = __dmul_rn(a, __ldg(A.inv + c + o));
      t = __dadd_rn(t, __dmul_rn(a, ys[__ldg(P.lab + c + o)]));
    }
  }
  return t;
}

// 32 per-lane values -> lane l holds the warp sum of value l (fixed butterfly: deterministic)
__device__ __forceinline__ double small_transpose_sum(double (&v)[32], int lane) {
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

// out[q] = sum over the blocks of part[q * G + b] (G <= 160): each warp takes 8 quantities at
// a time, lane l sums blocks l, l + 32, ... in order with all 40 loads issued first, reduce8's
// fixed butterfly combines the lanes (deterministic)
__device__ __forceinline__ void small_reduce(const double* part, int nq, double* out) {
  const int G = gridDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q0 = 8 * warp; q0 < nq; q0 += 8 * kWarps) {
    double a[8][5];
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
      for (int i = 0; i < 5; ++i) {
        const bool on = q0 + k < nq && lane + 32 * i < G;
        const double* p = part + (size_t)(on ? q0 + k : 0) * G + (on ? lane + 32 * i : 0);
        a[k][i] = on ? __ldcg(p) : 0.0;
      }
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double t = 0.0;
#pragma unroll
      for (int i = 0; i < 5; ++i) t += a[k][i];
      v[k] = t;
    }
    const double r = reduce8(v, lane);
    if ((lane & 3) == 0 && q0 + (lane >> 2) < nq) out[q0 + (lane >> 2)] = r;
  }
  __syncthreads();
}

// Grid barrier of the persistent small-cycle grid: thread 0 of each block arrives with an
// acq_rel atomic (release is cumulative over the block's writes ordered by the preceding
// __syncthreads); the last to arrive runs lead() with the whole block, then releases the
// others with a release store of the generation they poll with acquire loads.
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
template <class F>
__device__ __forceinline__ void small_barrier(unsigned* count, unsigned* gen, F lead) {
  __shared__ int s_lead;
  __shared__ unsigned s_gen;
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = ld_acquire_u32(gen);
    s_gen = g;
    s_lead = (atom_add_acq_rel(count, 1u) == gridDim.x - 1) ? 1 : 0;
  }
  __syncthreads();
  if (s_lead) {
    DK_TL(TL_SMALL, 7);
    lead();
    __syncthreads();
    DK_TL(TL_SMALL, 8);
    if (threadIdx.x == 0) {
      *reinterpret_cast<volatile unsigned*>(count) = 0u;
      st_release_u32(gen, s_gen + 1u);
    }
  } else if (threadIdx.x == 0) {
    while (*reinterpret_cast<volatile unsigned*>(gen) == s_gen) __nanosleep(20);
    (void)ld_acquire_u32(gen);  // acquire once the release is seen
  }
  __syncthreads();
}

// Block partials of nq <= 128 quantities (thread values vals(q)) to part[q * G + b]: batches
// of 32 transposed-summed within the warp, then the warps in order.
template <class F>
__device__ __forceinline__ void small_partials(int nq, double* red, double* part, F vals) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q0 = 0; q0 < nq; q0 += 32) {
    double v[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) v[k] = (q0 + k < nq) ? vals(q0 + k) : 0.0;
    const double t = small_transpose_sum(v, lane);
    if (q0 + lane < nq) red[(q0 + lane) * kWarps + warp] = t;
  }
  __syncthreads();
  for (int q = threadIdx.x; q < nq; q += blockDim.x) {
    double t = 0.0;
    for (int w2 = 0; w2 < kWarps; ++w2) t += red[q * kWarps + w2];
    __stcg(part + (size_t)q * gridDim.x + blockIdx.x, t);
  }
  __syncthreads();
}

// Plain grid barrier of the small-cycle grid: a per-launch arrival counter (zeroed before
// the launch); barrier k waits for (k + 1) G arrivals.  Release-add to arrive (cumulative
// over the block's writes ordered by __syncthreads), relaxed polling, one acquire.
__device__ __forceinline__ void red_add_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void small_sync(unsigned* counter, unsigned& target) {
  target += gridDim.x;
  __syncthreads();
  if (threadIdx.x == 0) {
    red_add_release(counter, 1u);
    while (ld_relaxed_u32(counter) < target) __nanosleep(20);
    (void)ld_acquire_u32(counter);
  }
  __syncthreads();
}

// ======================================================================================
// Small problems (BASELINE config 1: 32 k cells, the whole basis L2-resident): the cycle's m
// Arnoldi steps in ONE persistent cooperative grid over all SMs, CPT cells per thread
// (consecutive threads own consecutive cells), instead of 5 latency-bound launches per step.
// Per step j:
//   w = A M^-1 (sigma_j u_j) (k_stencil's arithmetic), kept in registers; per-block label
//   sums of w (warp-segmented runs of consecutive cells, fixed trees)          | barrier
//   s = Z^T w, y = E^-1 s in every block; w -= A_p Z y; block partials of U^T w, of the Gram
//   column U^T u_j and of ||w||^2                                                | barrier
//   the H column and the re-orthogonalisation test (iter_finish's arithmetic) in every
//   block; u = w - U coef (+ the second pass when the test fired), stored as basis row j+1;
//   block partial of ||u||^2                                                     | barrier
//   Givens, convergence / breakdown, sigma_{j+1} (finish_iteration_block's arithmetic)
// The control state (sigma, cs, sn, the Gram matrix, the residual estimate, the counters) is
// replicated in every block's shared memory — the blocks compute identical values from the
// same partials in the same order — so no block waits for another's control section; block
// 0 alone writes the solver's device state, exactly what the multi-kernel path writes.
// Chosen by shape (cycle_small_ok); DK_NO_SMALL disables it.
// ======================================================================================
template <int DEFL, bool PRE, bool AM, int CPT>
__global__ void __launch_bounds__(kThreads, 1) k_cycle_small(Dia A, Dia Aam, Prolong P,
                                                          const int* __restrict__ lab, int d,
                                                          const double* __restrict__ Einv,
                                                          int ld, double* V, long long vstride,
                                                          long long n_pad, double* part,
                                                          unsigned* counter, Scal sc) {
  extern __shared__ __align__(16) double sm[];
  const int m = sc.m, M1 = m + 1;
  double* gm = sm;                   // (m+1)^2 Gram matrix, full
  double* tot = gm + M1 * M1;        // reduced quantities (2 M1 + 1)
  double* red = tot + 2 * M1 + 8;    // [q][warp] block partial staging (2 M1 + 33)
  __shared__ double ys[kSmallMaxD], sdv[kSmallMaxD];
  __shared__ double sig[kMaxCycleSmall + 1], csv[kMaxCycleSmall], snv[kMaxCycleSmall];
  __shared__ double hcol[kMaxCycleSmall + 1], cf[kMaxCycleSmall], absc[kMaxCycleSmall];
  __shared__ double rsum[kWarps][CPT][kSmallRuns];
  __shared__ int rlab[kWarps][CPT][kSmallRuns];
  __shared__ int rcnt[kWarps][CPT];
  __shared__ double s_gcur, s_tol, s_denom;
  __shared__ int s_its, s_min, s_max, s_cycle, s_active, s_reorth, s_broke, s_final;
  __shared__ double s_hn;
  State* st = sc.st;
  const bool w0 = blockIdx.x == 0;  // the writer of the device state
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long cell[CPT];
  bool ok[CPT];
#pragma unroll
  for (int e = 0; e < CPT; ++e) {
    cell[e] = (long long)blockIdx.x * blockDim.x + threadIdx.x + e * stride;
    ok[e] = cell[e] < n_pad;
    if (!ok[e]) cell[e] = 0;  // a padded slot: reads stay in bounds, results unused
  }
  int L[CPT];
#pragma unroll
  for (int e = 0; e < CPT; ++e) L[e] = (DEFL == DK_LABELS && ok[e]) ? __ldg(lab + cell[e]) : -1;
  unsigned target = 0;
#ifdef DK_TIMELINE
  unsigned long long tacc[24] = {0}, tprev = 0;
  auto tmark = [&](int k) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (k > 0) tacc[k] += t - tprev;
    tprev = t;
  };
#define SMALL_MARK(k) \
  if (blockIdx.x == 0 && threadIdx.x == 0) tmark(k)
#else
#define SMALL_MARK(k)
#endif
  pdl_wait();
  if (threadIdx.x == 0) {  // the restart's state (written before this launch)
    s_active = st->active;
    s_its = st->iterations;
    s_tol = st->tol;
    s_denom = st->denom;
    s_min = st->min_iters;
    s_max = st->max_iters;
    s_cycle = st->cycle;
    s_gcur = sc.g[0];
    sig[0] = sc.sigma[0];
  }
  if (threadIdx.x == 0) s_final = s_active;
  __syncthreads();
  for (int j = 0; j < m && s_active; ++j) {
    SMALL_MARK(0);
    const int nvec = j + 1;
    const double sgj = sig[j];
    const double* vj = V + (long long)j * vstride;
    // ---- stencil: every coefficient and neighbour in flight, then the ordered sums
    double w[CPT];
#pragma unroll
    for (int e = 0; e < CPT; ++e) {
      const long long c = cell[e];
      double a[kMaxDiag], x[kMaxDiag], mi[kMaxDiag];
#pragma unroll
      for (int q = 0; q < kMaxDiag; ++q) {
        const bool on = q < A.ndiag;
        const long long o = on ? A.off[q] : 0;
        a[q] = on ? dia_coef(A, q, c) : 0.0;
        x[q] = on ? __ldcg(vj + c + o) : 0.0;
        mi[q] = (on && PRE) ? __ldg(A.inv + c + o) : 1.0;
      }
      double r = 0.0;
#pragma unroll
      for (int q = 0; q < kMaxDiag; ++q) {
        if (q >= A.ndiag) break;
        double y = __dmul_rn(x[q], sgj);
        if (PRE) y = __dmul_rn(y, mi[q]);
        r = __dadd_rn(r, __dmul_rn(a[q], y));
      }
      w[e] = ok[e] ? r : 0.0;
    }
    if (DEFL == DK_LABELS) {
      // warp-segmented label runs of consecutive cells: inclusive segmented scan, the run's
      // last lane records (label, sum)
#pragma unroll
      for (int e = 0; e < CPT; ++e) {
        const int Lp = __shfl_up_sync(0xffffffffu, L[e], 1);
        const bool head = lane == 0 || Lp != L[e];
        double v = L[e] >= 0 ? w[e] : 0.0;
        const unsigned hm = __ballot_sync(0xffffffffu, head);
        const int seg_start = 31 - __clz(hm & ((2u << lane) - 1u));
#pragma unroll
        for (int dlt = 1; dlt < 32; dlt <<= 1) {
          const double u = __shfl_up_sync(0xffffffffu, v, dlt);
          if (lane >= dlt && lane - dlt >= seg_start) v = __dadd_rn(u, v);
        }
        const bool tail = lane == 31 || ((hm >> (lane + 1)) & 1u);
        const unsigned tm = __ballot_sync(0xffffffffu, tail && L[e] >= 0);
        if (lane == 0) rcnt[warp][e] = __popc(tm);
        if (tail && L[e] >= 0) {
          const int k = __popc(tm & ((1u << lane) - 1u));
          rsum[warp][e][k] = v;
          rlab[warp][e][k] = L[e];
        }
      }
      __syncthreads();
      if (!s_final) break;  // the previous step's convergence test (speculative stencil)
      // block partial of label l: the runs in (warp, slot, run) order
      for (int l = threadIdx.x; l < d; l += blockDim.x) {
        double t = 0.0;
        for (int w2 = 0; w2 < kWarps; ++w2)
#pragma unroll
          for (int e = 0; e < CPT; ++e) {
            const int nr = rcnt[w2][e];
            for (int k = 0; k < nr; ++k)
              if (rlab[w2][e][k] == l) t += rsum[w2][e][k];
          }
        __stcg(part + (size_t)l * gridDim.x + blockIdx.x, t);
      }
      SMALL_MARK(1);
      small_sync(counter, target);
      SMALL_MARK(2);
      // ---- s = Z^T w (blocks in order), y = E^-1 s: every block
      small_reduce(part, d, sdv);
      SMALL_MARK(3);
      for (int l = threadIdx.x; l < d; l += blockDim.x) {
        const double* Er = Einv + (long long)l * ld;
        double t = 0.0;
        int k = 0;
        for (; k + 8 <= d; k += 8) {  // the row's loads in flight, then the ordered sum
          double e8[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) e8[u] = __ldg(Er + k + u);
#pragma unroll
          for (int u = 0; u < 8; ++u) t = fma(e8[u], sdv[k + u], t);
        }
        for (; k < d; ++k) t = fma(__ldg(Er + k), sdv[k], t);
        ys[l] = t;
      }
      __syncthreads();
      SMALL_MARK(4);
#pragma unroll
      for (int e = 0; e < CPT; ++e)
        if (ok[e]) w[e] = __dsub_rn(w[e], prolong_cell_smem<AM>(Aam, P, ys, cell[e]));
    }
    if (DEFL != DK_LABELS) {
      __syncthreads();
      if (!s_final) break;  // the previous step's convergence test (speculative stencil)
    }
    // ---- block partials: U^T w, U^T u_j, ||w||^2
    double uj[CPT];
#pragma unroll
    for (int e = 0; e < CPT; ++e) uj[e] = __ldcg(vj + cell[e]);
    SMALL_MARK(5);
    {
      // batches of 32 basis rows: every load of the batch in flight, each row serving both
      // dots (U_v . w and the Gram entry U_v . u_j); quantity v, nvec + v; ||w||^2 last
      const int nq = 2 * nvec + 1;
      for (int v0 = 0; v0 < nvec; v0 += 32) {
        double pv[32][CPT];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const bool on = v0 + k < nvec;
          const double* Vr = V + (long long)(on ? v0 + k : 0) * vstride;
#pragma unroll
          for (int e = 0; e < CPT; ++e) pv[k][e] = on ? __ldcg(Vr + cell[e]) : 0.0;
        }
        double hv[32], gv[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          double th = 0.0, tg = 0.0;
#pragma unroll
          for (int e = 0; e < CPT; ++e) {
            th = fma(pv[k][e], w[e], th);
            tg = fma(pv[k][e], uj[e], tg);
          }
          hv[k] = th;
          gv[k] = tg;
        }
        const double th = small_transpose_sum(hv, lane);
        const double tg = small_transpose_sum(gv, lane);
        if (v0 + lane < nvec) {
          red[(v0 + lane) * kWarps + warp] = th;
          red[(nvec + v0 + lane) * kWarps + warp] = tg;
        }
      }
      {
        double t = 0.0;
#pragma unroll
        for (int e = 0; e < CPT; ++e) t = fma(w[e], w[e], t);
        t = warp_sum(t);
        if (lane == 0) red[(2 * nvec) * kWarps + warp] = t;
      }
      __syncthreads();
      for (int q = threadIdx.x; q < nq; q += blockDim.x) {
        double t = 0.0;
        for (int w2 = 0; w2 < kWarps; ++w2) t += red[q * kWarps + w2];
        __stcg(part + (size_t)q * gridDim.x + blockIdx.x, t);
      }
      __syncthreads();
    }
    SMALL_MARK(6);
    small_sync(counter, target);
    SMALL_MARK(7);
    // ---- the H column and the re-orthogonalisation test (iter_finish's arithmetic)
    small_reduce(part, 2 * nvec + 1, tot);
    SMALL_MARK(13);
    for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
      const double h = tot[v] * sig[v];  // h_i = V_i . w  (krylov.py:164-165)
      hcol[v] = h;
      cf[v] = h * sig[v];
      const double g = tot[nvec + v] * sig[v] * sgj;  // V_i . V_j
      gm[v * M1 + j] = g;
      gm[j * M1 + v] = g;
      if (w0) {
        sc.H[(size_t)j * M1 + v] = h;
        sc.coef[v] = cf[v];
        sc.Gm[(size_t)j * M1 + v] = g;
      }
    }
    __syncthreads();
    SMALL_MARK(14);
    for (int i = threadIdx.x; i < nvec; i += blockDim.x) {  // corr_i = h_i - sum_k G_ik h_k
      double c4[4] = {0.0, 0.0, 0.0, 0.0};  // four interleaved chains, fixed combination
      int k = 0;
      for (; k + 4 <= nvec; k += 4)
#pragma unroll
        for (int u = 0; u < 4; ++u) c4[u] = fma(gm[i * M1 + k + u], hcol[k + u], c4[u]);
      for (; k < nvec; ++k) c4[0] = fma(gm[i * M1 + k], hcol[k], c4[0]);
      const double c = hcol[i] - ((c4[0] + c4[1]) + (c4[2] + c4[3]));
      absc[i] = fabs(c);
      if (w0) sc.gcol[i] = c;
    }
    __syncthreads();
    SMALL_MARK(15);
    if (threadIdx.x < 32) {  // max |corr| (order-free)
      double mx = 0.0;
      for (int i = threadIdx.x; i < nvec; i += 32) mx = fmax(mx, absc[i]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (threadIdx.x == 0) absc[kMaxCycleSmall - 1] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const double wnorm0 = sqrt(tot[2 * nvec]);  // krylov.py:162
      const double mx = absc[kMaxCycleSmall - 1];
      s_reorth = mx > 1e-8 * fmax(wnorm0, 1e-300);  // krylov.py:168
      if (w0) {
        st->wnorm0 = wnorm0;
        st->reorth = s_reorth;
        if (s_reorth) st->reorths += 1;
      }
    }
    __syncthreads();
    SMALL_MARK(8);
    // ---- u = w - U coef
    double u[CPT];
#pragma unroll
    for (int e = 0; e < CPT; ++e) u[e] = w[e];
#pragma unroll 8
    for (int v = 0; v < nvec; ++v) {
      const double c = cf[v];
      const double* Vr = V + (long long)v * vstride;
#pragma unroll
      for (int e = 0; e < CPT; ++e) u[e] = __dsub_rn(u[e], __dmul_rn(c, __ldcg(Vr + cell[e])));
    }
    if (s_reorth) {
      // the second Gram-Schmidt pass (krylov.py:169-170): corr = V^T u, u -= V corr
      small_partials(nvec, red, part, [&](int v) {
        double t = 0.0;
        const double* Vr = V + (long long)v * vstride;
#pragma unroll
        for (int e = 0; e < CPT; ++e) t = fma(__ldcg(Vr + cell[e]), u[e], t);
        return t;
      });
      small_sync(counter, target);
      small_reduce(part, nvec, tot);
      for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
        const double cr = tot[v] * sig[v];
        hcol[v] += cr;
        cf[v] = cr * sig[v];
        absc[v] = cr;
        if (w0) {
          sc.H[(size_t)j * M1 + v] = hcol[v];
          sc.corr[v] = cf[v];
        }
      }
      __syncthreads();
      if (w0)
        for (int i = threadIdx.x; i < nvec; i += blockDim.x) {
          double c = absc[i];
          for (int k = 0; k < nvec; ++k) c -= gm[i * M1 + k] * absc[k];
          sc.gcol[i] = c;
        }
#pragma unroll 8
      for (int v = 0; v < nvec; ++v) {
        const double c = cf[v];
        const double* Vr = V + (long long)v * vstride;
#pragma unroll
        for (int e = 0; e < CPT; ++e) u[e] = __dsub_rn(u[e], __dmul_rn(c, __ldcg(Vr + cell[e])));
      }
    }
    double* un = V + (long long)(j + 1) * vstride;
#pragma unroll
    for (int e = 0; e < CPT; ++e)
      if (ok[e]) un[cell[e]] = u[e];
    SMALL_MARK(9);
    small_partials(1, red, part, [&](int) {
      double t = 0.0;
#pragma unroll
      for (int e = 0; e < CPT; ++e) t = fma(u[e], u[e], t);
      return t;
    });
    SMALL_MARK(10);
    small_sync(counter, target);
    SMALL_MARK(11);
    // ---- Givens, convergence / breakdown, sigma_{j+1} (finish_iteration_block's arithmetic).
    // The breakdown test and sigma_{j+1} come first; the block then starts the next step's
    // stencil while thread 0 finishes the rotations and the convergence test, which the next
    // step checks before its first global write (the same decision in every block).
    small_reduce(part, 1, tot);
    SMALL_MARK(16);
    if (threadIdx.x < 32) {  // |H column| for the breakdown test (warp 0)
      const double hj1 = sqrt(tot[0]);
      double hn = 0.0;
      for (int i = threadIdx.x; i <= j; i += 32) hn = fma(hcol[i], hcol[i], hn);
      hn = warp_sum(hn);
      if (threadIdx.x == 0) {
        hn = sqrt(fma(hj1, hj1, hn));
        s_hn = hn;
        absc[j + 1] = hj1;
        s_broke = hj1 <= 1e-13 * fmax(1.0, hn);  // :192-194 (convergence is tested first)
        if (!s_broke) sig[j + 1] = 1.0 / hj1;     // V[j+1] = w / hj1 (:197)
        s_active = !s_broke && j + 1 < m && s_its + 1 < s_max;  // provisional
      }
    }
    __syncthreads();
    SMALL_MARK(17);
    if (threadIdx.x == 0) {
      const double hj1 = absc[j + 1];
      double* col = absc;  // the rotated column (j + 2 <= kMaxCycleSmall)
      double run = hcol[0];  // the rotated entry carried in a register
      for (int i = 0; i < j; ++i) {  // _givens_update, krylov.py:90-104
        const double nx = hcol[i + 1];
        const double t = __dadd_rn(__dmul_rn(csv[i], run), __dmul_rn(snv[i], nx));
        run = __dadd_rn(__dmul_rn(-snv[i], run), __dmul_rn(csv[i], nx));
        col[i] = t;
      }
      col[j] = run;
      const double den = hypot(col[j], col[j + 1]);
      double c = 1.0, sn = 0.0;
      if (den != 0.0) {
        c = col[j] / den;
        sn = col[j + 1] / den;
      }
      csv[j] = c;
      snv[j] = sn;
      col[j] = den;
      col[j + 1] = 0.0;
      const double gj = s_gcur;
      const double gn = __dmul_rn(-sn, gj);
      const double resnorm = fabs(gn);
      s_gcur = gn;
      s_its += 1;
      int active = 1, converged = 0, broke = 0, warn = 0;
      if (resnorm <= s_tol * s_denom && s_its >= s_min) {  // :189-191
        converged = 1;
        active = 0;
        broke = 1;
      } else if (s_broke) {  // :192-194
        warn = 1;
        active = 0;
        broke = 1;
      } else if (j + 1 >= m || s_its >= s_max) {
        active = 0;
      }
      if (w0) {
        sc.H[(size_t)j * M1 + j + 1] = hj1;  // krylov.py:172
        sc.cs[j] = c;
        sc.sn[j] = sn;
        sc.g[j + 1] = gn;
        sc.g[j] = __dmul_rn(c, gj);
        st->cols = j + 1;
        st->iterations = s_its;
        sc.hist[s_its] = resnorm;
        sc.restart_of[s_its] = s_cycle;
        st->reorth = 0;
        st->last_broke = broke;
        if (converged) st->converged = 1;
        if (warn) st->warning = DK_WARNING_BREAKDOWN;
        if (!broke) sc.sigma[j + 1] = sig[j + 1];
        if (!active) st->active = 0;
      }
      s_final = active;
    }
    if (w0 && threadIdx.x < 32) {  // the rotated column (warp 0, after its lane 0 formed it)
      __syncwarp();
      double* Rc = sc.R + (size_t)j * M1;
      for (int i = threadIdx.x; i <= j + 1; i += 32) Rc[i] = absc[i];
    }
    SMALL_MARK(12);
  }
#ifdef DK_TIMELINE
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int k = 1; k <= 20; ++k) tl_mark_value(TL_SMALL, k, tacc[k]);
#endif
}

size_t cycle_small_smem(int m) {
  const size_t M1 = (size_t)m + 1;
  return (M1 * M1 + (2 * M1 + 8) + (2 * M1 + 33) * kWarps) * sizeof(double);
}

// cells per thread over one block per SM
static int small_cpt(long long n_pad) {
  const long long threads = (long long)num_sms() * kThreads;
  static const int force = getenv("DK_SMALL_CPT") ? atoi(getenv("DK_SMALL_CPT")) : 0;
  for (int c = 1; c <= 4; c <<= 1)
    if ((long long)c * threads >= n_pad) return (force > c && force <= 4) ? force : c;
  return 0;
}

static unsigned small_grid(long long n_pad, int cpt) {
  const long long need = (n_pad + (long long)cpt * kThreads - 1) / ((long long)cpt * kThreads);
  return (unsigned)std::min<long long>(need, num_sms());
}

bool cycle_small_ok(long long n_pad, int m, int d) {
  if (getenv("DK_NO_SMALL")) return false;
  if (m + 1 > kMaxCycleSmall || d > kSmallMaxD) return false;
  const int cpt = small_cpt(n_pad);
  if (cpt == 0) return false;
  // the grid must be co-resident (the cooperative launch fails otherwise)
  int per_sm = 0;
  const size_t smem = cycle_small_smem(m);
  if (smem_optin((const void*)k_cycle_small<DK_LABELS, true, false, 4>, smem) ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &per_sm, k_cycle_small<DK_LABELS, true, false, 4>, kThreads, smem) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return (long long)per_sm * num_sms() >= small_grid(n_pad, cpt);
}

template <int DEFL, bool PRE, bool AM, int CPT>
static void cycle_small_t(const Dia& A, const Dia& Aam, const Prolong& P, const int* lab, int d,
                          const double* Einv, int ld, double* V, long long vstride,
                          long long n_pad, double* part, double* yg, const Scal& sc,
                          cudaStream_t s) {
  const size_t smem = cycle_small_smem(sc.m);
  // the arrival counter of small_sync (zeroed per launch; after the group tickets)
  unsigned* counter = sc.gticket + kGroupTickets;
  cudaMemsetAsync(counter, 0, sizeof(unsigned), s);
  (void)yg;
  smem_optin((const void*)k_cycle_small<DEFL, PRE, AM, CPT>, smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(small_grid(n_pad, CPT));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // co-residency guaranteed or the launch fails
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  pdl_skip_next() = false;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, k_cycle_small<DEFL, PRE, AM, CPT>, A, Aam, P,
                                           lab, d, Einv, ld, V, vstride, n_pad, part, counter,
                                           sc);
  if (e != cudaSuccess) launch_error() = e;
}

template <int DEFL, bool PRE, bool AM>
static void cycle_small_c(const Dia& A, const Dia& Aam, const Prolong& P, const int* lab, int d,
                          const double* Einv, int ld, double* V, long long vstride,
                          long long n_pad, double* part, double* yg, const Scal& sc,
                          cudaStream_t s) {
  switch (small_cpt(n_pad)) {
    case 1: cycle_small_t<DEFL, PRE, AM, 1>(A, Aam, P, lab, d, Einv, ld, V, vstride, n_pad, part, yg, sc, s); break;
    case 2: cycle_small_t<DEFL, PRE, AM, 2>(A, Aam, P, lab, d, Einv, ld, V, vstride, n_pad, part, yg, sc, s); break;
    default: cycle_small_t<DEFL, PRE, AM, 4>(A, Aam, P, lab, d, Einv, ld, V, vstride, n_pad, part, yg, sc, s); break;
  }
}

void launch_cycle_small(int defl, bool pre, bool am, const Dia& A, const Dia& Aam,
                        const Prolong& P, const RunMap& rm, const double* Einv, int ld, double* V,
                        long long vstride, long long n_pad, double* part, double* yg,
                        const Scal& sc, cudaStream_t s) {
  const int* lab = rm.lab;
  const int d = rm.d;
  if (defl == DK_NONE) {
    if (pre) cycle_small_c<DK_NONE, true, false>(A, Aam, P, lab, d, Einv, ld, V, vstride, n_pad, part, yg, sc, s);
    else cycle_small_c<DK_NONE, false, false>(A, Aam, P, lab, d, Einv, ld, V, vstride, n_pad, part, yg, sc, s);
  } else if (am) {
    if (pre) cycle_small_c<DK_LABELS, true, true>(A, Aam, P, lab, d, Einv, ld, V, vstride, n_pad, part, yg, sc, s);
    else cycle_small_c<DK_LABELS, false, true>(A, Aam, P, lab, d, Einv, ld, V, vstride, n_pad, part, yg, sc, s);
  } else {
    if (pre) cycle_small_c<DK_LABELS, true, false>(A, Aam, P, lab, d, Einv, ld, V, vstride, n_pad, part, yg, sc, s);
    else cycle_small_c<DK_LABELS, false, false>(A, Aam, P, lab, d, Einv, ld, V, vstride, n_pad, part, yg, sc, s);
  }
}

static size_t gs_smem(const Scal& sc, int nvec) {
  int slots = (kWarps > 3 * (sc.m + 1) ? kWarps : 3 * (sc.m + 1));
  if (slots < 261) slots = 261;  // reduce_grouped scratch
  // early start: the projection's group partials, staged (only when early start is on)
  if (sc.post != nullptr && slots < (sc.m + 1) * sc.ng) slots = (sc.m + 1) * sc.ng;
  return ((size_t)nvec + (size_t)slots) * sizeof(double);
}

bool gs_can_fuse(int G, const Scal& sc) {
  int per_sm = 0;
  const size_t smem = gs_smem(sc, sc.m + 1);
  if (smem_optin((const void*)k_gs<false>, smem) != 0) {
    cudaGetLastError();
    return false;
  }
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gs<false>, kThreads, smem) !=
      cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return (long long)per_sm * num_sms() >= G;
}

void launch_gs(bool reorth, const double* w_in, double* u_out, const double* V, long long vstride,
               int nvec, long long n_pad, double* part, int G, const Scal& sc, int j,
               const int* gate, bool fuse, cudaStream_t s) {
  const size_t smem = gs_smem(sc, nvec);
  smem_optin(reorth ? (const void*)k_gs<true> : (const void*)k_gs<false>, smem);
  if (reorth)
    launch_pdl(k_gs<true>, dim3(G), dim3(kThreads), smem, s, w_in, u_out, V, vstride, nvec,
               n_pad, part, G, sc, j, gate, 0, (const unsigned*)nullptr);
  else
    if (fuse && !getenv("DK_NO_COOP")) coop_next() = true;  // the fused pass's grid barrier
    launch_pdl(k_gs<false>, dim3(G), dim3(kThreads), smem, s, w_in, u_out, V, vstride, nvec,
               n_pad, part, G, sc, j, gate, fuse ? 1 : 0,
               (const unsigned*)(fuse && sc.post != nullptr ? sc.post + (sc.m + 1) + j
                                                            : nullptr));
}

// ======================================================================================
// Cycle end (krylov.py:199-212): drop dependent trailing columns, y = R^-1 g by column-
// oriented back substitution (one warp; each y_i sees the same operation order as the
// sequential loop), coefficients for x += M^-1 V y.
// ======================================================================================
__global__ void __launch_bounds__(32) k_cycle_end(Scal sc) {
  pdl_wait();
  State* st = sc.st;
  if (sc.post != nullptr)  // re-arm the early-start flags (the last iteration's is still set)
    for (int i = threadIdx.x; i < 2 * (sc.m + 1); i += 32) sc.post[i] = 0u;
  if (!st->cycle_open) {
    // no cycle ran (a finished solve's gated pass through the restart loop's body): the
    // previous cycle's x update must not be applied again
    if (threadIdx.x == 0) st->xupdate = 0;
    return;
  }
  extern __shared__ double sm[];
  const int m = sc.m;
  const int lane = threadIdx.x;
  int cols = st->cols;
  __syncwarp();
  if (lane == 0) {
    st->cycle_open = 0;
    st->active = 0;
    st->cycle_cols = cols;
  }
  if (cols == 0) {  // krylov.py:199-200
    if (lane == 0) {
      st->running = 0;
      st->last_cols = 0;
      st->xupdate = 0;
    }
    return;
  }
  const double r00 = fabs(sc.R[0]);
  while (cols > 1 && fabs(sc.R[(size_t)(cols - 1) * (m + 1) + (cols - 1)]) < 1e-14 * r00) --cols;
  // R (column k holds rows 0..k, ld m + 1) staged in shared memory for cycles up to
  // kStageGram columns, read from global memory beyond
  const bool stage = m <= kStageGram;
  const int ldr = stage ? cols : m + 1;
  double* y = sm;                  // cols
  const double* R = sc.R;
  if (stage) {
    double* Rs = sm + cols;
    for (int e = lane; e < cols * cols; e += 32)
      Rs[e] = sc.R[(size_t)(e / cols) * (m + 1) + (e % cols)];
    R = Rs;
  }
  for (int i = lane; i < cols; i += 32) y[i] = sc.g[i];
  __syncwarp();
  for (int k = cols - 1; k >= 0; --k) {
    const double* Rk = R + (size_t)k * ldr;
    if (lane == 0) y[k] = y[k] / Rk[k];
    __syncwarp();
    const double yk = y[k];
    for (int i = lane; i < k; i += 32) y[i] = __dsub_rn(y[i], __dmul_rn(yk, Rk[i]));
    __syncwarp();
  }
  for (int i = lane; i < cols; i += 32) {
    sc.y[i] = y[i];
    sc.coef[i] = y[i] * sc.sigma[i];
  }
  if (lane == 0) {
    st->last_cols = cols;
    st->xupdate = 1;
    st->cycle += 1;
    const bool done = st->converged || st->iterations >= st->max_iters;  // krylov.py:127
    st->running = done ? 0 : 1;
  }
}

void launch_cycle_end(const Scal& sc, cudaStream_t s) {
  const size_t m = (size_t)sc.m;
  const size_t smem = (m + 1 + (sc.m <= kStageGram ? m * m : 0)) * sizeof(double);
  smem_optin((const void*)k_cycle_end, 160 * 1024);
  launch_pdl(k_cycle_end, dim3(1), dim3(32), smem, s, sc);
}
// x += M^-1 (sum_{i<cols} y_i V_i)   (krylov.py:206)
__global__ void __launch_bounds__(kThreads) k_xupdate(Dia A, double* __restrict__ x,
                                                      const double* __restrict__ V,
                                                      long long vstride, long long n_pad,
                                                      Scal sc) {
  pdl_wait();
  State* st = sc.st;
  if (!st->xupdate) return;
  const int cols = st->last_cols;
  extern __shared__ double cf[];
  for (int q = threadIdx.x; q < cols; q += blockDim.x) cf[q] = sc.coef[q];
  __syncthreads();
  const long long npair = n_pad / 2;
  for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < npair;
       p += (long long)gridDim.x * blockDim.x) {
    const long long i = 2 * p;
    double t0 = 0.0, t1 = 0.0;
    for (int v = 0; v < cols; ++v) {
      const double2 q = ld2(V + (long long)v * vstride + i);
      t0 = fma(cf[v], q.x, t0);
      t1 = fma(cf[v], q.y, t1);
    }
    if (A.inv != nullptr) {
      t0 = __dmul_rn(t0, A.inv[i]);
      t1 = __dmul_rn(t1, A.inv[i + 1]);
    }
    double2 xv = *reinterpret_cast<double2*>(x + i);
    xv.x = __dadd_rn(xv.x, t0);
    xv.y = __dadd_rn(xv.y, t1);
    st2(x + i, xv);
  }
}

void launch_xupdate(const Dia& A, double* x, const double* V, long long vstride, long long n_pad,
                    const Scal& sc, cudaStream_t s) {
  const size_t smem = (size_t)(sc.m + 1) * sizeof(double);
  launch_pdl(k_xupdate, dim3(num_sms() * 8), dim3(kThreads), smem, s, A, x, V, vstride, n_pad, sc);
}

// ======================================================================================
// Elementwise helpers for x* / P2 / reconstruct (deflation.py:61-68,88).
// ======================================================================================
__global__ void k_recon(const int* __restrict__ lab, const double* __restrict__ y,
                        const double* __restrict__ xs, const double* __restrict__ xh,
                        double* __restrict__ out, long long n_pad, int mode) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n_pad;
       i += (long long)gridDim.x * blockDim.x) {
    const int L = lab[i];
    const double zy = L >= 0 ? y[L] : 0.0;
    if (mode == 0) out[i] = __dadd_rn(xs[i], __dsub_rn(xh[i], zy));  // x* + (xh - Z y)
    else if (mode == 1) out[i] = zy;                                  // Z y
    else out[i] = __dsub_rn(xh[i], zy);                               // v - Z y
  }
}

void launch_recon(const int* lab, const double* y, const double* xs, const double* xh, double* out,
                  long long n_pad, cudaStream_t s) {
  k_recon<<<num_sms() * 8, kThreads, 0, s>>>(lab, y, xs, xh, out, n_pad, 0);
}
void launch_bcast(const int* lab, const double* y, double* out, long long n_pad, cudaStream_t s) {
  k_recon<<<num_sms() * 8, kThreads, 0, s>>>(lab, y, nullptr, nullptr, out, n_pad, 1);
}
void launch_sub_bcast(const int* lab, const double* y, const double* v, double* out,
                      long long n_pad, cudaStream_t s) {
  k_recon<<<num_sms() * 8, kThreads, 0, s>>>(lab, y, nullptr, v, out, n_pad, 2);
}

__global__ void __launch_bounds__(kThreads) k_norm(const double* __restrict__ v, long long n_pad,
                                                   double* __restrict__ part, int G,
                                                   unsigned int* ticket, double* dst) {
  __shared__ double red[kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc = 0.0;
  const long long nchunks = n_pad / kChunk;
  for (long long ch = blockIdx.x; ch < nchunks; ch += gridDim.x) {
    const long long cb = ch * kChunk + 2 * threadIdx.x;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double2 x = ld2cg(v + cb + 512 * k);
      acc = fma(x.x, x.x, acc);
      acc = fma(x.y, x.y, acc);
    }
  }
  acc = warp_sum(acc);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kWarps; ++w) s += red[w];
    part[blockIdx.x] = s;
  }
  if (!last_block(ticket)) return;
  __shared__ double fin[1];
  reduce_partials(part, 1, G, fin);
  if (threadIdx.x == 0) *dst = sqrt(fin[0]);
}

void launch_norm(const double* v, long long n_pad, double* part, int G, unsigned int* ticket,
                 double* dst, cudaStream_t s) {
  k_norm<<<G, kThreads, 0, s>>>(v, n_pad, part, G, ticket, dst);
}

__global__ void k_init_state(Scal sc, double tol, int m, int max_iters, int min_iters) {
  State* st = sc.st;
  st->running = 1;
  st->cycle_open = 0;
  st->active = 0;
  st->reorth = 0;
  st->iterations = 0;
  st->cycle = 0;
  st->converged = 0;
  st->warning = 0;
  st->cols = 0;
  st->last_cols = 0;
  st->denom_set = 0;
  st->has_prev = 0;
  st->reorths = 0;
  st->m = m;
  st->max_iters = max_iters;
  st->min_iters = min_iters;
  st->tol = tol;
  st->denom = 1.0;
  st->beta = 0.0;
  st->prev_beta = 0.0;
  st->wnorm0 = 0.0;
  st->xupdate = 0;
  st->cycle_cols = 0;
  st->last_broke = 0;
  st->loop_left = 0;
  for (int i = 0; i < 4; ++i) st->ticket[i] = 0u;
}

void launch_init_state(const Scal& sc, double tol, int m, int max_iters, int min_iters,
                       cudaStream_t s) {
  k_init_state<<<1, 1, 0, s>>>(sc, tol, m, max_iters, min_iters);
}

// continue a solve across calls (RDGMRES switches the deflation context between cycles,
// harmonic.py:163-178): the counters, the convergence denominator and the restart history
__global__ void k_resume_state(Scal sc, int iterations, int cycles, int warning, int has_prev,
                               double denom, double prev_beta) {
  State* st = sc.st;
  st->iterations = iterations;
  st->cycle = cycles;
  st->warning = warning;
  st->has_prev = has_prev;
  st->denom = denom;
  st->denom_set = 1;
  st->prev_beta = prev_beta;
}

void launch_resume_state(const Scal& sc, int iterations, int cycles, int warning, int has_prev,
                         double denom, double prev_beta, cudaStream_t s) {
  k_resume_state<<<1, 1, 0, s>>>(sc, iterations, cycles, warning, has_prev, denom, prev_beta);
}

// ---- device-decided restart loop (krylov.py:127 `while not converged and it < max_iters`) --
// The cycle graph is the body of a conditional WHILE node; its last kernel decides whether
// another cycle starts: the solve is still running and the caller's cycle budget is not spent.
__global__ void k_loop_arm(State* st, int cycles) { st->loop_left = cycles; }
__global__ void k_loop_cond(State* st, cudaGraphConditionalHandle h) {
  pdl_wait();
  const int left = st->loop_left - 1;
  st->loop_left = left;
  cudaGraphSetConditional(h, (st->running && left > 0) ? 1u : 0u);
}
void launch_loop_arm(const Scal& sc, int cycles, cudaStream_t s) {
  k_loop_arm<<<1, 1, 0, s>>>(sc.st, cycles);
}
void launch_loop_cond(const Scal& sc, cudaGraphConditionalHandle h, cudaStream_t s) {
  launch_pdl(k_loop_cond, dim3(1), dim3(1), 0, s, sc.st, h);
}

DK_TL_SETTER(tl_set_kernels)

}  // namespace dk
