// dk_internal.cuh — shared device-side definitions for the deflated-GMRES hot path.
//
// HBM layout:
//   * every length-n vector is stored "guarded": [guard zeros | n_pad cells | guard zeros],
//     n_pad = n rounded up to kTile, guard = max |stencil offset| rounded up to 256, so the
//     7-point stencil reads v[i + off] without bounds checks (the DIA coefficient is 0 there);
//   * the Krylov basis V is (m+1) rows of stride n_pad + guard sharing the zero guards;
//   * A is DIA: ndiag (<= 7) rows of n_pad fp64 coefficients, offsets ascending (CSR column
//     order, so row sums are formed in the same order as scipy's csr_matvec);
//   * labels (deflation column per cell, -1 = none) are int32, guarded with -1.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "../../include/dk.h"

namespace dk {

constexpr int kThreads = 256;        // threads per streaming block
constexpr int kTile = 2048;          // cells per stencil/restriction tile (8 per thread)
constexpr int kChunk = 2048;         // cells per Gram-Schmidt chunk (8 per thread)
constexpr int kMaxDiag = DK_MAX_DIAGONALS;
constexpr int kWarps = kThreads / 32;
static_assert(kWarps % 4 == 0, "k_project's basis sweep gives each warp one quarter-chunk");

// A(i, i + off[q]) = co[q][i + csh[q]].  Non-symmetric operators store every diagonal
// (csh = 0).  A symmetric operator stores the centre and the positive diagonals only; the
// negative diagonal -o reads the +o array at the neighbour, a(i, i-o) = a(i-o, i) = up_o[i-o]
// (csh = -o) — 4 arrays instead of 7, the same values in the same summation order.
struct Dia {
  int ndiag;
  int center;                  // index of offset 0, or -1
  long long off[kMaxDiag];     // ascending
  const double* co[kMaxDiag];  // guarded coefficient arrays
  long long csh[kMaxDiag];     // index shift into co[q]
  const double* inv;           // guarded Jacobi inverse diagonal, nullptr = identity
};

__device__ __forceinline__ double dia_coef(const Dia& A, int q, long long i) {
  return __ldg(A.co[q] + i + A.csh[q]);
}

// Scalar state of one solve; lives in device memory and is owned by the single-thread
// "control" sections (last block of a reduction kernel, cycle-end kernel).
struct State {
  int running;     // solve not finished: gates the restart kernels
  int cycle_open;  // the current cycle passed its restart test: gates the cycle end
  int active;      // inner iterations of the current cycle still to run: gates the Arnoldi kernels
  int reorth;      // current iteration needs a second Gram-Schmidt pass
  int iterations;
  int cycle;
  int converged;
  int warning;
  int cols;
  int last_cols;
  int denom_set;
  int has_prev;
  int reorths;
  int xupdate;     // cycle end produced an x update (gates k_xupdate)
  int cycle_cols;  // columns of the last cycle before the dependent-column drop
  int last_broke;  // the last iteration ended its cycle by convergence or breakdown
  int loop_left;   // cycles the device-side restart loop (WHILE graph) may still start
  int m, max_iters, min_iters;
  double tol, denom, beta, prev_beta, wnorm0;
  unsigned int ticket[4];
};

struct Scal {
  State* st;
  double* sigma;   // [m+1]  1 / ||u_i||: V_i = sigma_i * u_i (lazy normalisation)
  double* coef;    // [m+1]  Gram-Schmidt / x-update coefficients for the stored u_i
  double* corr;    // [m+1]  re-orthogonalisation coefficients (stored-u scale)
  double* H;       // [(m+1) m] pristine Hessenberg, column-major (column j contiguous)
  double* R;       // [(m+1) m] Givens-rotated triangle, column-major
  double* cs;      // [m]
  double* sn;      // [m]
  double* g;       // [m+1]
  double* y;       // [m+1]
  double* Gm;      // [(m+1)(m+1)] basis Gram matrix V^T V, column j holds rows 0..j
  double* gcol;    // [m+1]  V^T u of the last Gram-Schmidt vector u (normalised basis rows):
                   //        sigma_{j+1} gcol is the next Gram column (no extra pass over V)
  unsigned int* gticket;  // [kGroupTickets] counters of reduce_grouped
  double* gpart;          // [quantities x kGroupTickets] group partials of reduce_grouped
  double* hist;    // [max_iters+1]
  int* restart_of; // [max_iters+1]
  unsigned* post;  // [2(m+1)] early-start counters (nullptr: off): post[j] counts the group
                   // totals of k_gs(j)'s norm, post[m+1+j] those of the projection's dots; the
                   // next grid starts when all ng are in
  double* gpart_gs;  // group partials of k_gs's norm (apart from the projection's)
  int ng;            // groups of the grouped reductions
  int m;
  // split iteration: the basis sweep h' = U^T w runs concurrently with the
  // coarse solve; h = sigma h' - C y with C's rows c_i = Z^T A_p^T v_i
  int split;             // 0: off
  double* hraw;          // [2(m+1)] reduced U^T w (0..m) and U^T u_j (m+1..2m+1)
  const double* cmat;    // C, (m+1) rows of stride ldc, label order
  long long ldc;
  int dco;               // d (columns of C)
};

// volatile (L2) load of a flag or scalar another grid still running may write
__device__ __forceinline__ unsigned ld_flag(const unsigned* p) {
  return *reinterpret_cast<const volatile unsigned*>(p);
}

// ---- programmatic dependent launch ----------------------------------------------------
// Every kernel of the solve sequence is launched with programmatic stream serialisation:
// it may be scheduled while its predecessor drains, waits (griddepcontrol.wait) for the
// predecessor's completion and memory before touching any data, and lets its own
// successor launch once its blocks have finished their main sweep.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// first launch error since the last reset (launches inside stream capture report late)
inline cudaError_t& launch_error() {
  static thread_local cudaError_t e = cudaSuccess;
  return e;
}

// set before the first launch of a stream capture: a graph's root kernel has no kernel
// predecessor to overlap with and is launched without the programmatic attribute
inline bool& pdl_skip_next() {
  static thread_local bool f = false;
  return f;
}

// set before a launch: the grid's blocks wait on one another, so it is launched cooperative
// (all blocks co-resident or the launch fails — never a partly resident grid that spins
// while another solve holds the SMs)
inline bool& coop_next() {
  static thread_local bool f = false;
  return f;
}

// set before a launch: an L2 access-policy window (persisting set-aside) for that launch
inline const cudaAccessPolicyWindow*& access_window_next() {
  static thread_local const cudaAccessPolicyWindow* w = nullptr;
  return w;
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[3];
  int na = 0;
  if (coop_next()) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
  }
  if (!pdl_skip_next()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (access_window_next() != nullptr) {
    attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[na].val.accessPolicyWindow = *access_window_next();
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  pdl_skip_next() = false;
  access_window_next() = nullptr;
  coop_next() = false;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
  if (e != cudaSuccess) launch_error() = e;
  return e;
}

// ---- timeline instrumentation (diagnostic builds with -DDK_TIMELINE only) ------------
// Thread 0 of a block records (globaltimer ns, kernel kind, phase, block) at phase points;
// tools/timeline.py reads the records back (dk_timeline_* in dk_api.cu) and lays out the
// kernels of one iteration.  Each translation unit holds its own copy of the buffer handle.
struct TlBuf {
  unsigned long long* rec;
  unsigned* cnt;
  unsigned cap;
};
#ifdef DK_TIMELINE
static __device__ TlBuf g_tl;
__device__ __forceinline__ void tl_mark(unsigned kind, unsigned phase) {
  if (threadIdx.x == 0 && g_tl.rec != nullptr) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned i = atomicAdd(g_tl.cnt, 1u);
    if (i < g_tl.cap) {
      g_tl.rec[2 * i] = t;
      g_tl.rec[2 * i + 1] = ((unsigned long long)kind << 56) |
                            ((unsigned long long)phase << 48) | (unsigned long long)blockIdx.x;
    }
  }
}
// per-warp variant (lane 0 of each warp; "block" field = block * 32 + warp)
__device__ __forceinline__ void tl_mark_warp(unsigned kind, unsigned phase) {
  if ((threadIdx.x & 31) == 0 && g_tl.rec != nullptr) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    const unsigned i = atomicAdd(g_tl.cnt, 1u);
    if (i < g_tl.cap) {
      g_tl.rec[2 * i] = t;
      g_tl.rec[2 * i + 1] = ((unsigned long long)kind << 56) |
                            ((unsigned long long)phase << 48) |
                            (unsigned long long)(blockIdx.x * 32 + (threadIdx.x >> 5));
    }
  }
}
// a value record (the "time" field carries v): per-phase sums of persistent kernels
__device__ __forceinline__ void tl_mark_value(unsigned kind, unsigned phase,
                                              unsigned long long v) {
  if (g_tl.rec != nullptr) {
    const unsigned i = atomicAdd(g_tl.cnt, 1u);
    if (i < g_tl.cap) {
      g_tl.rec[2 * i] = v;
      g_tl.rec[2 * i + 1] = ((unsigned long long)kind << 56) |
                            ((unsigned long long)(phase | 0x80) << 48) |
                            (unsigned long long)blockIdx.x;
    }
  }
}
#define DK_TL(kind, phase) ::dk::tl_mark(kind, phase)
#define DK_TLW(kind, phase) ::dk::tl_mark_warp(kind, phase)
#define DK_TL_SETTER(fn) \
  void fn(const TlBuf& b) { cudaMemcpyToSymbol(g_tl, &b, sizeof(TlBuf)); }
#else
#define DK_TL(kind, phase) ((void)0)
#define DK_TLW(kind, phase) ((void)0)
#define DK_TL_SETTER(fn)
#endif
enum TlKind { TL_STENCIL = 1, TL_RESTRICT = 2, TL_TG1 = 3, TL_TG2 = 4, TL_PROJECT = 5, TL_GS = 6,
              TL_TG1W = 7, TL_TG2W = 8, TL_DOTS = 9, TL_SMALL = 10 };

// ---- small device helpers -------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double2 ld2(const double* p) {
  return __ldg(reinterpret_cast<const double2*>(p));
}
__device__ __forceinline__ double2 ld2cg(const double* p) {
  return __ldcg(reinterpret_cast<const double2*>(p));
}
// Streaming loads of the Krylov basis and of E^-1 (GB per iteration, each byte used once per
// pass) carry an L2 evict-first policy so they do not push the small per-iteration vectors
// (w, u, M^-1, labels, A's diagonals: ~70 MB at 1.1 M cells) out of the 126 MB L2.
__device__ __forceinline__ unsigned long long l2_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// set-up constants re-read every iteration (the W tile stream): kept in L2 across the
// per-iteration basis sweeps, which carry evict-first
__device__ __forceinline__ unsigned long long l2_evict_last() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// no priority change: the launch's access-policy window (persisting set-aside) applies
__device__ __forceinline__ unsigned long long l2_evict_unchanged() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ double2 ld2_stream(const double* ptr, unsigned long long pol) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(ptr), "l"(pol));
  return v;
}
// Set-up constants read once per iteration (operator diagonals, M^-1, labels, prolongation
// map) also stream with evict-first: only the W tile stream (evict-last) is meant to stay in
// L2 across iterations.
__device__ __forceinline__ int2 ldi2_stream(const int* ptr, unsigned long long pol) {
  int2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;"
               : "=r"(v.x), "=r"(v.y)
               : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ int4 ldi4_stream(const int* ptr, unsigned long long pol) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(ptr), "l"(pol));
  return v;
}
__device__ __forceinline__ unsigned short ldu16_stream(const void* ptr, unsigned long long pol) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;"
               : "=h"(v)
               : "l"(ptr), "l"(pol));
  return v;
}
// Bulk prefetch of [p, p + bytes) into L2 (16 B aligned, bytes a multiple of 16): issued by
// early-started grids for data that is already final while they wait for their start flag.
__device__ __forceinline__ void l2_prefetch(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// ---- 1D TMA bulk copies completing on an mbarrier (cp.async.bulk, UBLKCP in SASS) --------
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init1(unsigned long long* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)));
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// one elected thread: expect `bytes` on bar, then bulk-copy them global -> shared (evict-first)
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes,
                                            unsigned long long* bar, unsigned long long pol) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
// ring pipelines: one arrive carrying the byte count of every copy of a stage (copies issued
// later complete on the same phase), then plain bulk copies with or without an L2 policy
__device__ __forceinline__ void mbar_arrive_expect(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar, unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
// generic-proxy shared-memory accesses of this thread ordered before later async-proxy
// (bulk copy) accesses to the same locations
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// global memory made visible to this thread (flag acquire) ordered before its bulk copies
__device__ __forceinline__ void fence_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait_parity(unsigned long long* bar, unsigned parity) {
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, "
        "0, p; }"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  }
}

__device__ __forceinline__ void st2(double* p, double2 v) {
  *reinterpret_cast<double2*>(p) = v;
}
// per-iteration vectors (w, u) with an explicit L2 priority (DK_VEC_EF builds: evict-first)
__device__ __forceinline__ void st2_vec(double* p, double2 v) {
#ifdef DK_VEC_EF
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x),
               "d"(v.y), "l"(pol)
               : "memory");
#else
  st2(p, v);
#endif
}
__device__ __forceinline__ double2 ld2_vec(const double* p) {
#ifdef DK_VEC_EF
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  double2 v;
  asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(pol));
  return v;
#else
  return __ldcg(reinterpret_cast<const double2*>(p));
#endif
}

// Every block calls this after writing its partials; returns true in exactly one block
// (the last to finish), which may then read all partials.  Resets the ticket.
__device__ __forceinline__ bool last_block(unsigned int* ticket) {
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int t = atomicAdd(ticket, 1u);
    s_last = (t == gridDim.x - 1) ? 1 : 0;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    if (threadIdx.x == 0) *ticket = 0u;
  }
  return s_last != 0;
}

// Deterministic reduction of q quantities laid out [q][G] by the calling block (one warp
// per quantity, lanes stride, fixed xor tree).  Result to out[q] (shared or global).
__device__ __forceinline__ void reduce_partials(const double* part, int nq, int G, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int q = warp; q < nq; q += nw) {
    double s = 0.0;
    for (int b = lane; b < G; b += 32) s += __ldcg(part + (size_t)q * G + b);
    s = warp_sum(s);
    if (lane == 0) out[q] = s;
  }
  __syncthreads();
}

// Two-level deterministic reduction of per-block partials part[q * G + b], q < nq <= 64 per
// pass: blocks are grouped by kGroup consecutive ids; the last block of a group sums its
// group's partials (four threads per quantity, eight independent loads each) into
// gpart[q * ng + g]; the last group to finish sums the group partials into out[q].  Returns
// true in that one block.  One L2 round trip per level instead of G / 32 dependent loads per
// quantity for a single-level sweep.  gticket: kGroupTickets zeroed counters (reset on exit).
constexpr int kGroup = 32, kGroupTickets = 32;
// The final level's arithmetic for quantity q by one thread (bitwise equal to the block's):
// early-started consumers recompute a total from the group partials themselves.
__device__ __forceinline__ double grouped_total(const double* gpart, int q, int ng,
                                               bool global = true) {
  double t[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    double v[8];
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const double* a = gpart + (size_t)q * ng + 8 * h + b;
      v[b] = (8 * h + b < ng) ? (global ? __ldcg(a) : *a) : 0.0;
    }
    double a = 0.0;
#pragma unroll
    for (int b = 0; b < 8; ++b) a += v[b];
    t[h] = a;
  }
  return ((t[0] + t[1]) + t[2]) + t[3];
}

// post_cnt (nullptr: none): every group's last block adds one once its group partials are
// visible; a consumer that sees ng arrivals may form the totals with grouped_total.
__device__ __forceinline__ bool reduce_grouped(const double* part, int nq, int G,
                                               unsigned int* gticket, double* gpart,
                                               double* out, unsigned* post_cnt = nullptr) {
  __shared__ int s_flag;
  const int ng = (G + kGroup - 1) / kGroup;
  const int g = blockIdx.x / kGroup, gb = g * kGroup;
  const int gsz = (G - gb < kGroup) ? G - gb : kGroup;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_flag = (atomicAdd(&gticket[g], 1u) == (unsigned)(gsz - 1));
  __syncthreads();
  if (!s_flag) return false;
  __threadfence();
  if (threadIdx.x == 0) gticket[g] = 0u;
  for (int q0 = 0; q0 < nq; q0 += (int)blockDim.x / 4) {
    const int q = q0 + (int)threadIdx.x / 4, h = threadIdx.x & 3;
    if (q < nq) {
      const double* p = part + (size_t)q * G + gb + 8 * h;
      double v[8];
#pragma unroll
      for (int b = 0; b < 8; ++b) v[b] = (8 * h + b < gsz) ? __ldcg(p + b) : 0.0;
      double t = 0.0;
#pragma unroll
      for (int b = 0; b < 8; ++b) t += v[b];
      out[4 * (q - q0) + h] = t;
    }
    __syncthreads();
    if (h == 0 && q < nq) {
      const double* t = out + 4 * (q - q0);
      __stcg(gpart + (size_t)q * ng + g, ((t[0] + t[1]) + t[2]) + t[3]);
    }
    __syncthreads();
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0 && post_cnt != nullptr) atomicAdd(post_cnt, 1u);
  if (threadIdx.x == 0)
    s_flag = (atomicAdd(&gticket[kGroupTickets - 1], 1u) == (unsigned)(ng - 1));
  __syncthreads();
  if (!s_flag) return false;
  __threadfence();
  if (threadIdx.x == 0) gticket[kGroupTickets - 1] = 0u;
  // ng <= 31 group partials per quantity, in group order
  double* tmp = out + nq;
  for (int q0 = 0; q0 < nq; q0 += (int)blockDim.x / 4) {
    const int q = q0 + (int)threadIdx.x / 4, h = threadIdx.x & 3;
    if (q < nq) {
      const double* p = gpart + (size_t)q * ng + 8 * h;
      double v[8];
#pragma unroll
      for (int b = 0; b < 8; ++b) v[b] = (8 * h + b < ng) ? __ldcg(p + b) : 0.0;
      double t = 0.0;
#pragma unroll
      for (int b = 0; b < 8; ++b) t += v[b];
      tmp[4 * (q - q0) + h] = t;
    }
    __syncthreads();
    if (h == 0 && q < nq) {
      const double* t = tmp + 4 * (q - q0);
      out[q] = ((t[0] + t[1]) + t[2]) + t[3];
    }
    __syncthreads();
  }
  return true;
}

}  // namespace dk
