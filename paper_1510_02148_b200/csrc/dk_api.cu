// dk_api.cu — the C ABI (include/dk.h): handles, buffers, the GMRES(m) cycle driver.
//
// The driver issues one restart cycle (restart residual, m Arnoldi steps, cycle end) as a
// fixed kernel sequence; every kernel is gated by a device flag, so the sequence is captured
// once into a CUDA graph and replayed per cycle.  The host reads one int per cycle to decide
// whether another cycle is needed — the reference's per-iteration Python control flow
// (krylov.py:127-212) runs on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "dk_launch.h"

using namespace dk;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return DK_ECUDA;
}

#define DK_TRY(x)                                        \
  do {                                                   \
    cudaError_t _e = (x);                                \
    if (_e != cudaSuccess) return cuda_fail(_e, #x);     \
  } while (0)

// record the first error of a launch sequence (graph capture reports late)
#define DK_LOG_ERR(x)                                                    \
  do {                                                                   \
    cudaError_t _e = (x);                                                \
    if (_e != cudaSuccess && launch_error() == cudaSuccess) launch_error() = _e; \
  } while (0)

long long round_up(long long v, long long m) { return (v + m - 1) / m * m; }

// ---- profiling classes ---------------------------------------------------------------
enum ProfClass {
  PC_STENCIL = 0,
  PC_RESTRICT,
  PC_GEMV,
  PC_PROJECT,
  PC_GS,
  PC_REORTH,
  PC_CYCLE,
  PC_XUPDATE,
  PC_RESTART,
  PC_COARSE_REDUCE,
  PC_DOTS,
  PC_COUNT
};
const char* kProfNames[PC_COUNT] = {"stencil_restrict", "restrict_final", "coarse_gemv",
                                    "prolong_dots",     "gs_update",      "gs_reorth",
                                    "cycle_end",        "x_update",       "restart",
                                    "coarse_reduce",    "basis_dots"};

unsigned long long g_ctx_serial = 0;

// below this many deflation columns E^-1 is L2-resident and the plain GEMV is used
constexpr int kSymvMinD = 256;
// the packed solve stages s in shared memory next to its tile buffers (227 KB per CTA)
constexpr int kSymvMaxD = 12288;
// largest dense (non-indicator) deflation basis
constexpr int kDenseMaxD = 64;

}  // namespace

struct dk_defl;

struct dk_op {
  int dev = 0;
  long long n = 0, n_pad = 0, guard = 0, vlen = 0;
  int ndiag = 0, center = -1;
  long long off[kMaxDiag] = {0};
  double* dia = nullptr;           // nstore guarded coefficient rows
  const double* co[kMaxDiag] = {nullptr};
  long long csh[kMaxDiag] = {0};
  int sym = 0;                     // bitwise symmetric: centre + positive diagonals stored
  int nstore = 0;
  double* inv_base = nullptr;
  double* inv = nullptr;
  cudaStream_t own = nullptr, stream = nullptr;
  int G = 1;
  // vectors (guarded)
  double *w_base = nullptr, *x_base = nullptr, *b_base = nullptr, *x0_base = nullptr,
         *t_base = nullptr;
  double *w = nullptr, *x = nullptr, *b = nullptr, *x0 = nullptr, *t = nullptr;
  double* V_base = nullptr;
  long long vstride = 0;
  int v_rows = 0;
  double* part = nullptr;
  int part_q = 0;
  double* nrm = nullptr;  // [4] device norms
  unsigned int* tickets = nullptr;
  bool gs_fuse = false;  // second Gram-Schmidt pass inside k_gs (whole grid co-resident)
  // split iteration: the basis sweep runs on `aux` beside the coarse solve
  bool split = false;
  bool small = false;  // the cycle's Arnoldi steps in one persistent grid (k_cycle_small)
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int G_dots = 1;
  unsigned int* gticket = nullptr;  // reduce_grouped counters
  double* gpart = nullptr;          // reduce_grouped group partials [part_q x kGroupTickets]
  int* one = nullptr;  // device constant 1 (gate of ungated launches)
  // solver state
  State* st = nullptr;
  State* st_host = nullptr;  // pinned
  double* scal = nullptr;
  int scal_m = 0;
  double* hist = nullptr;
  int* rof = nullptr;
  int hist_cap = 0;
  Scal sc{};
  // graph cache
  cudaGraphExec_t gexec = nullptr;
  unsigned long long g_ctx = ~0ull;
  unsigned long long seen_ctx = ~0ull;  // (context, m) of the previous solve
  int seen_m = -1;
  int g_m = -1;
  bool g_loop = false;      // gexec is the WHILE-loop graph (device-decided restarts)
  bool loop_broken = false; // the loop graph could not be built on this driver: flat graph
  int host_syncs = 0;       // host synchronisations of the last solve's cycle loop
  int used_loop = 0;        // the last solve's cycles ran under the device-side loop
  // profiling
  bool prof = false;
  double prof_ms[PC_COUNT] = {0};
  long long prof_n[PC_COUNT] = {0};
  double prof_bytes[PC_COUNT] = {0};
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  std::vector<std::pair<int, size_t>> ev_marks;  // (class, index of start event)
  std::vector<double> ev_bytes;
  int launches = 0;
  bool has_last = false;
  unsigned long long g_split = 0;  // split flag the graph was captured with
  int cur_j = 0;                   // iteration being issued (split_fork)
};

struct dk_defl {
  dk_op* op = nullptr;
  unsigned long long serial = 0;
  int d = 0, ld = 0, ap = DK_AP_A;
  int* lab_base = nullptr;
  int* lab = nullptr;
  int* tile_run_off = nullptr;
  double* run_part = nullptr;
  int* lab_run_ptr = nullptr;
  int* run_slot = nullptr;
  int* long_ids = nullptr;
  long long nruns = 0, nlabelled = 0;
  double* E = nullptr;
  double* Einv = nullptr;
  int* piv = nullptr;
  double* xs_base = nullptr;
  double* xs = nullptr;
  double* s = nullptr;
  double* y = nullptr;
  double* qv_base = nullptr;
  double* own_base = nullptr;           // compact prolongation (k_prolong_setup)
  unsigned char* mask_base = nullptr;
  int2* flab_base = nullptr;            // first two foreign labels per cell
  double2* fco_base = nullptr;          // and their summed coefficients
  Prolong pro{};
  // symmetric coarse solve (E symmetric): packed upper tile triangle of E^-1 + partials
  int sym = 0;
  long long ntiles = 0;
  double* P = nullptr;
  double* rowpart = nullptr;
  double* colpart = nullptr;
  int* seg_ptr = nullptr;   // row-part segment slots per tile row
  int* seg_slot = nullptr;
  // SPD E in nested-dissection order (dk_profile.cu): y = P^T W^T W P s through two tile
  // streams of W = L^-1; Einv then holds W (permuted) and E^-1 is formed only on request
  int prof = 0;
  int* perm = nullptr;   // perm[i] = label at position i
  int* iperm = nullptr;  // position of label L
  double* tv = nullptr;  // t = W s~
  double* T1 = nullptr;  // W's nonzero tiles by block row (both passes read them)
  TileGemv tg1{}, tg2{};
  float ms[4] = {0, 0, 0, 0};
  RunMap rm{};
  double nmasked = 0;  // masked (third+ foreign label) coefficients (byte accounting)
  // split iteration: run sums of A_p^T v_j and C = [c_0 .. c_m] (c_j = Z^T A_p^T v_j)
  double* run_part2 = nullptr;
  double* cmat = nullptr;
  int cmat_rows = 0;
  long long ldc = 0;
  // dense basis (non-indicator Z, d <= kDenseMaxD): rows Z_k and A_p Z_k, guarded like V
  int dense = 0;
  double* Z_base = nullptr;
  double* AZ_base = nullptr;
  double* Z = nullptr;
  double* AZ = nullptr;
  long long zs = 0;
};

namespace {

Dia make_dia(const dk_op* op, bool with_inv) {
  Dia A{};
  A.ndiag = op->ndiag;
  A.center = op->center;
  for (int k = 0; k < kMaxDiag; ++k) {
    A.off[k] = k < op->ndiag ? op->off[k] : 0;
    A.co[k] = k < op->ndiag ? op->co[k] : nullptr;
    A.csh[k] = k < op->ndiag ? op->csh[k] : 0;
  }
  A.inv = with_inv ? op->inv : nullptr;
  return A;
}

int defl_kind(const dk_defl* c) { return !c ? DK_NONE : c->dense ? DK_DENSE : DK_LABELS; }

// Cache of GB-sized device buffers (Krylov basis, E, E^-1, the packed E^-1): kept across
// operators and contexts instead of returned to the pool, whose re-growth (mapping fresh
// memory for a 1 GB block) occasionally took 0.03-1 s.  Same-stream reuse only (the library
// stream of the device), so stream order alone protects a recycled block.
struct BigBlock {
  void* p;
  size_t bytes;
  int dev;
};
std::mutex g_big_mu;
std::vector<BigBlock> g_big_free;
std::vector<BigBlock> g_big_live;
constexpr size_t kBigMin = 64ull << 20;
constexpr size_t kBigCacheCap = 48ull << 30;

cudaError_t big_alloc(void** out, size_t bytes, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (bytes >= kBigMin) {
    std::lock_guard<std::mutex> lk(g_big_mu);
    int best = -1;
    for (int i = 0; i < (int)g_big_free.size(); ++i) {
      const BigBlock& b = g_big_free[i];
      if (b.dev == dev && b.bytes >= bytes && b.bytes <= 2 * bytes &&
          (best < 0 || b.bytes < g_big_free[best].bytes))
        best = i;
    }
    if (best >= 0) {
      *out = g_big_free[best].p;
      g_big_live.push_back(g_big_free[best]);
      g_big_free.erase(g_big_free.begin() + best);
      return cudaSuccess;
    }
  }
  cudaError_t e = cudaMallocAsync(out, bytes, s);
  if (e == cudaSuccess && bytes >= kBigMin) {
    std::lock_guard<std::mutex> lk(g_big_mu);
    g_big_live.push_back({*out, bytes, dev});
  }
  return e;
}

void big_free(void* p, cudaStream_t s) {
  if (!p) return;
  // the block may be handed to another stream next: let this stream's work on it finish
  cudaStreamSynchronize(s);
  {
    std::lock_guard<std::mutex> lk(g_big_mu);
    for (size_t i = 0; i < g_big_live.size(); ++i) {
      if (g_big_live[i].p != p) continue;
      const BigBlock b = g_big_live[i];
      g_big_live.erase(g_big_live.begin() + i);
      size_t cached = 0;
      for (const BigBlock& f : g_big_free) cached += f.bytes;
      if (cached + b.bytes <= kBigCacheCap) {
        g_big_free.push_back(b);
        return;
      }
      break;
    }
  }
  cudaFreeAsync(p, s);
}

// DK_TRACE=1: host-side phase timestamps of the set-up path on stderr (diagnostics)
struct Trace {
  bool on = getenv("DK_TRACE") != nullptr;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const double ms = std::chrono::duration<double, std::milli>(
                          std::chrono::steady_clock::now() - t0).count();
    fprintf(stderr, "[dk] %8.3f ms %s\n", ms, what);
  }
};

// pinned State mirrors are recycled across operators: cudaFreeHost / cudaMallocHost are slow
// and synchronising, and an operator is created per matrix
std::mutex g_pinned_mu;
std::vector<State*> g_pinned_free;

cudaError_t pinned_state(State** out) {
  {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    if (!g_pinned_free.empty()) {
      *out = g_pinned_free.back();
      g_pinned_free.pop_back();
      return cudaSuccess;
    }
  }
  return cudaMallocHost(out, sizeof(State));
}

void pinned_state_release(State* p) {
  std::lock_guard<std::mutex> lk(g_pinned_mu);
  g_pinned_free.push_back(p);
}

// flag <- 0 unless lo[i + o] == up[i] for i in [0, count)  (bitwise symmetry of a pair)
__global__ void k_check_pair(const double* __restrict__ up, const double* __restrict__ lo,
                             long long o, long long count, int* flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
       i += (long long)gridDim.x * blockDim.x)
    if (lo[i + o] != up[i]) atomicExch(flag, 0);
}

int alloc_vec(dk_op* op, double** base, double** ptr) {
  DK_TRY(cudaMallocAsync(base, (size_t)op->vlen * sizeof(double), op->stream));
  DK_TRY(cudaMemsetAsync(*base, 0, (size_t)op->vlen * sizeof(double), op->stream));
  *ptr = *base + op->guard;
  return DK_OK;
}

// copy n values (host or device source) into a guarded device vector
int upload(dk_op* op, double* dst, const double* src) {
  if (src == nullptr) {
    DK_TRY(cudaMemsetAsync(dst, 0, (size_t)op->n * sizeof(double), op->stream));
  } else {
    DK_TRY(cudaMemcpyAsync(dst, src, (size_t)op->n * sizeof(double), cudaMemcpyDefault,
                           op->stream));
  }
  return DK_OK;
}

int download(dk_op* op, double* dst, const double* src, long long count) {
  DK_TRY(cudaMemcpyAsync(dst, src, (size_t)count * sizeof(double), cudaMemcpyDefault, op->stream));
  return DK_OK;
}

// per-block partials: room for q quantities per launch
int ensure_part(dk_op* op, int q) {
  if (op->part_q < q) {
    if (op->part) DK_TRY(cudaFreeAsync(op->part, op->stream));
    if (op->gpart) DK_TRY(cudaFreeAsync(op->gpart, op->stream));
    // [q][grid] partials: grids of up to max(G, SMs) blocks (the persistent small cycle)
    DK_TRY(cudaMallocAsync(&op->part, (size_t)q * std::max(op->G, num_sms()) * sizeof(double),
                           op->stream));
    DK_TRY(cudaMallocAsync(&op->gpart, (size_t)q * kGroupTickets * sizeof(double), op->stream));
    op->part_q = q;
    op->g_m = -1;  // the graph refers to the old buffer
  }
  return DK_OK;
}

int ensure_work(dk_op* op, int m, int max_iters) {
  if (op->v_rows < m + 1) {
    if (op->V_base) big_free(op->V_base, op->stream);
    op->V_base = nullptr;
    op->vstride = op->n_pad + op->guard;
    const size_t total = (size_t)op->guard + (size_t)(m + 1) * op->vstride;
    DK_TRY(big_alloc((void**)&op->V_base, total * sizeof(double), op->stream));
    DK_TRY(cudaMemsetAsync(op->V_base, 0, total * sizeof(double), op->stream));
    op->v_rows = m + 1;
    op->g_m = -1;  // graph refers to the old basis
  }
  // per-block partials: up to (m+1)+1 quantities (dots, norm) per launch
  {
    const int rc = ensure_part(op, std::max(2 * m + 4, kDenseMaxD + 4));
    if (rc) return rc;
  }
  if (op->scal_m < m) {
    if (op->scal) DK_TRY(cudaFreeAsync(op->scal, op->stream));
    const size_t cnt = 9 * (size_t)(m + 1) + 2 * (size_t)(m + 1) * m + 2 * (size_t)m +
                       (size_t)(m + 1) * (m + 1);
    DK_TRY(cudaMallocAsync(&op->scal, cnt * sizeof(double), op->stream));
    DK_TRY(cudaMemsetAsync(op->scal, 0, cnt * sizeof(double), op->stream));
    op->scal_m = m;
    op->g_m = -1;
  }
  if (op->hist_cap < max_iters + 1) {
    if (op->hist) DK_TRY(cudaFreeAsync(op->hist, op->stream));
    if (op->rof) DK_TRY(cudaFreeAsync(op->rof, op->stream));
    DK_TRY(cudaMallocAsync(&op->hist, (size_t)(max_iters + 1) * sizeof(double), op->stream));
    DK_TRY(cudaMallocAsync(&op->rof, (size_t)(max_iters + 1) * sizeof(int), op->stream));
    op->hist_cap = max_iters + 1;
    op->g_m = -1;
  }
  // scalar layout for this m
  double* p = op->scal;
  Scal& sc = op->sc;
  sc.st = op->st;
  sc.m = m;
  sc.sigma = p; p += m + 1;
  sc.coef = p; p += m + 1;
  sc.corr = p; p += m + 1;
  sc.g = p; p += m + 1;
  sc.y = p; p += m + 1;
  sc.H = p; p += (size_t)(m + 1) * m;
  sc.R = p; p += (size_t)(m + 1) * m;
  sc.cs = p; p += m;
  sc.sn = p; p += m;
  sc.Gm = p; p += (size_t)(m + 1) * (m + 1);
  sc.gcol = p; p += m + 1;
  sc.gticket = op->gticket;
  sc.gpart = op->gpart;
  sc.ng = (op->G + kGroup - 1) / kGroup;
  // early start of each iteration's stencil on k_gs's published sigma (needs the fused second
  // Gram-Schmidt pass: k_gs then always finishes the iteration itself).  The fused pass needs
  // the whole k_gs grid co-resident at the shared-memory size it launches with, which early
  // start enlarges (group partials): check with early start, then without it.
  const bool no_fuse = getenv("DK_NO_GS_FUSE") != nullptr;
  sc.post = getenv("DK_NO_EARLY") == nullptr ? reinterpret_cast<unsigned*>(p) : nullptr;
  op->gs_fuse = !no_fuse && gs_can_fuse(op->G, sc);
  if (!op->gs_fuse && sc.post != nullptr) {
    sc.post = nullptr;
    op->gs_fuse = !no_fuse && gs_can_fuse(op->G, sc);
  }
  if (!op->gs_fuse) sc.post = nullptr;
  p += m + 1;
  sc.hraw = p;
  p += 2 * (size_t)(m + 1);
  sc.split = 0;
  sc.cmat = nullptr;
  sc.ldc = 0;
  sc.dco = 0;
  sc.gpart_gs = op->gpart + (size_t)(op->part_q - 1) * kGroupTickets;  // past the dots' rows
  sc.hist = op->hist;
  sc.restart_of = op->rof;
  return DK_OK;
}

// The W tile store is read twice per iteration.  DK_W_PERSIST=1: an L2 persisting set-aside
// of its size for the tile GEMV launches (device-wide limit raised to the largest store in
// use, never lowered).  Measured slower than the evict-last hints (6,250 vs 6,600 it/s at
// config 3) and it does not keep pass 1's tiles resident either: off.
void set_tile_window(dk_defl* c, size_t bytes) {
  c->tg1.win_bytes = c->tg2.win_bytes = 0;
  if (!getenv("DK_W_PERSIST")) return;
  int dev = 0, maxp = 0, maxw = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  if (bytes > (size_t)maxp || bytes > (size_t)maxw) return;
  size_t cur = 0;
  cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
  if (cur < bytes && cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, bytes) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  c->tg1.win_base = c->tg2.win_base = c->T1;
  c->tg1.win_bytes = c->tg2.win_bytes = bytes;
}

// ---- launch bookkeeping (profiling) ---------------------------------------------------
cudaEvent_t next_event(dk_op* op) {
  if (op->ev_used == op->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    op->ev_pool.push_back(e);
  }
  return op->ev_pool[op->ev_used++];
}

struct ProfScope {
  dk_op* op;
  int cls;
  size_t idx = 0;
  double bytes;
  ProfScope(dk_op* o, int c, double by) : op(o), cls(c), bytes(by) {
    op->launches += 1;
    if (op->prof) {
      idx = op->ev_used;
      cudaEventRecord(next_event(op), op->stream);
    }
  }
  ~ProfScope() {
    if (op->prof) {
      cudaEventRecord(next_event(op), op->stream);
      op->ev_marks.push_back({cls, idx});
      op->ev_bytes.push_back(bytes);
    }
  }
};

void prof_collect(dk_op* op) {
  if (!op->prof) return;
  cudaStreamSynchronize(op->stream);
  for (size_t k = 0; k < op->ev_marks.size(); ++k) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, op->ev_pool[op->ev_marks[k].second],
                         op->ev_pool[op->ev_marks[k].second + 1]);
    op->prof_ms[op->ev_marks[k].first] += ms;
    op->prof_n[op->ev_marks[k].first] += 1;
    op->prof_bytes[op->ev_marks[k].first] += op->ev_bytes[k];
  }
  op->ev_marks.clear();
  op->ev_bytes.clear();
  op->ev_used = 0;
}

// ---- the deflation building blocks ------------------------------------------------------
// s = Z^T (mode-applied v) ; y = E^-1 s
void split_fork(dk_op* op, dk_defl* c, const double* vj);

// split_row (split iteration, ST_APPLY): also c_j = Z^T A_p^T v_j into that row of C, and the
// basis sweep forked onto the auxiliary stream right after the stencil
void coarse_solve(dk_op* op, dk_defl* c, int mode, bool pre, bool write, const double* v,
                  const double* scale, const double* b, double* out, const int* gate,
                  const unsigned* wait = nullptr, double* split_row = nullptr) {
  const Dia A = make_dia(op, pre);
  const double n = (double)op->n;
  if (c->dense) {  // stencil (stored), then s = Z^T w and y = E^-1 s in one multi-dot kernel
    const double* src = v;
    if (mode != ST_IDENT) {
      double* dst = write ? out : c->qv_base + op->guard;
      ProfScope ps(op, PC_STENCIL,
                   (16.0 + 8.0 * op->nstore + (pre ? 8.0 : 0.0) + (mode == ST_RESID ? 8.0 : 0.0)) *
                       n);
      launch_stencil(mode, pre, true, A, op->n_pad, v, scale, b, dst, nullptr, gate, op->stream,
                     wait, op->sc.gpart_gs, op->sc.ng);
      src = dst;
    }
    ProfScope ps(op, PC_RESTRICT, 8.0 * (c->d + 1) * n);
    launch_zdots(src, c->Z, c->zs, c->d, op->n_pad, op->part, op->G, op->tickets + 2, c->Einv,
                 c->ld, c->y, 1, gate, op->stream);
    return;
  }
  {
    // v, labels, the output if stored; the operator and M^-1 unless the identity
    const double by = 12.0 + (write ? 8.0 : 0.0) +
                      (mode == ST_IDENT ? 0.0 : 8.0 * op->nstore + (pre ? 8.0 : 0.0));
    ProfScope ps(op, PC_STENCIL, by * n);
    if (split_row != nullptr)
      launch_stencil_split(pre, c->ap == DK_AP_AM, A, op->n_pad, v, scale, out, c->rm,
                           c->run_part2, gate, op->stream, wait, op->sc.gpart_gs, op->sc.ng);
    else
      launch_stencil(mode, pre, write, A, op->n_pad, v, scale, b, out, &c->rm, gate, op->stream,
                     wait, op->sc.gpart_gs, op->sc.ng);
  }
  if (split_row != nullptr) split_fork(op, c, v);
  const double rbytes = (split_row ? 2.0 : 1.0) * (12.0 * (double)c->nlabelled + 8.0 * c->d);
  if (c->prof) {  // s~ = P Z^T w, then the two tile streams (t = W s~, y = P^T W^T t)
    if (split_row != nullptr) {
      {
        ProfScope ps(op, PC_RESTRICT, rbytes);
        launch_restrict_final(c->rm, c->s, gate, op->stream, c->run_part2, split_row);
      }
      ProfScope ps(op, PC_GEMV, 8.0 * 1024.0 * (double)(c->tg1.nt + c->tg2.nt));
      launch_tgemv(c->tg1, c->s, c->tv, nullptr, c->d, gate, op->stream);
      launch_tgemv(c->tg2, c->tv, c->y, c->perm, c->d, gate, op->stream);
      return;
    }
    // pass 1 folds in the column sums (cooperative pass with a grid barrier)
    ProfScope ps(op, PC_GEMV, rbytes + 8.0 * 1024.0 * (double)(c->tg1.nt + c->tg2.nt));
    launch_tgemv_restrict(c->tg1, c->rm, c->s, c->tv, c->d, gate, op->stream);
    launch_tgemv(c->tg2, c->tv, c->y, c->perm, c->d, gate, op->stream);
    return;
  }
  {
    ProfScope ps(op, PC_RESTRICT, rbytes);
    launch_restrict_final(c->rm, c->s, gate, op->stream, split_row ? c->run_part2 : nullptr,
                          split_row);
  }
  {
    if (c->sym) {
      // packed tiles + column partials written and read back
      {
        ProfScope ps(op, PC_GEMV, 8.0 * 1024.0 * (double)c->ntiles + 256.0 * (double)c->ntiles);
        launch_symv(c->P, c->d, c->s, c->rowpart, c->colpart, c->y, gate, op->stream);
      }
      ProfScope ps(op, PC_COARSE_REDUCE, 256.0 * (double)c->ntiles);
      launch_symv_reduce(c->d, c->rowpart, c->colpart, c->seg_ptr, c->seg_slot, c->y, gate,
                         op->stream);
    } else {
      ProfScope ps(op, PC_GEMV, 8.0 * (double)c->d * c->ld);
      launch_gemv(c->Einv, c->d, c->ld, c->s, c->y, gate, op->stream);
    }
  }
}

// The split iteration's basis sweep: h' = U^T w and the Gram column U^T u_j (reduced into
// sc.hraw), on the auxiliary stream between ev_fork (after the stencil) and ev_join (waited
// before the projection's fix-up).  An event-profiled solve keeps it on the main stream.
void split_fork(dk_op* op, dk_defl* c, const double* vj) {
  (void)c;
  (void)vj;
  State* st = op->st;
  Scal sc = op->sc;
  if (op->prof) sc.post = nullptr;
  const int j = op->cur_j;
  const int nvec = j + 1;
  double* V = op->V_base + op->guard;
  const double n = (double)op->n;
  cudaStream_t s = op->prof ? op->stream : op->aux;
  if (!op->prof) {
    DK_LOG_ERR(cudaEventRecord(op->ev_fork, op->stream));
    DK_LOG_ERR(cudaStreamWaitEvent(op->aux, op->ev_fork, 0));
  }
  {
    ProfScope ps(op, PC_DOTS, (8.0 + 8.0 * nvec) * n);
    launch_project(PJ_DOTS, DK_NONE, false, make_dia(op, false), Prolong{}, nullptr, op->w,
                   op->w, V, op->vstride, nvec, op->n_pad, op->part, op->G_dots, sc, j,
                   &st->active, s, op->prof);
  }
  if (!op->prof) DK_LOG_ERR(cudaEventRecord(op->ev_join, op->aux));
}

// One GMRES(m) cycle as a fixed kernel sequence (restart, m Arnoldi steps, cycle end).
void issue_restart(dk_op* op, dk_defl* c) {
  State* st = op->st;
  const bool pre = op->inv != nullptr;
  const bool am = c && c->ap == DK_AP_AM;
  const Dia A = make_dia(op, pre);
  const Dia Aam = make_dia(op, am);
  const double n = (double)op->n;
  if (c) {
    coarse_solve(op, c, ST_RESID, false, true, op->x, nullptr, op->b, op->w, &st->running);
  } else {
    ProfScope ps(op, PC_STENCIL, (8.0 * op->nstore + 24.0) * n);
    launch_stencil(ST_RESID, false, true, A, op->n_pad, op->x, nullptr, op->b, op->w, nullptr,
                   &st->running, op->stream);
  }
  // w in/out; with deflation the compact prolongation: labels 4, own 8, mask 1 per cell and
  // one coefficient + label (+ M^-1 for A_p = AM) per foreign-label entry; dense: A_p Z rows
  const double pro_bytes = !c ? 0.0 : c->dense ? 8.0 * c->d * n
                                               : 37.0 * n + (am ? 20.0 : 12.0) * c->nmasked;
  ProfScope ps(op, PC_RESTART, 16.0 * n + pro_bytes);
  launch_project(PJ_RESTART, defl_kind(c), am, Aam, c ? c->pro : Prolong{}, c ? c->y : nullptr,
                 op->w, op->V_base + op->guard, nullptr, op->vstride, 0, op->n_pad, op->part,
                 op->G, op->sc, 0, &st->running, op->stream);
}

int read_state(dk_op* op);
int setup_split(dk_op* op, dk_defl* c, int m);

void issue_iteration(dk_op* op, dk_defl* c, int j) {
  op->cur_j = j;
  // an event-profiled (launch-per-kernel) solve serialises the kernel boundaries, so each
  // kernel's event time is its own (no early start across the control tails)
  Scal sc = op->sc;
  if (op->prof) sc.post = nullptr;
  State* st = op->st;
  const bool pre = op->inv != nullptr;
  const bool am = c && c->ap == DK_AP_AM;
  const Dia A = make_dia(op, pre);
  const Dia Aam = make_dia(op, am);
  const double n = (double)op->n;
  double* V = op->V_base + op->guard;
  const int nvec = j + 1;
  const double pro_bytes = !c ? 0.0 : c->dense ? 8.0 * c->d * n
                                               : 37.0 * n + (am ? 20.0 : 12.0) * c->nmasked;
  // from the second iteration of a cycle on, the stencil starts on k_gs's published sigma
  const unsigned* wait = (sc.post != nullptr && j >= 1) ? sc.post + (j - 1) : nullptr;
  if (c && op->split) {
    // split iteration: stencil (+ c_j), fork of the basis sweep h' = U^T w onto aux, the
    // coarse solve here, join; then w -= A_p Z y, h = sigma h' - C y and the H column
    coarse_solve(op, c, ST_APPLY, pre, true, V + (long long)j * op->vstride, sc.sigma + j,
                 nullptr, op->w, &st->active, wait, c->cmat + (long long)j * c->ldc);
    if (!op->prof) DK_LOG_ERR(cudaStreamWaitEvent(op->stream, op->ev_join, 0));
    {
      ProfScope ps(op, PC_PROJECT,
                   24.0 * n + pro_bytes + 8.0 * (double)nvec * (c->d + 1) + 8.0 * c->d);
      launch_project(PJ_FIX, DK_LABELS, am, Aam, c->pro, c->y, op->w, op->w, V, op->vstride,
                     nvec, op->n_pad, op->part, op->G, sc, j, &st->active, op->stream,
                     op->prof);
    }
  } else if (c) {
    coarse_solve(op, c, ST_APPLY, pre, true, V + (long long)j * op->vstride, sc.sigma + j,
                 nullptr, op->w, &st->active, wait);
  } else {
    ProfScope ps(op, PC_STENCIL, (8.0 * op->nstore + (pre ? 24.0 : 16.0)) * n);
    launch_stencil(ST_APPLY, pre, true, A, op->n_pad, V + (long long)j * op->vstride,
                   sc.sigma + j, nullptr, op->w, nullptr, &st->active, op->stream, wait,
                   sc.gpart_gs, sc.ng);
  }
  if (!(c && op->split)) {
    ProfScope ps(op, PC_PROJECT,
                 c ? (24.0 + 8.0 * nvec) * n + pro_bytes : (16.0 + 8.0 * nvec) * n);
    launch_project(PJ_ITER, defl_kind(c), am, Aam, c ? c->pro : Prolong{}, c ? c->y : nullptr,
                   op->w, op->w, V, op->vstride, nvec, op->n_pad, op->part, op->G, sc, j,
                   &st->active, op->stream);
  }
  {
    ProfScope ps(op, PC_GS, (16.0 + 8.0 * nvec) * n);
    launch_gs(false, op->w, V + (long long)(j + 1) * op->vstride, V, op->vstride, nvec,
              op->n_pad, op->part, op->G, sc, j, &st->active, op->gs_fuse, op->stream);
  }
  if (op->gs_fuse) return;  // the second pass, when needed, runs inside k_gs
  // second Gram-Schmidt pass, gated on the device-side test (krylov.py:167-170)
  if (op->prof) {
    if (read_state(op) || !op->st_host->reorth) return;
  }
  {
    ProfScope ps(op, PC_REORTH, (16.0 + 16.0 * nvec) * n);
    launch_project(PJ_REDOTS, DK_NONE, false, A, Prolong{}, nullptr,
                   V + (long long)(j + 1) * op->vstride, nullptr, V, op->vstride, nvec, op->n_pad,
                   op->part, op->G, sc, j, &st->reorth, op->stream);
    launch_gs(true, V + (long long)(j + 1) * op->vstride, V + (long long)(j + 1) * op->vstride, V,
              op->vstride, nvec, op->n_pad, op->part, op->G, sc, j, &st->reorth, false,
              op->stream);
  }
}

// the m Arnoldi steps of a cycle as one persistent cooperative grid (small problems)
void issue_cycle_small(dk_op* op, dk_defl* c, int m) {
  const bool pre = op->inv != nullptr;
  const bool am = c && c->ap == DK_AP_AM;
  Scal sc = op->sc;
  sc.post = nullptr;
  ProfScope ps(op, PC_PROJECT, 0.0);
  launch_cycle_small(c ? DK_LABELS : DK_NONE, pre, am, make_dia(op, pre), make_dia(op, am),
                     c ? c->pro : Prolong{}, c ? c->rm : RunMap{}, c ? c->Einv : nullptr,
                     c ? c->ld : 0, op->V_base + op->guard, op->vstride, op->n_pad, op->part,
                     c ? c->y : nullptr, sc, op->stream);
  (void)m;
}

void issue_cycle_end(dk_op* op) {
  const bool pre = op->inv != nullptr;
  const Dia A = make_dia(op, pre);
  {
    ProfScope ps(op, PC_CYCLE, 0.0);
    launch_cycle_end(op->sc, op->stream);
  }
  ProfScope ps(op, PC_XUPDATE, 0.0);
  launch_xupdate(A, op->x, op->V_base + op->guard, op->vstride, op->n_pad, op->sc, op->stream);
}

int read_state(dk_op* op) {
  DK_TRY(cudaMemcpyAsync(op->st_host, op->st, sizeof(State), cudaMemcpyDeviceToHost, op->stream));
  DK_TRY(cudaStreamSynchronize(op->stream));
  return DK_OK;
}

// One GMRES cycle recorded into the capturing stream (restart, m Arnoldi steps, cycle end).
static void issue_cycle(dk_op* op, dk_defl* c, int m) {
  issue_restart(op, c);
  if (op->small) issue_cycle_small(op, c, m);
  else
    for (int j = 0; j < m; ++j) issue_iteration(op, c, j);
  issue_cycle_end(op);
}

static int end_capture(dk_op* op, cudaGraph_t* g) {
  const cudaError_t le = launch_error();
  launch_error() = cudaSuccess;
  const cudaError_t ce = cudaStreamEndCapture(op->stream, g);
  if (le != cudaSuccess) return cuda_fail(le, "kernel launch during graph capture");
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture");
  return DK_OK;
}

// The restart loop on the device (krylov.py:127): a graph holding one conditional WHILE node
// whose body is the cycle followed by k_loop_cond.  One launch runs every remaining cycle; the
// host reads the state once, after the loop.  Returns a cuda error when the driver rejects
// any step (the caller then builds the flat one-cycle graph).
static cudaError_t build_loop_graph(dk_op* op, dk_defl* c, int m, cudaGraphExec_t* out) {
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaGraphCreate(&g, 0);
  if (e != cudaSuccess) return e;
  cudaGraphConditionalHandle h;
  e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNode_t node;
  cudaGraphNodeParams cp = {};
  if (e == cudaSuccess) {
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    e = cudaGraphAddNode(&node, g, nullptr, 0, &cp);
  }
  if (e == cudaSuccess) {
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    launch_error() = cudaSuccess;
    e = cudaStreamBeginCaptureToGraph(op->stream, body, nullptr, nullptr, 0,
                                      cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
      pdl_skip_next() = true;
      const int l0 = op->launches;
      issue_cycle(op, c, m);
      launch_loop_cond(op->sc, h, op->stream);
      op->launches = l0;
      const cudaError_t le = launch_error();
      launch_error() = cudaSuccess;
      cudaGraph_t got = nullptr;
      e = cudaStreamEndCapture(op->stream, &got);
      if (e == cudaSuccess) e = le;
    }
  }
  if (e == cudaSuccess) e = cudaGraphInstantiate(out, g, 0);
  if (g) cudaGraphDestroy(g);
  if (e != cudaSuccess) cudaGetLastError();  // clear the sticky-free error for the fallback
  return e;
}

int build_graph(dk_op* op, dk_defl* c, int m) {
  const unsigned long long key =
      (c ? c->serial : 0ull) * 4 + (op->split ? 1 : 0) + (op->small ? 2 : 0);
  if (op->gexec && op->g_m == m && op->g_ctx == key) return DK_OK;
  if (op->gexec) {
    cudaGraphExecDestroy(op->gexec);
    op->gexec = nullptr;
  }
  static const bool loop_off = getenv("DK_NO_LOOP_GRAPH") != nullptr;
  if (!loop_off && !op->loop_broken && !op->split) {
    const cudaError_t le = build_loop_graph(op, c, m, &op->gexec);
    if (le == cudaSuccess) {
      op->g_m = m;
      op->g_ctx = key;
      op->g_loop = true;
      return DK_OK;
    }
    op->gexec = nullptr;
    op->loop_broken = true;
    if (getenv("DK_TRACE"))
      fprintf(stderr, "dk: WHILE-loop graph rejected (%s); one graph launch per cycle\n",
              cudaGetErrorString(le));
  }
  cudaGraph_t g;
  launch_error() = cudaSuccess;
  DK_TRY(cudaStreamBeginCapture(op->stream, cudaStreamCaptureModeThreadLocal));
  pdl_skip_next() = true;
  const int l0 = op->launches;
  issue_cycle(op, c, m);
  op->launches = l0;
  {
    const int rc = end_capture(op, &g);
    if (rc) return rc;
  }
  cudaError_t e = cudaGraphInstantiate(&op->gexec, g, 0);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
  op->g_m = m;
  op->g_ctx = key;
  op->g_loop = false;
  return DK_OK;
}

// Split iteration for label deflation with the symmetric 7-point stencil
// (DK_SPLIT=1: on): the auxiliary stream and events, run_part2 and C, the Scal fields.
int setup_split(dk_op* op, dk_defl* c, int m) {
  Scal& sc = op->sc;
  sc.split = 0;
  op->split = false;
  // opt-in (DK_SPLIT=1): measured slower than the fused projection at config 3 — the basis
  // sweep and the tile GEMV cannot share the SMs
  if (!c || c->dense || !getenv("DK_SPLIT")) return DK_OK;
  if (!sym7_supported(make_dia(op, op->inv != nullptr))) return DK_OK;
  if (!op->aux) {
    DK_TRY(cudaStreamCreateWithFlags(&op->aux, cudaStreamNonBlocking));
    DK_TRY(cudaEventCreateWithFlags(&op->ev_fork, cudaEventDisableTiming));
    DK_TRY(cudaEventCreateWithFlags(&op->ev_join, cudaEventDisableTiming));
  }
  if (!c->run_part2)
    DK_TRY(cudaMallocAsync(&c->run_part2, (size_t)std::max<long long>(c->nruns, 1) * sizeof(double),
                           op->stream));
  if (c->cmat_rows < m + 1) {
    if (c->cmat) DK_TRY(cudaFreeAsync(c->cmat, op->stream));
    c->ldc = round_up(c->d, 32);
    DK_TRY(cudaMallocAsync(&c->cmat, (size_t)(m + 1) * c->ldc * sizeof(double), op->stream));
    c->cmat_rows = m + 1;
    op->g_m = -1;  // a graph of this context refers to the old C
  }
  // the basis sweep leaves SM room for the coarse solve beside it
  static int per_sm = -1;
  if (per_sm < 0) {
    const char* e = getenv("DK_DOTS_CTAS_PER_SM");
    per_sm = e ? std::max(1, atoi(e)) : 2;
  }
  op->G_dots = std::min(op->G, per_sm * num_sms());
  sc.split = 1;
  sc.cmat = c->cmat;
  sc.ldc = c->ldc;
  sc.dco = c->d;
  op->split = true;
  return DK_OK;
}

__global__ void k_scale_copy(const double* __restrict__ u, const double* __restrict__ sig,
                             double* __restrict__ out, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = u[i] * (*sig);
}

}  // namespace

// =========================================================================================
extern "C" {

const char* dk_last_error(void) { return g_err.c_str(); }

int dk_version(void) { return 1; }

int dk_device_count(int32_t* count) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) c = 0;
  cudaGetLastError();
  *count = c;
  return DK_OK;
}

int dk_set_device(int32_t device) {
  DK_TRY(cudaSetDevice(device));
  return DK_OK;
}

int dk_op_create(dk_op** out, int64_t n, int32_t ndiag, const int64_t* offsets,
                 const double* diags, const double* inv_diag) {
  if (!out) return fail(DK_EINVAL, "null handle pointer");
  *out = nullptr;
  if (n < 1) return fail(DK_EINVAL, "operator dimension must be >= 1");
  if (n > (1ll << 31) - (1ll << 24)) return fail(DK_EUNSUPPORTED, "n too large for int32 labels");
  if (ndiag < 1 || ndiag > kMaxDiag)
    return fail(DK_EUNSUPPORTED, "the device path supports 1..7 diagonals (7-point stencil)");
  int cnt = 0;
  if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt < 1) {
    cudaGetLastError();
    return fail(DK_ECUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  }
  std::vector<std::pair<long long, int>> order;
  for (int k = 0; k < ndiag; ++k) {
    if (offsets[k] <= -n || offsets[k] >= n) return fail(DK_EINVAL, "diagonal offset out of range");
    order.push_back({(long long)offsets[k], k});
  }
  std::sort(order.begin(), order.end());
  for (int k = 1; k < ndiag; ++k)
    if (order[k].first == order[k - 1].first) return fail(DK_EINVAL, "duplicate diagonal offset");
  dk_op* op = new dk_op();
  DK_TRY(cudaGetDevice(&op->dev));
  {
    // one library stream per device, shared by every operator: the stream-ordered pool then
    // reuses freed GB-sized blocks (V, E, E^-1) across operators and contexts without
    // cross-stream dependencies (per-operator streams occasionally made the pool map new
    // memory, ~1 s for the E buffers)
    static std::mutex mu;
    static cudaStream_t dev_stream[64] = {nullptr};
    std::lock_guard<std::mutex> lk(mu);
    if (op->dev < 0 || op->dev >= 64) return fail(DK_EINVAL, "device ordinal out of range");
    if (!dev_stream[op->dev])
      DK_TRY(cudaStreamCreateWithFlags(&dev_stream[op->dev], cudaStreamNonBlocking));
    op->own = dev_stream[op->dev];
  }
  {
    // keep up to 16 GB of freed pool memory for the next context (E, E^-1, V are GB-sized)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, op->dev) == cudaSuccess) {
      unsigned long long thr = 16ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  op->stream = op->own;
  op->n = n;
  op->n_pad = round_up(n, kTile);
  long long mo = 0;
  for (int k = 0; k < ndiag; ++k) mo = std::max(mo, std::llabs(order[k].first));
  op->guard = round_up(std::max(mo + 2, 256ll), 256);
  op->vlen = op->n_pad + 2 * op->guard;
  op->ndiag = ndiag;
  for (int k = 0; k < ndiag; ++k) {
    op->off[k] = order[k].first;
    if (order[k].first == 0) op->center = k;
  }
  const long long nch = op->n_pad / kChunk;
  // reduction grid: up to 4 blocks per SM stream the chunks (fixed block -> chunk map, so the
  // per-block partial sums, and hence every reduction, are deterministic)
  op->G = (int)std::min<long long>(nch, (long long)num_sms() * 4);
  // reduce_grouped's group counters share gticket with the fused pass's barrier (the last
  // three slots): at most kGroupTickets - 3 groups
  op->G = std::min(op->G, (kGroupTickets - 3) * kGroup);
  // all diagonals, guarded, ascending offsets
  DK_TRY(cudaMallocAsync(&op->dia, (size_t)ndiag * op->vlen * sizeof(double), op->stream));
  DK_TRY(cudaMemsetAsync(op->dia, 0, (size_t)ndiag * op->vlen * sizeof(double), op->stream));
  for (int k = 0; k < ndiag; ++k) {
    DK_TRY(cudaMemcpyAsync(op->dia + (size_t)k * op->vlen + op->guard,
                           diags + (size_t)order[k].second * n, (size_t)n * sizeof(double),
                           cudaMemcpyDefault, op->stream));
  }
  // bitwise symmetric pattern and values -> keep centre + positive diagonals only
  {
    int sym = 1;
    for (int k = 0; k < ndiag && sym; ++k) {
      const long long o = op->off[k];
      if (o <= 0) continue;
      int partner = -1;
      for (int q = 0; q < ndiag; ++q)
        if (op->off[q] == -o) partner = q;
      if (partner < 0) {
        sym = 0;
        break;
      }
      int* f = nullptr;
      int one_h = 1;
      DK_TRY(cudaMallocAsync(&f, sizeof(int), op->stream));
      DK_TRY(cudaMemcpyAsync(f, &one_h, sizeof(int), cudaMemcpyHostToDevice, op->stream));
      k_check_pair<<<num_sms() * 4, 256, 0, op->stream>>>(op->dia + (size_t)k * op->vlen + op->guard,
                                                    op->dia + (size_t)partner * op->vlen +
                                                        op->guard,
                                                    o, n - o, f);
      DK_TRY(cudaMemcpyAsync(&one_h, f, sizeof(int), cudaMemcpyDeviceToHost, op->stream));
      DK_TRY(cudaStreamSynchronize(op->stream));
      cudaFreeAsync(f, op->stream);
      sym = one_h;
    }
    int npos = 0, nneg = 0;
    for (int k = 0; k < ndiag; ++k) {
      if (op->off[k] > 0) ++npos;
      if (op->off[k] < 0) ++nneg;
    }
    if (npos != nneg) sym = 0;
    op->sym = sym;
    for (int k = 0; k < ndiag; ++k) {
      const long long o = op->off[k];
      int src = k;
      long long sh = 0;
      if (sym && o < 0) {
        for (int q = 0; q < ndiag; ++q)
          if (op->off[q] == -o) src = q;
        sh = o;  // a(i, i+o) = up_{-o}[i + o]
      }
      op->co[k] = op->dia + (size_t)src * op->vlen + op->guard;
      op->csh[k] = sh;
    }
    if (sym) {  // release the negative diagonals' storage by compaction
      double* compact = nullptr;
      int nst = 0;
      for (int k = 0; k < ndiag; ++k)
        if (op->off[k] >= 0) ++nst;
      DK_TRY(cudaMallocAsync(&compact, (size_t)nst * op->vlen * sizeof(double), op->stream));
      int slot = 0;
      long long pos_slot[kMaxDiag];
      for (int k = 0; k < ndiag; ++k) {
        if (op->off[k] < 0) continue;
        DK_TRY(cudaMemcpyAsync(compact + (size_t)slot * op->vlen, op->dia + (size_t)k * op->vlen,
                               (size_t)op->vlen * sizeof(double), cudaMemcpyDeviceToDevice,
                               op->stream));
        pos_slot[k] = slot++;
      }
      for (int k = 0; k < ndiag; ++k) {
        const long long o = op->off[k];
        int src = k;
        if (o < 0)
          for (int q = 0; q < ndiag; ++q)
            if (op->off[q] == -o) src = q;
        op->co[k] = compact + (size_t)pos_slot[src] * op->vlen + op->guard;
      }
      cudaFreeAsync(op->dia, op->stream);
      op->dia = compact;
      op->nstore = nst;
    } else {
      op->nstore = ndiag;
    }
  }
  if (inv_diag) {
    int rc = alloc_vec(op, &op->inv_base, &op->inv);
    if (rc) return rc;
    rc = upload(op, op->inv, inv_diag);
    if (rc) return rc;
  }
  int rc;
  if ((rc = alloc_vec(op, &op->w_base, &op->w))) return rc;
  if ((rc = alloc_vec(op, &op->x_base, &op->x))) return rc;
  if ((rc = alloc_vec(op, &op->b_base, &op->b))) return rc;
  if ((rc = alloc_vec(op, &op->x0_base, &op->x0))) return rc;
  if ((rc = alloc_vec(op, &op->t_base, &op->t))) return rc;
  DK_TRY(cudaMallocAsync(&op->st, sizeof(State), op->stream));
  DK_TRY(cudaMemsetAsync(op->st, 0, sizeof(State), op->stream));
  DK_TRY(pinned_state(&op->st_host));
  DK_TRY(cudaMallocAsync(&op->nrm, 4 * sizeof(double), op->stream));
  DK_TRY(cudaMallocAsync(&op->tickets, 4 * sizeof(unsigned int), op->stream));
  DK_TRY(cudaMallocAsync(&op->gticket, (kGroupTickets + 1) * sizeof(unsigned int), op->stream));
  DK_TRY(cudaMemsetAsync(op->gticket, 0, (kGroupTickets + 1) * sizeof(unsigned int), op->stream));
  {
    const int one_h = 1;
    DK_TRY(cudaMallocAsync(&op->one, sizeof(int), op->stream));
    DK_TRY(cudaMemcpyAsync(op->one, &one_h, sizeof(int), cudaMemcpyHostToDevice, op->stream));
  }
  DK_TRY(cudaMemsetAsync(op->tickets, 0, 4 * sizeof(unsigned int), op->stream));
  rc = ensure_work(op, 1, 1);
  if (rc) return rc;
  DK_TRY(cudaStreamSynchronize(op->stream));
  *out = op;
  return DK_OK;
}

int dk_op_destroy(dk_op* op) {
  if (!op) return DK_OK;
  cudaStreamSynchronize(op->stream);
  if (op->gexec) cudaGraphExecDestroy(op->gexec);
  for (auto e : op->ev_pool) cudaEventDestroy(e);
  if (op->aux) {
    cudaStreamSynchronize(op->aux);
    cudaStreamDestroy(op->aux);
  }
  if (op->ev_fork) cudaEventDestroy(op->ev_fork);
  if (op->ev_join) cudaEventDestroy(op->ev_join);
  // all device buffers of an operator come from the stream-ordered pool
  big_free(op->V_base, op->stream);
  void* bufs[] = {op->dia,     op->inv_base, op->w_base, op->x_base, op->b_base,
                  op->x0_base, op->t_base, op->part,     op->nrm,    op->tickets, op->one,
                  op->st,     op->scal,    op->hist,     op->rof,    op->gticket, op->gpart};
  for (void* p : bufs)
    if (p) cudaFreeAsync(p, op->stream);
  cudaStreamSynchronize(op->stream);
  if (op->st_host) pinned_state_release(op->st_host);
  // op->own is the shared library stream of the device: not destroyed
  delete op;
  return DK_OK;
}

int dk_op_set_precond(dk_op* op, const double* inv_diag) {
  if (!op) return fail(DK_EINVAL, "null operator");
  if (inv_diag == nullptr) {
    op->inv = nullptr;
  } else {
    if (!op->inv_base) {
      int rc = alloc_vec(op, &op->inv_base, &op->inv);
      if (rc) return rc;
    }
    op->inv = op->inv_base + op->guard;
    int rc = upload(op, op->inv, inv_diag);
    if (rc) return rc;
    DK_TRY(cudaStreamSynchronize(op->stream));
  }
  if (op->gexec) {  // the graph bakes the preconditioner in
    cudaGraphExecDestroy(op->gexec);
    op->gexec = nullptr;
    op->g_m = -1;
  }
  return DK_OK;
}

int dk_op_set_stream(dk_op* op, void* stream) {
  if (!op) return fail(DK_EINVAL, "null operator");
  cudaStreamSynchronize(op->stream);
  op->stream = stream ? (cudaStream_t)stream : op->own;
  if (op->gexec) {
    cudaGraphExecDestroy(op->gexec);
    op->gexec = nullptr;
    op->g_m = -1;
  }
  return DK_OK;
}

int dk_op_spmv(dk_op* op, const double* x, double* y) {
  if (!op || !x || !y) return fail(DK_EINVAL, "null argument");
  int rc = upload(op, op->t, x);
  if (rc) return rc;
  const Dia A = make_dia(op, false);
  launch_stencil(ST_APPLY, false, true, A, op->n_pad, op->t, nullptr, nullptr, op->w, nullptr,
                 nullptr, op->stream);
  DK_TRY(cudaGetLastError());
  rc = download(op, y, op->w, op->n);
  if (rc) return rc;
  DK_TRY(cudaStreamSynchronize(op->stream));
  return DK_OK;
}

int dk_op_profile(dk_op* op, int32_t enable) {
  if (!op) return fail(DK_EINVAL, "null operator");
  op->prof = enable != 0;
  for (int k = 0; k < PC_COUNT; ++k) {
    op->prof_ms[k] = 0;
    op->prof_n[k] = 0;
    op->prof_bytes[k] = 0;
  }
  return DK_OK;
}

int dk_op_profile_read(dk_op* op, int32_t cap, const char** names, double* ms, int64_t* launches,
                       double* bytes) {
  if (!op) return fail(DK_EINVAL, "null operator");
  const int k = std::min<int>(cap, PC_COUNT);
  for (int i = 0; i < k; ++i) {
    names[i] = kProfNames[i];
    ms[i] = op->prof_ms[i];
    launches[i] = op->prof_n[i];
    bytes[i] = op->prof_bytes[i];
  }
  return k;
}

// ---- deflation ----------------------------------------------------------------------------
int dk_defl_create(dk_defl** out, dk_op* op, const int32_t* col_of_cell, int32_t d,
                   int32_t ap_choice, const double* b) {
  if (!out || !op || !col_of_cell) return fail(DK_EINVAL, "null argument");
  *out = nullptr;
  if (d < 1) return fail(DK_EINVAL, "Z must be n x d with d >= 1");
  if (ap_choice != DK_AP_A && ap_choice != DK_AP_AM)
    return fail(DK_EINVAL, "A_p_choice must be 'A' or 'AM'");
  if (ap_choice == DK_AP_AM && op->inv == nullptr) {
    // A M^-1 with the identity preconditioner is A itself
    ap_choice = DK_AP_A;
  }
  Trace tr;
  const long long n = op->n, n_pad = op->n_pad;
  // host copy of the labels (input may live on the device)
  std::vector<int> lab(n_pad);
  {
    cudaPointerAttributes pa{};
    const bool on_device = cudaPointerGetAttributes(&pa, col_of_cell) == cudaSuccess &&
                           (pa.type == cudaMemoryTypeDevice || pa.type == cudaMemoryTypeManaged);
    cudaGetLastError();  // a plain host pointer may leave an error behind on old drivers
    if (on_device)
      DK_TRY(cudaMemcpy(lab.data(), col_of_cell, (size_t)n * sizeof(int), cudaMemcpyDefault));
    else
      std::memcpy(lab.data(), col_of_cell, (size_t)n * sizeof(int));
    std::fill(lab.begin() + n, lab.end(), -1);
  }
  // one pass: validation, column sizes and the runs (maximal equal-label ranges in linear
  // order; every tile start is a head)
  std::vector<long long> count(d, 0);
  const long long ntiles = n_pad / kTile;
  std::vector<int> tile_off(ntiles + 1, 0);
  std::vector<int> run_label;
  {
    // host threads scan disjoint tile ranges; their runs are concatenated in tile order, so
    // the result does not depend on the thread count
    struct Part {
      std::vector<int> runs, off;  // runs of the range; first run of each of its tiles
      std::vector<long long> count;
      bool bad = false;
    };
    unsigned hw = std::thread::hardware_concurrency();
    int nthr = (int)std::min<long long>(std::min<unsigned>(hw ? hw : 1u, 8u), ntiles / 64);
    if (nthr < 1) nthr = 1;
    std::vector<Part> parts(nthr);
    auto scan = [&](int p) {
      Part& P = parts[p];
      const long long t0 = ntiles * p / nthr, t1 = ntiles * (p + 1) / nthr;
      P.count.assign(d, 0);
      P.off.reserve(t1 - t0);
      P.runs.reserve((t1 - t0) * kTile / 8 + 16);
      const int* lb = lab.data();
      for (long long t = t0; t < t1; ++t) {
        P.off.push_back((int)P.runs.size());
        const long long i0 = t * kTile;
        int prev = lb[i0];
        if (prev < -1 || prev >= d) {
          P.bad = true;
          return;
        }
        P.runs.push_back(prev);
        if (prev >= 0) P.count[prev]++;
        for (long long i = i0 + 1; i < i0 + kTile; ++i) {
          const int L = lb[i];
          if (L != prev) {
            if (L < -1 || L >= d) {
              P.bad = true;
              return;
            }
            P.runs.push_back(L);
            prev = L;
          }
          if (L >= 0) P.count[L]++;
        }
      }
    };
    if (nthr == 1) {
      scan(0);
    } else {
      std::vector<std::thread> th;
      for (int p = 1; p < nthr; ++p) th.emplace_back(scan, p);
      scan(0);
      for (auto& t : th) t.join();
    }
    size_t total = 0;
    for (const Part& P : parts) {
      if (P.bad) return fail(DK_EINVAL, "column label out of range");
      total += P.runs.size();
    }
    run_label.reserve(total + 16);
    for (int p = 0; p < nthr; ++p) {
      const Part& P = parts[p];
      const long long t0 = ntiles * p / nthr;
      const int base = (int)run_label.size();
      for (size_t k = 0; k < P.off.size(); ++k) tile_off[t0 + (long long)k] = base + P.off[k];
      run_label.insert(run_label.end(), P.runs.begin(), P.runs.end());
      for (int L = 0; L < d; ++L) count[L] += P.count[L];
    }
  }
  tile_off[ntiles] = (int)run_label.size();
  for (int L = 0; L < d; ++L)
    if (count[L] == 0) {
      // an empty indicator column makes E exactly singular (deflation.py:27-28 / sparse.py:135)
      return fail(DK_ESINGULAR, "zero pivot in LU factorization");
    }
  const long long nruns = (long long)run_label.size();
  if (nruns >= (1ll << 31)) return fail(DK_EUNSUPPORTED, "too many label runs");
  std::vector<int> ptr(d + 1, 0);
  for (long long r = 0; r < nruns; ++r)
    if (run_label[r] >= 0) ptr[run_label[r] + 1]++;
  for (int L = 0; L < d; ++L) ptr[L + 1] += ptr[L];
  // label-major slot of every run: the stencil writes run partials there, so each column's
  // runs are contiguous (in run order) for the restriction's final sum
  std::vector<int> slot(std::max<long long>(nruns, 1));
  {
    std::vector<int> fillp(ptr.begin(), ptr.end() - 1);
    int spare = ptr[d];
    for (long long r = 0; r < nruns; ++r)
      slot[r] = run_label[r] >= 0 ? fillp[run_label[r]]++ : spare++;
  }
  tr.mark("labels + run map (host)");
  dk_defl* c = new dk_defl();
  c->op = op;
  c->serial = ++g_ctx_serial;
  c->d = d;
  c->ld = (int)round_up(d, 2);
  c->ap = ap_choice;
  c->nruns = nruns;
  c->nlabelled = ptr[d];
  cudaStream_t s = op->stream;
  auto cleanup_fail = [&](cudaError_t e, const char* where) {
    dk_defl_destroy(c);
    return cuda_fail(e, where);
  };
#define DKD(x)                                           \
  do {                                                   \
    cudaError_t _e = (x);                                \
    if (_e != cudaSuccess) return cleanup_fail(_e, #x);  \
  } while (0)
  DKD(cudaMallocAsync(&c->lab_base, (size_t)op->vlen * sizeof(int), s));
  DKD(cudaMemsetAsync(c->lab_base, 0xff, (size_t)op->vlen * sizeof(int), s));  // -1
  c->lab = c->lab_base + op->guard;
  DKD(cudaMemcpyAsync(c->lab, lab.data(), (size_t)n * sizeof(int), cudaMemcpyHostToDevice, s));
  DKD(cudaMallocAsync(&c->tile_run_off, tile_off.size() * sizeof(int), s));
  DKD(cudaMemcpyAsync(c->tile_run_off, tile_off.data(), tile_off.size() * sizeof(int),
                      cudaMemcpyHostToDevice, s));
  DKD(cudaMallocAsync(&c->run_part, (size_t)nruns * sizeof(double), s));
  DKD(cudaMallocAsync(&c->lab_run_ptr, ptr.size() * sizeof(int), s));
  DKD(cudaMemcpyAsync(c->lab_run_ptr, ptr.data(), ptr.size() * sizeof(int), cudaMemcpyHostToDevice,
                      s));
  DKD(cudaMallocAsync(&c->run_slot, (slot.size() + 4) * sizeof(int), s));
  DKD(cudaMemcpyAsync(c->run_slot, slot.data(), slot.size() * sizeof(int), cudaMemcpyHostToDevice,
                      s));
  tr.mark("run map uploaded");
  // the O(d^2) buffers come from the stream-ordered pool (cached across contexts)
  DKD(big_alloc((void**)&c->E, (size_t)d * c->ld * sizeof(double), s));
  DKD(big_alloc((void**)&c->Einv, (size_t)d * c->ld * sizeof(double), s));
  tr.mark("E, E^-1 allocated");
  DKD(cudaMallocAsync(&c->piv, (size_t)d * sizeof(int), s));
  const size_t dvec = (size_t)round_up(d, 32) * sizeof(double);  // k_tgemv reads 32-blocks
  DKD(cudaMallocAsync(&c->s, dvec, s));
  DKD(cudaMallocAsync(&c->y, dvec, s));
  DKD(cudaMallocAsync(&c->tv, dvec, s));
  DKD(cudaMemsetAsync(c->s, 0, dvec, s));
  DKD(cudaMemsetAsync(c->y, 0, dvec, s));
  DKD(cudaMemsetAsync(c->tv, 0, dvec, s));
  DKD(cudaMallocAsync(&c->xs_base, (size_t)op->vlen * sizeof(double), s));
  DKD(cudaMemsetAsync(c->xs_base, 0, (size_t)op->vlen * sizeof(double), s));
  c->xs = c->xs_base + op->guard;
  DKD(cudaMallocAsync(&c->qv_base, (size_t)op->vlen * sizeof(double), s));
  DKD(cudaMemsetAsync(c->qv_base, 0, (size_t)op->vlen * sizeof(double), s));
  DKD(cudaMallocAsync(&c->own_base, (size_t)op->vlen * sizeof(double), s));
  DKD(cudaMemsetAsync(c->own_base, 0, (size_t)op->vlen * sizeof(double), s));
  DKD(cudaMallocAsync(&c->mask_base, (size_t)op->vlen, s));
  DKD(cudaMemsetAsync(c->mask_base, 0, (size_t)op->vlen, s));
  DKD(cudaMallocAsync(&c->flab_base, (size_t)op->vlen * sizeof(int2), s));
  DKD(cudaMemsetAsync(c->flab_base, 0xff, (size_t)op->vlen * sizeof(int2), s));
  DKD(cudaMallocAsync(&c->fco_base, (size_t)op->vlen * sizeof(double2), s));
  DKD(cudaMemsetAsync(c->fco_base, 0, (size_t)op->vlen * sizeof(double2), s));
  c->pro.lab = c->lab;
  c->pro.own = c->own_base + op->guard;
  c->pro.flab = c->flab_base + op->guard;
  c->pro.fco = c->fco_base + op->guard;
  c->pro.mask = c->mask_base + op->guard;
  {
    unsigned long long* dcnt = nullptr;
    unsigned long long hcnt = 0;
    DKD(cudaMallocAsync(&dcnt, sizeof(unsigned long long), s));
    DKD(cudaMemsetAsync(dcnt, 0, sizeof(unsigned long long), s));
    launch_prolong_setup(ap_choice == DK_AP_AM, make_dia(op, ap_choice == DK_AP_AM), c->lab, n_pad,
                         c->own_base + op->guard, c->flab_base + op->guard,
                         c->fco_base + op->guard, c->mask_base + op->guard, dcnt, s);
    DKD(cudaMemcpyAsync(&hcnt, dcnt, sizeof(hcnt), cudaMemcpyDeviceToHost, s));
    DKD(cudaFreeAsync(dcnt, s));
    DKD(cudaStreamSynchronize(s));
    c->nmasked = (double)hcnt;
  }
  DKD(cudaGetLastError());
  c->rm.lab = c->lab;
  c->rm.tile_run_off = c->tile_run_off;
  c->rm.run_part = c->run_part;
  c->rm.lab_run_ptr = c->lab_run_ptr;
  c->rm.run_slot = c->run_slot;
  c->rm.d = d;
  {
    std::vector<int> long_ids;
    for (int L = 0; L < d; ++L)
      if (ptr[L + 1] - ptr[L] > kShortRuns) long_ids.push_back(L);
    c->rm.nlong = (int)long_ids.size();
    if (!long_ids.empty()) {
      DKD(cudaMallocAsync(&c->long_ids, long_ids.size() * sizeof(int), s));
      DKD(cudaMemcpyAsync(c->long_ids, long_ids.data(), long_ids.size() * sizeof(int),
                          cudaMemcpyHostToDevice, s));
      DKD(cudaStreamSynchronize(s));
    }
    c->rm.long_ids = c->long_ids;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  const bool am = ap_choice == DK_AP_AM;
  tr.mark("buffers + prolongation map");
  int err = build_coarse(make_dia(op, am), am, c->lab, n_pad, c->rm, c->E, c->ld,
                         c->qv_base + op->guard, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&c->ms[0], e0, e1);
  if (err) return cleanup_fail((cudaError_t)err, "build_coarse");
  // keep a copy of E for inspection (the factorisations run in place on the copy)
  const size_t ebytes = (size_t)d * c->ld * sizeof(double);
  double* Ework = nullptr;
  DKD(big_alloc((void**)&Ework, ebytes, s));
  DKD(cudaMemcpyAsync(Ework, c->E, ebytes, cudaMemcpyDeviceToDevice, s));
  tr.mark("E assembled + copied");
  const bool symmetric = !am && coarse_is_symmetric(c->E, d, c->ld, s);
  tr.mark("symmetry check");
  bool inverted = false, spd_failed = false;
  if (symmetric && d >= kSymvMinD && !getenv("DK_NO_ND")) {
    // nested dissection of the label graph: keep it when W's tiles stream in fewer bytes
    // (two passes) than the packed triangle of E^-1
    std::vector<int> gptr, gcol, perm;
    std::vector<NDTreeNode> tree;
    err = coarse_pattern(c->E, d, c->ld, gptr, gcol, s);
    if (err) {
      big_free(Ework, s);
      return cleanup_fail((cudaError_t)err, "coarse_pattern");
    }
    tr.mark("pattern of E");
    nd_order(d, gptr, gcol, perm, &tree);
    tr.mark("nested dissection");
    if (2 * nd_profile_tiles(d, gptr, gcol, perm) < symv_tiles(d) || getenv("DK_FORCE_ND")) {
      std::vector<int> iperm(d);
      for (int i = 0; i < d; ++i) iperm[perm[i]] = i;
      DKD(cudaMallocAsync(&c->perm, (size_t)d * sizeof(int), s));
      DKD(cudaMallocAsync(&c->iperm, (size_t)d * sizeof(int), s));
      DKD(cudaMemcpyAsync(c->perm, perm.data(), (size_t)d * sizeof(int), cudaMemcpyHostToDevice,
                          s));
      DKD(cudaMemcpyAsync(c->iperm, iperm.data(), (size_t)d * sizeof(int),
                          cudaMemcpyHostToDevice, s));
      launch_permute_sym(c->E, d, c->ld, c->perm, Ework, s);
      double min_sq = 0.0;
      cudaEvent_t f0, f1;
      cudaEventCreate(&f0);
      cudaEventCreate(&f1);
      cudaEventRecord(f0, s);
      DKD(cudaMemsetAsync(c->Einv, 0, ebytes, s));
      err = nd_tree_inverse(Ework, d, c->ld, tree, c->Einv, &min_sq, s, &gptr, &gcol, &iperm);
      cudaEventRecord(f1, s);
      cudaEventSynchronize(f1);
      cudaEventElapsedTime(&c->ms[1], f0, f1);
      c->ms[2] = 0.f;
      cudaEventDestroy(f0);
      cudaEventDestroy(f1);
      tr.mark("W = L^-1 along the dissection tree");
      if (err) {
        big_free(Ework, s);
        return cleanup_fail((cudaError_t)err, "spd_inverse");
      }
      if (min_sq >= 1e-280) {
        cudaEvent_t p0, p1;
        cudaEventCreate(&p0);
        cudaEventCreate(&p1);
        cudaEventRecord(p0, s);
        std::vector<int> fW(d);
        int* df = nullptr;
        DKD(cudaMallocAsync(&df, (size_t)d * sizeof(int), s));
        launch_row_first_nz(c->Einv, d, c->ld, df, s);
        DKD(cudaMemcpyAsync(fW.data(), df, (size_t)d * sizeof(int), cudaMemcpyDeviceToHost, s));
        DKD(cudaFreeAsync(df, s));
        DKD(cudaStreamSynchronize(s));
        TileGemvHost h1, h2;
        err = profile_streams(c->Einv, d, c->ld, fW, h1, h2, s);
        if (err) {
          big_free(Ework, s);
          return cleanup_fail(err > 0 ? (cudaError_t)err : cudaErrorUnknown, "profile_streams");
        }
        DKD(big_alloc((void**)&c->T1, (size_t)h1.nt * 1024 * sizeof(double), s));
        c->tg1.T = c->T1;
        c->tg2.T = c->T1;  // pass 2 applies pass 1's tiles transposed
        err = upload_stream(c->Einv, d, c->ld, true, h1, c->tg1, s);
        if (!err) err = upload_stream(c->Einv, d, c->ld, false, h2, c->tg2, s);
        if (!err) set_tile_window(c, (size_t)h1.nt * 1024 * sizeof(double));
        if (err) {
          big_free(Ework, s);
          return cleanup_fail((cudaError_t)err, "upload_stream");
        }
        cudaEventRecord(p1, s);
        DKD(cudaStreamSynchronize(s));
        float pm = 0.f;
        cudaEventElapsedTime(&pm, p0, p1);
        c->ms[2] += pm;  // the tile streams belong to the inverse's set-up share
        cudaEventDestroy(p0);
        cudaEventDestroy(p1);
        c->prof = 1;
        c->rm.s_pos = c->iperm;
        // opt-in L2 prefetches riding on the latency-bound kernels (measured slower, DESIGN.md
        // §5): DK_WPF=1 — the ring stencil prefetches the tile store for the coarse kernels
        // that follow it; DK_PF2=1|2 — that tile pass prefetches the projection's per-cell
        // prolongation constants (DK_PF2_N of its five streams)
        if (getenv("DK_WPF")) {
          c->rm.pf_base = c->T1;
          c->rm.pf_bytes = (unsigned long long)h1.nt * 1024ull * sizeof(double);
        }
        {
          const int which = getenv("DK_PF2") ? atoi(getenv("DK_PF2")) : 0;
          TileGemv* tg = which == 1 ? &c->tg1 : which == 2 ? &c->tg2 : nullptr;
          if (tg != nullptr) {
            const unsigned long long np = (unsigned long long)op->n_pad;
            const char* ptr[5] = {(const char*)c->pro.fco, (const char*)c->pro.flab,
                                  (const char*)c->pro.own, (const char*)c->pro.lab,
                                  (const char*)c->pro.mask};
            const unsigned long long by[5] = {16 * np, 8 * np, 8 * np, 4 * np, np};
            const int lim = getenv("DK_PF2_N") ? atoi(getenv("DK_PF2_N")) : 5;
            tg->npf = 0;
            for (int k = 0; k < 5 && k < lim; ++k) {
              if (((unsigned long long)(uintptr_t)ptr[k] & 15ull) != 0 || (by[k] & 15ull) != 0)
                break;
              tg->pf[k] = ptr[k];
              tg->pf_bytes[k] = by[k];
              tg->npf = k + 1;
            }
          }
        }
        inverted = true;
        tr.mark("W tile streams");
      } else {
        spd_failed = true;
        DKD(cudaMemcpyAsync(Ework, c->E, ebytes, cudaMemcpyDeviceToDevice, s));
      }
    }
  }
  if (symmetric && !inverted && !spd_failed) {  // SPD E: Cholesky-based inverse
    double min_sq = 0.0;
    tr.mark("E assembled");
    err = spd_inverse(Ework, d, c->ld, c->Einv, &min_sq, &c->ms[1], &c->ms[2], s);
    tr.mark("E^-1 (Cholesky path)");
    if (err) {
      big_free(Ework, s);
      return cleanup_fail((cudaError_t)err, "spd_inverse");
    }
    if (min_sq >= 1e-280) {  // E^-1 is in Ework: it becomes Einv, the W scratch is released
      std::swap(Ework, c->Einv);
      inverted = true;
    } else {
      DKD(cudaMemcpyAsync(Ework, c->E, ebytes, cudaMemcpyDeviceToDevice, s));
    }
  }
  if (!inverted) {
    double min_piv = 0.0;
    err = lu_and_inverse(Ework, d, c->ld, c->Einv, c->piv, &min_piv, &c->ms[1], &c->ms[2], s);
    if (err) {
      big_free(Ework, s);
      return cleanup_fail((cudaError_t)err, "lu_and_inverse");
    }
    if (!(min_piv >= 1e-300)) {  // sparse.py:135-136 (NaN pivots are singular too)
      big_free(Ework, s);
      dk_defl_destroy(c);
      return fail(DK_ESINGULAR, "zero pivot in LU factorization");
    }
  }
  big_free(Ework, s);
  // symmetric E (symmetric A, A_p = A): stream only the upper tile triangle of E^-1
  if (d >= kSymvMinD && d <= kSymvMaxD && symmetric && !c->prof) {
    c->sym = 1;
    c->ntiles = symv_tiles(d);
    DKD(big_alloc((void**)&c->P, (size_t)c->ntiles * 1024 * sizeof(double), s));
    DKD(cudaMallocAsync(&c->rowpart, (size_t)c->ntiles * 32 * sizeof(double), s));
    DKD(cudaMallocAsync(&c->colpart, (size_t)c->ntiles * 32 * sizeof(double), s));
    launch_symv_pack(c->Einv, d, c->ld, c->P, s);
    DKD(cudaGetLastError());
    std::vector<int> sp, ss;
    symv_segments(d, sp, ss);
    DKD(cudaMallocAsync(&c->seg_ptr, sp.size() * sizeof(int), s));
    DKD(cudaMallocAsync(&c->seg_slot, ss.size() * sizeof(int), s));
    DKD(cudaMemcpyAsync(c->seg_ptr, sp.data(), sp.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    DKD(cudaMemcpyAsync(c->seg_slot, ss.data(), ss.size() * sizeof(int), cudaMemcpyHostToDevice,
                        s));
    DKD(cudaStreamSynchronize(s));
  }
  tr.mark("packed E^-1");
  // x* = Z E^-1 Z^T b  (deflation.py:88)
  cudaEventRecord(e0, s);
  if (b) {
    int rc = upload(op, op->t, b);
    if (rc) {
      dk_defl_destroy(c);
      return rc;
    }
    coarse_solve(op, c, ST_IDENT, false, false, op->t, nullptr, nullptr, nullptr, nullptr);
    launch_bcast(c->lab, c->y, c->xs, n_pad, s);
  }
  cudaEventRecord(e1, s);
  DKD(cudaStreamSynchronize(s));
  cudaEventElapsedTime(&c->ms[3], e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  DKD(cudaGetLastError());
  *out = c;
#undef DKD
  return DK_OK;
}

// Dense basis context (deflation.py:71-89 for a general n x d Z, d <= kDenseMaxD): rows Z_k
// (written by `fill`), A_p Z_k by the stencil, E_ik = Z_i . A_p Z_k by multi-dots, pivoted
// LU + E^-1 (the reference's singularity rule), x* = Z E^-1 Z^T b.
int dk_dense_lu(int64_t n, const double* a, double* lu, int32_t* piv, double* min_pivot) {
  if (n < 1 || n >= (1ll << 31)) return fail(DK_EINVAL, "matrix order must be in [1, 2^31)");
  if (!a || !lu || !piv) return fail(DK_EINVAL, "null argument");
  int cnt = 0;
  if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt < 1) {
    cudaGetLastError();
    return fail(DK_ECUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  }
  const int d = (int)n;
  const size_t row = (size_t)d * sizeof(double);
  cudaStream_t s;
  DK_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  double* E = nullptr;
  int* dpiv = nullptr;
  double mp = 0.0;
  cudaError_t e = cudaMallocAsync(&E, row * d, s);
  if (e == cudaSuccess) e = cudaMallocAsync(&dpiv, (size_t)d * sizeof(int), s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(E, a, row * d, cudaMemcpyDefault, s);
  // the pivoted panel path always: pivots are LAPACK getrf's (first row of maximal |a|)
  if (e == cudaSuccess) e = (cudaError_t)lu_factor(E, d, d, dpiv, false, &mp, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(lu, E, row * d, cudaMemcpyDefault, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(piv, dpiv, (size_t)d * sizeof(int), cudaMemcpyDefault, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(E, s);
  cudaFreeAsync(dpiv, s);
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (e != cudaSuccess) return cuda_fail(e, "dk_dense_lu");
  if (min_pivot) *min_pivot = mp;
  if (!(mp >= 1e-300)) return fail(DK_ESINGULAR, "zero pivot in LU factorization");
  return DK_OK;
}

int dk_lu_solve(int64_t n, const double* lu, const int32_t* piv, int64_t nrhs, const double* b,
                double* x) {
  if (n < 1 || n >= (1ll << 31)) return fail(DK_EINVAL, "matrix order must be in [1, 2^31)");
  if (nrhs < 1 || nrhs >= (1ll << 31)) return fail(DK_EINVAL, "nrhs must be >= 1");
  if (!lu || !piv || !b || !x) return fail(DK_EINVAL, "null argument");
  int cnt = 0;
  if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt < 1) {
    cudaGetLastError();
    return fail(DK_ECUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  }
  const int d = (int)n, nc = (int)nrhs;
  cudaStream_t s;
  DK_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  double *E = nullptr, *X = nullptr;
  int* dpiv = nullptr;
  cudaError_t e = cudaMallocAsync(&E, (size_t)d * d * sizeof(double), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&X, (size_t)d * nc * sizeof(double), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&dpiv, (size_t)d * sizeof(int), s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(E, lu, (size_t)d * d * sizeof(double), cudaMemcpyDefault, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dpiv, piv, (size_t)d * sizeof(int), cudaMemcpyDefault, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(X, b, (size_t)d * nc * sizeof(double), cudaMemcpyDefault, s);
  if (e == cudaSuccess) {
    lu_solve_rows(E, d, d, dpiv, X, nc, nc, false, s);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(x, X, (size_t)d * nc * sizeof(double), cudaMemcpyDefault, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(E, s);
  cudaFreeAsync(X, s);
  cudaFreeAsync(dpiv, s);
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (e != cudaSuccess) return cuda_fail(e, "dk_lu_solve");
  return DK_OK;
}

}  // extern "C"
template <class Fill>
static int defl_create_dense(dk_defl** out, dk_op* op, int32_t d, int32_t ap_choice,
                             const double* b, Fill fill) {
  if (!out || !op) return fail(DK_EINVAL, "null argument");
  *out = nullptr;
  if (d < 1) return fail(DK_EINVAL, "Z must be n x d with d >= 1");
  if (d > kDenseMaxD)
    return fail(DK_EUNSUPPORTED, "dense deflation bases are limited to 64 columns");
  if (ap_choice != DK_AP_A && ap_choice != DK_AP_AM)
    return fail(DK_EINVAL, "A_p_choice must be 'A' or 'AM'");
  if (ap_choice == DK_AP_AM && op->inv == nullptr) ap_choice = DK_AP_A;
  cudaStream_t s = op->stream;
  {
    int rc = ensure_part(op, kDenseMaxD + 4);
    if (rc) return rc;
  }
  dk_defl* c = new dk_defl();
  c->op = op;
  c->serial = ++g_ctx_serial;
  c->d = d;
  c->ld = (int)round_up(d, 2);
  c->ap = ap_choice;
  c->dense = 1;
  c->zs = op->n_pad + op->guard;
  auto cleanup_fail = [&](cudaError_t e, const char* where) {
    dk_defl_destroy(c);
    return cuda_fail(e, where);
  };
#define DKD(x)                                           \
  do {                                                   \
    cudaError_t _e = (x);                                \
    if (_e != cudaSuccess) return cleanup_fail(_e, #x);  \
  } while (0)
  const size_t rows_bytes = ((size_t)op->guard + (size_t)d * c->zs) * sizeof(double);
  DKD(cudaMallocAsync(&c->Z_base, rows_bytes, s));
  DKD(cudaMallocAsync(&c->AZ_base, rows_bytes, s));
  DKD(cudaMemsetAsync(c->Z_base, 0, rows_bytes, s));
  DKD(cudaMemsetAsync(c->AZ_base, 0, rows_bytes, s));
  c->Z = c->Z_base + op->guard;
  c->AZ = c->AZ_base + op->guard;
  DKD(big_alloc((void**)&c->E, (size_t)d * c->ld * sizeof(double), s));
  DKD(big_alloc((void**)&c->Einv, (size_t)d * c->ld * sizeof(double), s));
  DKD(cudaMemsetAsync(c->E, 0, (size_t)d * c->ld * sizeof(double), s));
  DKD(cudaMallocAsync(&c->piv, (size_t)d * sizeof(int), s));
  DKD(cudaMallocAsync(&c->s, (size_t)c->ld * sizeof(double), s));
  DKD(cudaMallocAsync(&c->y, (size_t)c->ld * sizeof(double), s));
  DKD(cudaMemsetAsync(c->y, 0, (size_t)c->ld * sizeof(double), s));
  DKD(cudaMallocAsync(&c->xs_base, (size_t)op->vlen * sizeof(double), s));
  DKD(cudaMemsetAsync(c->xs_base, 0, (size_t)op->vlen * sizeof(double), s));
  c->xs = c->xs_base + op->guard;
  DKD(cudaMallocAsync(&c->qv_base, (size_t)op->vlen * sizeof(double), s));
  DKD(cudaMemsetAsync(c->qv_base, 0, (size_t)op->vlen * sizeof(double), s));
  {
    const int rc = fill(c);
    if (rc) {
      dk_defl_destroy(c);
      return rc;
    }
  }
  c->pro.az = c->AZ;
  c->pro.azs = c->zs;
  c->pro.dz = d;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  const bool am = ap_choice == DK_AP_AM;
  const Dia Ap = make_dia(op, am);
  for (int k = 0; k < d; ++k)  // A_p Z_k
    launch_stencil(ST_APPLY, am, true, Ap, op->n_pad, c->Z + (long long)k * c->zs, nullptr,
                   nullptr, c->AZ + (long long)k * c->zs, nullptr, nullptr, s);
  for (int k = 0; k < d; ++k)  // column k of E: Z_i . A_p Z_k
    launch_zdots(c->AZ + (long long)k * c->zs, c->Z, c->zs, d, op->n_pad, op->part, op->G,
                 op->tickets + 2, nullptr, 0, c->E + k, c->ld, nullptr, s);
  DKD(cudaGetLastError());
  cudaEventRecord(e1, s);
  DKD(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&c->ms[0], e0, e1);
  double* Ework = nullptr;
  DKD(big_alloc((void**)&Ework, (size_t)d * c->ld * sizeof(double), s));
  DKD(cudaMemcpyAsync(Ework, c->E, (size_t)d * c->ld * sizeof(double), cudaMemcpyDeviceToDevice,
                      s));
  double min_piv = 0.0;
  int err = lu_and_inverse(Ework, d, c->ld, c->Einv, c->piv, &min_piv, &c->ms[1], &c->ms[2], s);
  big_free(Ework, s);
  if (err) return cleanup_fail((cudaError_t)err, "lu_and_inverse");
  if (!(min_piv >= 1e-300)) {  // sparse.py:135-136
    dk_defl_destroy(c);
    return fail(DK_ESINGULAR, "zero pivot in LU factorization");
  }
  cudaEventRecord(e0, s);
  if (b) {  // x* = Z E^-1 Z^T b  (deflation.py:88)
    int rc = upload(op, op->t, b);
    if (rc) {
      dk_defl_destroy(c);
      return rc;
    }
    launch_zdots(op->t, c->Z, c->zs, d, op->n_pad, op->part, op->G, op->tickets + 2, c->Einv,
                 c->ld, c->y, 1, nullptr, s);
    launch_dense_recon(c->Z, c->zs, d, c->y, nullptr, nullptr, c->xs, op->n_pad, 1, s);
  }
  cudaEventRecord(e1, s);
  DKD(cudaStreamSynchronize(s));
  cudaEventElapsedTime(&c->ms[3], e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  DKD(cudaGetLastError());
  *out = c;
#undef DKD
  return DK_OK;
}
extern "C" {

int dk_defl_create_dense(dk_defl** out, dk_op* op, const double* Z, int32_t d, int32_t ap_choice,
                         const double* b) {
  if (!Z) return fail(DK_EINVAL, "null argument");
  return defl_create_dense(out, op, d, ap_choice, b, [&](dk_defl* c) -> int {
    DK_TRY(cudaMemcpy2DAsync(c->Z, (size_t)c->zs * sizeof(double), Z,
                             (size_t)op->n * sizeof(double), (size_t)op->n * sizeof(double), d,
                             cudaMemcpyDefault, op->stream));
    return DK_OK;
  });
}

int dk_defl_create_ritz(dk_defl** out, dk_op* op, const double* Y, int32_t rows, int32_t d,
                        int32_t ap_choice, const double* b) {
  if (!Y || !op) return fail(DK_EINVAL, "null argument");
  if (!op->has_last) return fail(DK_EINVAL, "no Arnoldi cycle to combine");
  if (rows < 1 || rows > op->st_host->last_cols)
    return fail(DK_EINVAL, "coefficient rows must be in [1, last cycle columns]");
  return defl_create_dense(out, op, d, ap_choice, b, [&](dk_defl* c) -> int {
    double* Yd = nullptr;
    DK_TRY(cudaMallocAsync(&Yd, (size_t)rows * d * sizeof(double), op->stream));
    DK_TRY(cudaMemcpyAsync(Yd, Y, (size_t)rows * d * sizeof(double), cudaMemcpyDefault,
                           op->stream));
    launch_combine_rows(op->V_base + op->guard, op->vstride, op->sc.sigma, rows, Yd, d, c->Z,
                        c->zs, op->n_pad, op->stream);
    DK_TRY(cudaGetLastError());
    DK_TRY(cudaFreeAsync(Yd, op->stream));
    return DK_OK;
  });
}

int dk_defl_destroy(dk_defl* c) {
  if (!c) return DK_OK;
  cudaStream_t s = c->op ? c->op->stream : nullptr;
  if (c->op) cudaStreamSynchronize(s);
  // every buffer of a context comes from the stream-ordered pool: no device-wide
  // synchronisation or OS-level free on destruction
  big_free(c->E, s);
  big_free(c->Einv, s);
  big_free(c->P, s);
  big_free(c->T1, s);
  free_stream(c->tg1, s);
  free_stream(c->tg2, s);
  void* bufs[] = {c->perm,     c->iperm,        c->tv,
                  c->Z_base,   c->AZ_base,
                  c->lab_base, c->tile_run_off, c->run_part, c->lab_run_ptr, c->run_slot,
                  c->piv,      c->xs_base,      c->s,        c->y,           c->qv_base,
                  c->rowpart,  c->colpart,      c->own_base, c->mask_base,   c->flab_base, c->fco_base, c->seg_ptr,
                  c->seg_slot, c->long_ids,    c->run_part2,    c->cmat};
  for (void* p : bufs)
    if (p) cudaFreeAsync(p, s);
  if (c->op) cudaStreamSynchronize(s);
  delete c;
  return DK_OK;
}

int dk_defl_apply_p1(dk_defl* c, const double* v, double* out) {
  if (!c || !v || !out) return fail(DK_EINVAL, "null argument");
  dk_op* op = c->op;
  int rc = upload(op, op->t, v);
  if (rc) return rc;
  coarse_solve(op, c, ST_IDENT, false, false, op->t, nullptr, nullptr, nullptr, nullptr);
  const bool am = c->ap == DK_AP_AM;
  launch_project(PJ_PLAIN, defl_kind(c), am, make_dia(op, am), c->pro, c->y, op->t, op->w, nullptr, 0, 0,
                 op->n_pad, op->part, op->G, op->sc, 0, op->one, op->stream);
  DK_TRY(cudaGetLastError());
  rc = download(op, out, op->w, op->n);
  if (rc) return rc;
  DK_TRY(cudaStreamSynchronize(op->stream));
  return DK_OK;
}

static int p2_into(dk_defl* c, const double* v, double* dst, bool add_xstar) {
  dk_op* op = c->op;
  int rc = upload(op, op->t, v);
  if (rc) return rc;
  const bool am = c->ap == DK_AP_AM;
  coarse_solve(op, c, ST_APPLY, am, false, op->t, nullptr, nullptr, nullptr, nullptr);
  if (c->dense)
    launch_dense_recon(c->Z, c->zs, c->d, c->y, c->xs, op->t, op->w, op->n_pad,
                       add_xstar ? 0 : 2, op->stream);
  else if (add_xstar) launch_recon(c->lab, c->y, c->xs, op->t, op->w, op->n_pad, op->stream);
  else launch_sub_bcast(c->lab, c->y, op->t, op->w, op->n_pad, op->stream);
  DK_TRY(cudaGetLastError());
  rc = download(op, dst, op->w, op->n);
  if (rc) return rc;
  DK_TRY(cudaStreamSynchronize(op->stream));
  return DK_OK;
}

int dk_defl_apply_p2(dk_defl* c, const double* v, double* out) {
  if (!c || !v || !out) return fail(DK_EINVAL, "null argument");
  return p2_into(c, v, out, false);
}

int dk_defl_reconstruct(dk_defl* c, const double* xhat, double* out) {
  if (!c || !xhat || !out) return fail(DK_EINVAL, "null argument");
  return p2_into(c, xhat, out, true);
}

int dk_defl_x_star(dk_defl* c, double* out) {
  if (!c || !out) return fail(DK_EINVAL, "null argument");
  int rc = download(c->op, out, c->xs, c->op->n);
  if (rc) return rc;
  DK_TRY(cudaStreamSynchronize(c->op->stream));
  return DK_OK;
}

int dk_defl_coarse(dk_defl* c, double* E, double* Einv) {
  if (!c) return fail(DK_EINVAL, "null argument");
  cudaStream_t s = c->op->stream;
  if (E)
    DK_TRY(cudaMemcpy2DAsync(E, (size_t)c->d * sizeof(double), c->E, (size_t)c->ld * sizeof(double),
                             (size_t)c->d * sizeof(double), c->d, cudaMemcpyDefault, s));
  if (Einv && c->prof) {  // E^-1 = P^T (W^T W) P, formed on request
    const size_t eb = (size_t)c->d * c->ld * sizeof(double);
    double *X = nullptr, *Y = nullptr;
    DK_TRY(big_alloc((void**)&X, eb, s));
    DK_TRY(big_alloc((void**)&Y, eb, s));
    lauum_into(c->Einv, c->d, c->ld, X, s);
    launch_unpermute_sym(X, c->d, c->ld, c->perm, Y, c->ld, s);
    DK_TRY(cudaMemcpy2DAsync(Einv, (size_t)c->d * sizeof(double), Y,
                             (size_t)c->ld * sizeof(double), (size_t)c->d * sizeof(double), c->d,
                             cudaMemcpyDefault, s));
    big_free(X, s);
    big_free(Y, s);
  } else if (Einv) {
    DK_TRY(cudaMemcpy2DAsync(Einv, (size_t)c->d * sizeof(double), c->Einv,
                             (size_t)c->ld * sizeof(double), (size_t)c->d * sizeof(double), c->d,
                             cudaMemcpyDefault, s));
  }
  DK_TRY(cudaStreamSynchronize(s));
  return DK_OK;
}

int dk_defl_coarse_kind(dk_defl* c, int32_t* kind, int64_t* tiles) {
  if (!c || !kind || !tiles) return fail(DK_EINVAL, "null argument");
  const long long nb = (c->d + 31) / 32;
  *kind = c->dense ? 3 : c->prof ? 2 : c->sym ? 1 : 0;
  *tiles = c->dense ? 0 : c->prof ? c->tg1.nt + c->tg2.nt : c->sym ? c->ntiles : nb * nb;
  return DK_OK;
}

int dk_defl_setup_ms(dk_defl* c, double* ms4) {
  if (!c || !ms4) return fail(DK_EINVAL, "null argument");
  for (int k = 0; k < 4; ++k) ms4[k] = c->ms[k];
  return DK_OK;
}

// ---- solver -------------------------------------------------------------------------------
int dk_gmres_ex(dk_op* op, dk_defl* c, const double* b, const double* x0, int32_t m, double tol,
                int32_t max_iters, int32_t min_iters, double* x_out, double* hist,
                int32_t* restart_of, double* hbar, double* gram, dk_solve_info* info,
                const dk_cycle_ctl* ctl_in, dk_cycle_ctl* ctl_out) {
  if (!op || !b || !x_out || !info) return fail(DK_EINVAL, "null argument");
  if (c && c->op != op) return fail(DK_EINVAL, "deflation context belongs to another operator");
  if (m < 1) return fail(DK_EINVAL, "cycle size must be >= 1");
  if (max_iters < 0) max_iters = 0;
  int rc = ensure_work(op, m, max_iters);
  if (rc) return rc;
  op->launches = 0;
  if ((rc = upload(op, op->b, b))) return rc;
  // resuming with x0 == NULL continues from the device-resident iterate (and keeps the
  // original x0 for the final relative residual)
  if (!(ctl_in && ctl_in->resume && x0 == nullptr)) {
    if ((rc = upload(op, op->x0, x0))) return rc;
    DK_TRY(cudaMemcpyAsync(op->x, op->x0, (size_t)op->n_pad * sizeof(double),
                           cudaMemcpyDeviceToDevice, op->stream));
  }
  if ((rc = setup_split(op, c, m))) return rc;
  // small problems: the cycle's Arnoldi steps in one persistent grid (not when profiling per
  // kernel, not with the nested-dissection / dense-basis coarse paths)
  op->small = !op->prof && !op->split && (!c || (!c->dense && !c->prof)) &&
              cycle_small_ok(op->n_pad, m, c ? c->d : 0);
  launch_init_state(op->sc, tol, m, max_iters, min_iters, op->stream);
  op->launches += 1;
  const bool resume = ctl_in && ctl_in->resume;
  if (resume) {  // continue a solve: counters, convergence denominator, restart history
    launch_resume_state(op->sc, ctl_in->iterations, ctl_in->cycles, ctl_in->warning,
                        ctl_in->has_prev, ctl_in->denom, ctl_in->prev_beta, op->stream);
    op->launches += 1;
  }
  const int max_cycles = ctl_in ? ctl_in->max_cycles : 0;
  // krylov.py:127: no cycle starts once max_iters is reached (the caller's earlier calls)
  const bool run_cycles = !(resume && ctl_in->iterations >= max_iters);
  // The cycle is a CUDA graph.  A repeated solve with the same (context, m) builds it up
  // front; a one-off solve (the public pdgmres path: a fresh context per call) launches its
  // first cycle eagerly and captures + instantiates the graph on the host while the GPU runs
  // that cycle, so the remaining cycles replay it (DK_NO_LATE_GRAPH: eager throughout).
  const unsigned long long key =
      (c ? c->serial : 0ull) * 4 + (op->split ? 1 : 0) + (op->small ? 2 : 0);
  bool use_graph =
      !op->prof && ((op->gexec && op->g_m == m && op->g_ctx == key) ||
                    (op->seen_m == m && op->seen_ctx == key));
  static const bool late_graph_off = getenv("DK_NO_LATE_GRAPH") != nullptr;
  op->seen_m = m;
  op->seen_ctx = key;
  if (use_graph) {
    rc = build_graph(op, c, m);
    if (rc) return rc;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, op->stream);
  // stencil (+ restrict + E^-1 s; dense: one multi-dot)
  const int coarse_launches =
      !c ? 1
         : c->dense ? 2
         : c->prof  ? 1 + (op->split ? 1 + tgemv_launches(c->tg1)
                                       : tgemv_restrict_launches(c->tg1)) +
                          tgemv_launches(c->tg2)
         : c->sym   ? 4
                    : 3;
  // restart (stencil chain + projection), m x (stencil chain, projection, update [+ the
  // separate second pass]), cycle end, x update
  const int per_cycle_launches =
      op->small ? coarse_launches + 1 + 1 + 2
                : coarse_launches + 1 +
                      m * (coarse_launches + (op->gs_fuse ? 2 : 4) + (op->split ? 1 : 0)) + 2;
  long long guard_cycles = run_cycles ? (long long)max_iters + 2 : 0;
  if (max_cycles > 0 && guard_cycles > max_cycles) guard_cycles = max_cycles;
  op->host_syncs = 0;
  op->used_loop = 0;
  for (long long cyc = 0; cyc < guard_cycles; ++cyc) {
    if (use_graph && op->g_loop) {
      // every remaining cycle in one launch: the WHILE node's condition is set on the device
      const long long left = guard_cycles - cyc;
      launch_loop_arm(op->sc, (int)std::min<long long>(left, INT_MAX), op->stream);
      DK_TRY(cudaGraphLaunch(op->gexec, op->stream));
      if ((rc = read_state(op))) return rc;
      op->host_syncs += 1;
      op->used_loop = 1;
      const long long ran = left - op->st_host->loop_left;
      op->launches += 1 + (int)ran * (per_cycle_launches + 1);
      break;
    }
    if (use_graph) {
      DK_TRY(cudaGraphLaunch(op->gexec, op->stream));
      op->launches += per_cycle_launches;
    } else if (!op->prof) {
      const int l0 = op->launches;
      issue_cycle(op, c, m);
      op->launches = l0 + per_cycle_launches;
      DK_TRY(launch_error());
      if (cyc == 0 && guard_cycles > 1 && !late_graph_off) {
        // the stream still holds this cycle's work; capture records only what follows.  The
        // state copy queued behind the cycle is polled, never waited for: a solve that ended
        // in its first cycle while the host was building the graph stops here.
        cudaEvent_t es;
        DK_TRY(cudaEventCreateWithFlags(&es, cudaEventDisableTiming));
        DK_TRY(cudaMemcpyAsync(op->st_host, op->st, sizeof(State), cudaMemcpyDeviceToHost,
                               op->stream));
        DK_TRY(cudaEventRecord(es, op->stream));
        rc = build_graph(op, c, m);
        const bool landed = cudaEventQuery(es) == cudaSuccess;
        cudaEventDestroy(es);
        if (rc) return rc;
        use_graph = true;  // from the next cycle on
        if (op->g_loop) {
          if (landed && !op->st_host->running) break;
          continue;  // no host wait in between: a finished solve's loop body is gated off
        }
      }
    } else {
      issue_restart(op, c);
      if ((rc = read_state(op))) return rc;
      for (int j = 0; j < m && op->st_host->active; ++j) {
        issue_iteration(op, c, j);
        if ((rc = read_state(op))) return rc;
      }
      issue_cycle_end(op);
      prof_collect(op);
    }
    if ((rc = read_state(op))) return rc;
    op->host_syncs += 1;
    if (!op->st_host->running) break;
  }
  cudaEventRecord(e1, op->stream);
  DK_TRY(cudaEventSynchronize(e1));
  float solve_ms = 0.f;
  cudaEventElapsedTime(&solve_ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  DK_TRY(cudaGetLastError());
  // finalize: reconstruct (krylov.py:220-221), true residuals (:222-225)
  double* xf = op->x;
  if (c) {
    const bool am = c->ap == DK_AP_AM;
    coarse_solve(op, c, ST_APPLY, am, false, op->x, nullptr, nullptr, nullptr, nullptr);
    if (c->dense)
      launch_dense_recon(c->Z, c->zs, c->d, c->y, c->xs, op->x, op->t, op->n_pad, 0, op->stream);
    else
      launch_recon(c->lab, c->y, c->xs, op->x, op->t, op->n_pad, op->stream);
    xf = op->t;
    op->launches += 4;
  }
  const Dia A = make_dia(op, false);
  launch_stencil(ST_RESID, false, true, A, op->n_pad, xf, nullptr, op->b, op->w, nullptr, nullptr,
                 op->stream);
  launch_norm(op->w, op->n_pad, op->part, op->G, op->tickets + 0, op->nrm + 0, op->stream);
  launch_stencil(ST_RESID, false, true, A, op->n_pad, op->x0, nullptr, op->b, op->w, nullptr,
                 nullptr, op->stream);
  launch_norm(op->w, op->n_pad, op->part, op->G, op->tickets + 1, op->nrm + 1, op->stream);
  op->launches += 4;
  DK_TRY(cudaGetLastError());
  double nr[2] = {0, 0};
  DK_TRY(cudaMemcpyAsync(nr, op->nrm, 2 * sizeof(double), cudaMemcpyDeviceToHost, op->stream));
  if ((rc = read_state(op))) return rc;
  const State& S = *op->st_host;
  if ((rc = download(op, x_out, xf, op->n))) return rc;
  if (hist) DK_TRY(cudaMemcpyAsync(hist, op->hist, (size_t)(S.iterations + 1) * sizeof(double),
                                   cudaMemcpyDefault, op->stream));
  if (restart_of)
    DK_TRY(cudaMemcpyAsync(restart_of, op->rof, (size_t)(S.iterations + 1) * sizeof(int),
                           cudaMemcpyDefault, op->stream));
  if (hbar)
    DK_TRY(cudaMemcpyAsync(hbar, op->sc.H, (size_t)(m + 1) * m * sizeof(double),
                           cudaMemcpyDefault, op->stream));
  std::vector<double> gm, gc, sg;
  if (gram) {
    gm.resize((size_t)(m + 1) * (m + 1));
    gc.resize(m + 1);
    sg.resize(m + 1);
    DK_TRY(cudaMemcpyAsync(gm.data(), op->sc.Gm, gm.size() * sizeof(double),
                           cudaMemcpyDeviceToHost, op->stream));
    DK_TRY(cudaMemcpyAsync(gc.data(), op->sc.gcol, gc.size() * sizeof(double),
                           cudaMemcpyDeviceToHost, op->stream));
    DK_TRY(cudaMemcpyAsync(sg.data(), op->sc.sigma, sg.size() * sizeof(double),
                           cudaMemcpyDeviceToHost, op->stream));
  }
  DK_TRY(cudaStreamSynchronize(op->stream));
  if (gram) {
    // V_{cols+1}^T V_cols of the last cycle, (m+1) x m column-major: the Gram matrix the
    // re-orthogonalisation test maintains, last row sigma_cols V^T u (0 if the cycle stopped
    // before storing that vector, as the reference leaves V[cols] zero)
    const int cols = S.last_cols;
    for (size_t e = 0; e < (size_t)(m + 1) * m; ++e) gram[e] = 0.0;
    for (int k = 0; k < cols; ++k)
      for (int i = 0; i <= cols; ++i) {
        double g;
        if (i == cols && cols == S.cycle_cols) g = S.last_broke ? 0.0 : sg[cols] * gc[k];
        else if (i <= k) g = gm[(size_t)k * (m + 1) + i];
        else g = gm[(size_t)i * (m + 1) + k];
        gram[(size_t)k * (m + 1) + i] = g;
      }
  }
  info->iterations = S.iterations;
  info->cycles = S.cycle;
  info->restarts = std::max(S.cycle - 1, 0);
  info->converged = S.converged;
  info->warning = S.warning;
  info->last_cols = S.last_cols;
  info->reorths = S.reorths;
  info->kernel_launches = op->launches;
  info->final_relres = nr[0] / (nr[1] > 0 ? nr[1] : 1.0);
  info->solve_seconds = solve_ms * 1e-3;
  op->has_last = S.cycle > 0;
  if (ctl_out) {
    ctl_out->max_cycles = max_cycles;
    ctl_out->resume = 1;
    ctl_out->iterations = S.iterations;
    ctl_out->cycles = S.cycle;
    ctl_out->warning = S.warning;
    ctl_out->has_prev = S.has_prev;
    ctl_out->converged = S.converged;
    ctl_out->running = S.running && !S.converged && S.iterations < max_iters && S.last_cols > 0;
    ctl_out->denom = S.denom;
    ctl_out->prev_beta = S.prev_beta;
  }
  return DK_OK;
}

int dk_gmres(dk_op* op, dk_defl* c, const double* b, const double* x0, int32_t m, double tol,
             int32_t max_iters, int32_t min_iters, double* x_out, double* hist,
             int32_t* restart_of, double* hbar, dk_solve_info* info) {
  return dk_gmres_ex(op, c, b, x0, m, tol, max_iters, min_iters, x_out, hist, restart_of, hbar,
                     nullptr, info, nullptr, nullptr);
}

int dk_op_solve_stats(dk_op* op, int32_t* host_syncs, int32_t* device_loop) {
  if (!op || !host_syncs || !device_loop) return fail(DK_EINVAL, "null argument");
  *host_syncs = op->host_syncs;
  *device_loop = op->used_loop;
  return DK_OK;
}

int dk_last_basis_vector(dk_op* op, int32_t i, double* out) {
  if (!op || !out) return fail(DK_EINVAL, "null argument");
  if (!op->has_last || i < 0 || i >= op->v_rows) return fail(DK_EINVAL, "no such basis vector");
  const State& S = *op->st_host;
  if (i > S.last_cols) return fail(DK_EINVAL, "basis index beyond the last cycle");
  double* V = op->V_base + op->guard;
  if (i == S.cycle_cols && S.last_broke) {
    // the reference never fills V[j+1] when the cycle stopped at j (krylov.py:195-197)
    DK_TRY(cudaMemsetAsync(op->t, 0, (size_t)op->n * sizeof(double), op->stream));
  } else {
    k_scale_copy<<<num_sms() * 4, 256, 0, op->stream>>>(V + (long long)i * op->vstride, op->sc.sigma + i,
                                                  op->t, op->n);
  }
  DK_TRY(cudaGetLastError());
  int rc = download(op, out, op->t, op->n);
  if (rc) return rc;
  DK_TRY(cudaStreamSynchronize(op->stream));
  return DK_OK;
}

int dk_levelset_labels_device(int64_t nx, int64_t ny, int64_t nz, const int64_t* band,
                              int32_t px, int32_t py, int32_t pz, int64_t* labels,
                              int64_t* ncomp, int64_t* comp_band) {
  if (nx < 1 || ny < 1 || nz < 1) return fail(DK_EINVAL, "cell counts must be >= 1");
  if (px < 1 || py < 1 || pz < 1 || px > nx || py > ny || pz > nz)
    return fail(DK_EINVAL, "subdomain counts must be in [1, cells]");
  if (!band || !labels || !ncomp || !comp_band) return fail(DK_EINVAL, "null argument");
  if (nx * ny * nz >= (1ll << 31)) return fail(DK_EUNSUPPORTED, "grid too large for int32 ids");
  int cnt = 0;
  if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt < 1) {
    cudaGetLastError();
    return fail(DK_ECUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  }
  cudaStream_t s;
  DK_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  std::string where;
  long long nc = 0;
  const int e = device_levelset_labels(nx, ny, nz, reinterpret_cast<const long long*>(band), px,
                                       py, pz, reinterpret_cast<long long*>(labels), &nc,
                                       reinterpret_cast<long long*>(comp_band), s, where);
  cudaStreamDestroy(s);
  if (e) return cuda_fail((cudaError_t)e, where.c_str());
  *ncomp = nc;
  return DK_OK;
}

int dk_assemble_tpfa(int32_t nx, int32_t ny, int32_t nz, double dx, double dy, double dz,
                     const double* kx, const double* ky, const double* kz, const double* q,
                     int32_t nfaces, const int32_t* face_ids, const double* face_values,
                     double boundary_perm, double* diags_out, double* b_out) {
  if (nx < 1 || ny < 1 || nz < 1) return fail(DK_EINVAL, "cell counts must be >= 1");
  if (!(dx > 0 && dy > 0 && dz > 0)) return fail(DK_EINVAL, "cell sizes must be positive");
  if (!kx || !ky || !kz || !diags_out || !b_out) return fail(DK_EINVAL, "null argument");
  if (nfaces < 0 || nfaces > 6 || (nfaces > 0 && (!face_ids || !face_values)))
    return fail(DK_EINVAL, "at most 6 Dirichlet faces");
  for (int f = 0; f < nfaces; ++f)
    if (face_ids[f] < 0 || face_ids[f] > 5) return fail(DK_EINVAL, "face id must be 0..5");
  if ((long long)nx * ny * nz >= (1ll << 31)) return fail(DK_EUNSUPPORTED, "grid too large");
  int cnt = 0;
  if (cudaGetDeviceCount(&cnt) != cudaSuccess || cnt < 1) {
    cudaGetLastError();
    return fail(DK_ECUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  }
  cudaStream_t s;
  DK_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  std::string where;
  const int e = device_assemble_tpfa(nx, ny, nz, dx, dy, dz, kx, ky, kz, q, nfaces, face_ids,
                                     face_values, boundary_perm, diags_out, b_out, s, where);
  cudaStreamDestroy(s);
  if (e) return cuda_fail((cudaError_t)e, where.c_str());
  return DK_OK;
}

}  // extern "C"

#ifdef DK_TIMELINE
// ---- diagnostic builds only: the kernel timeline (tools/timeline.py) -------------------
namespace dk {
void tl_set_kernels(const TlBuf& b);
void tl_set_profile(const TlBuf& b);
}  // namespace dk
static dk::TlBuf g_tl_host{};
extern "C" int dk_timeline_enable(uint32_t cap) {
  if (g_tl_host.rec) {
    cudaFree(g_tl_host.rec);
    cudaFree(g_tl_host.cnt);
    g_tl_host = {};
  }
  if (cap) {
    cudaMalloc(&g_tl_host.rec, (size_t)cap * 16);
    cudaMalloc(&g_tl_host.cnt, sizeof(unsigned));
    cudaMemset(g_tl_host.cnt, 0, sizeof(unsigned));
    g_tl_host.cap = cap;
  }
  dk::tl_set_kernels(g_tl_host);
  dk::tl_set_profile(g_tl_host);
  return (int)cudaDeviceSynchronize();
}
extern "C" int64_t dk_timeline_read(uint64_t* out, uint32_t cap) {
  unsigned n = 0;
  cudaDeviceSynchronize();
  cudaMemcpy(&n, g_tl_host.cnt, sizeof(unsigned), cudaMemcpyDeviceToHost);
  if (n > g_tl_host.cap) n = g_tl_host.cap;
  if (n > cap) n = cap;
  cudaMemcpy(out, g_tl_host.rec, (size_t)n * 16, cudaMemcpyDeviceToHost);
  cudaMemset(g_tl_host.cnt, 0, sizeof(unsigned));
  return n;
}
#endif
