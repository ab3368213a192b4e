// dk_setup.cu — problem set-up on the device:
//   * deflation-vector construction: 6-connected components of equal band inside each
//     subdomain box, numbered by first linear occurrence (physics.py:44-143) — lock-free
//     union-find whose roots are component minima, then a prefix scan over the roots;
//   * TPFA operator assembly straight into the DIA layout (testbed.py:133-211) with the
//     reference's exact arithmetic (separately rounded, face order +x, -x, +y, -y, +z, -z,
//     then the Dirichlet ghost faces in their given order).
// Both results are bit-identical to the host paths (tests/test_device_setup.py).
#include <cuda_runtime.h>

#include <cub/cub.cuh>
#include <string>
#include <vector>

#include "dk_launch.h"

namespace dk {

// ---- connected components ---------------------------------------------------------------
__device__ __forceinline__ int cc_find(int* p, int x) {
  const volatile int* vp = p;
  while (true) {
    const int px = vp[x];
    if (px == x) return x;
    const int ppx = vp[px];
    if (ppx != px) p[x] = ppx;  // path halving: any ancestor is a valid parent
    x = ppx;
  }
}

// link the larger root under the smaller: every root is the minimum index of its component
__device__ __forceinline__ void cc_unite(int* p, int a, int b) {
  while (true) {
    a = cc_find(p, a);
    b = cc_find(p, b);
    if (a == b) return;
    if (a > b) {
      const int t = a;
      a = b;
      b = t;
    }
    const int old = atomicCAS(&p[b], b, a);
    if (old == b) return;
    b = old;
  }
}

__global__ void k_cc_init(int* p, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    p[i] = (int)i;
}

__global__ void k_cc_hook(int* p, const long long* __restrict__ band, int nx, int ny, int nz,
                          const int* __restrict__ bx, const int* __restrict__ by,
                          const int* __restrict__ bz) {
  const long long nxy = (long long)nx * ny, n = nxy * nz;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int ix = (int)(i % nx), iy = (int)((i / nx) % ny), iz = (int)(i / nxy);
    const long long b = band[i];
    if (ix + 1 < nx && bx[ix] == bx[ix + 1] && band[i + 1] == b) cc_unite(p, (int)i, (int)(i + 1));
    if (iy + 1 < ny && by[iy] == by[iy + 1] && band[i + nx] == b)
      cc_unite(p, (int)i, (int)(i + nx));
    if (iz + 1 < nz && bz[iz] == bz[iz + 1] && band[i + nxy] == b)
      cc_unite(p, (int)i, (int)(i + nxy));
  }
}

// After hooking: point every cell at its root.  The walk must not path-halve — a halving
// store racing with the `p[i] = r` of another thread could replace a root pointer by a
// non-root ancestor; without halving, p[i] is written only by thread i.
__global__ void k_cc_compress(int* p, int* root_flag, long long n) {
  const volatile int* vp = p;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    int r = (int)i;
    for (int q = vp[r]; q != r; q = vp[r]) r = q;
    p[i] = r;
    root_flag[i] = (r == (int)i) ? 1 : 0;
  }
}

__global__ void k_cc_label(const int* __restrict__ p, const int* __restrict__ rank,
                           const long long* __restrict__ band, long long n,
                           long long* __restrict__ labels, long long* __restrict__ comp_band) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int r = p[i];
    labels[i] = rank[r];
    if (r == (int)i) comp_band[rank[i]] = band[i];
  }
}

static std::vector<int> block_map(long long nc, int parts) {
  std::vector<int> out(nc);
  const long long base = nc / parts, rem = nc % parts;
  long long start = 0;
  for (int b = 0; b < parts; ++b) {
    const long long size = base + (b < rem ? 1 : 0);
    for (long long i = start; i < start + size; ++i) out[i] = b;
    start += size;
  }
  return out;
}

int device_levelset_labels(long long nx, long long ny, long long nz, const long long* band_in,
                           int px, int py, int pz, long long* labels_out, long long* ncomp,
                           long long* comp_band_out, cudaStream_t s, std::string& err) {
  const long long n = nx * ny * nz;
  long long *band = nullptr, *labels = nullptr, *cband = nullptr;
  int *p = nullptr, *flag = nullptr, *rank = nullptr, *bxyz = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  int last_rank = 0, last_flag = 0;
  cudaError_t e = cudaSuccess;
  const unsigned grid = (unsigned)num_sms() * 8;
#define DKS(x)                     \
  do {                             \
    e = (x);                       \
    if (e != cudaSuccess) {        \
      err = #x;                    \
      goto done;                   \
    }                              \
  } while (0)
  {
    std::vector<int> bx = block_map(nx, px), by = block_map(ny, py), bz = block_map(nz, pz);
    std::vector<int> all;
    all.insert(all.end(), bx.begin(), bx.end());
    all.insert(all.end(), by.begin(), by.end());
    all.insert(all.end(), bz.begin(), bz.end());
    DKS(cudaMallocAsync(&band, n * sizeof(long long), s));
    DKS(cudaMallocAsync(&labels, n * sizeof(long long), s));
    DKS(cudaMallocAsync(&cband, n * sizeof(long long), s));
    DKS(cudaMallocAsync(&p, n * sizeof(int), s));
    DKS(cudaMallocAsync(&flag, n * sizeof(int), s));
    DKS(cudaMallocAsync(&rank, n * sizeof(int), s));
    DKS(cudaMallocAsync(&bxyz, all.size() * sizeof(int), s));
    DKS(cudaMemcpyAsync(band, band_in, n * sizeof(long long), cudaMemcpyDefault, s));
    DKS(cudaMemcpyAsync(bxyz, all.data(), all.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    DKS(cudaStreamSynchronize(s));
    k_cc_init<<<grid, 256, 0, s>>>(p, n);
    k_cc_hook<<<grid, 256, 0, s>>>(p, band, (int)nx, (int)ny, (int)nz, bxyz, bxyz + nx,
                                   bxyz + nx + ny);
    k_cc_compress<<<grid, 256, 0, s>>>(p, flag, n);
    DKS(cudaGetLastError());
    DKS(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, flag, rank, (int)n, s));
    DKS(cudaMallocAsync(&tmp, tmp_bytes, s));
    DKS(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flag, rank, (int)n, s));
    k_cc_label<<<grid, 256, 0, s>>>(p, rank, band, n, labels, cband);
    DKS(cudaGetLastError());
    DKS(cudaMemcpyAsync(&last_rank, rank + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    DKS(cudaMemcpyAsync(&last_flag, flag + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
    DKS(cudaStreamSynchronize(s));
    *ncomp = (long long)last_rank + last_flag;
    DKS(cudaMemcpyAsync(labels_out, labels, n * sizeof(long long), cudaMemcpyDefault, s));
    DKS(cudaMemcpyAsync(comp_band_out, cband, *ncomp * sizeof(long long), cudaMemcpyDefault, s));
    DKS(cudaStreamSynchronize(s));
  }
done:
  void* bufs[] = {band, labels, cband, p, flag, rank, bxyz, tmp};
  for (void* b : bufs)
    if (b) cudaFreeAsync(b, s);
  cudaStreamSynchronize(s);
  return (int)e;
#undef DKS
}

// ---- TPFA assembly ---------------------------------------------------------------------------
__device__ __forceinline__ double tpfa_t(double k1, double k2, double h1, double h2, double area) {
  if (!(k1 > 0.0 && k2 > 0.0)) return 0.0;
  // area / (0.5 * h1 / k1 + 0.5 * h2 / k2), each operation rounded as numpy does
  const double a = __ddiv_rn(__dmul_rn(0.5, h1), k1);
  const double b = __ddiv_rn(__dmul_rn(0.5, h2), k2);
  return __ddiv_rn(area, __dadd_rn(a, b));
}

struct Faces {
  int n;
  int id[6];      // 0 xmin, 1 xmax, 2 ymin, 3 ymax, 4 zmin, 5 zmax, in application order
  double val[6];
};

__global__ void k_tpfa(int nx, int ny, int nz, double dx, double dy, double dz,
                       const double* __restrict__ kx, const double* __restrict__ ky,
                       const double* __restrict__ kz, const double* __restrict__ q, Faces F,
                       double bperm, double* __restrict__ dia, double* __restrict__ b) {
  const long long nxy = (long long)nx * ny, n = nxy * nz;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int ix = (int)(i % nx), iy = (int)((i / nx) % ny), iz = (int)(i / nxy);
    const double axy = dy * dz, ayz = dx * dz, az = dx * dy;  // x-, y-, z-face areas
    const double txp = (nx > 1 && ix < nx - 1) ? tpfa_t(kx[i], kx[i + 1], dx, dx, axy) : 0.0;
    const double txm = (nx > 1 && ix > 0) ? tpfa_t(kx[i - 1], kx[i], dx, dx, axy) : 0.0;
    const double typ = (ny > 1 && iy < ny - 1) ? tpfa_t(ky[i], ky[i + nx], dy, dy, ayz) : 0.0;
    const double tym = (ny > 1 && iy > 0) ? tpfa_t(ky[i - nx], ky[i], dy, dy, ayz) : 0.0;
    const double tzp = (nz > 1 && iz < nz - 1) ? tpfa_t(kz[i], kz[i + nxy], dz, dz, az) : 0.0;
    const double tzm = (nz > 1 && iz > 0) ? tpfa_t(kz[i - nxy], kz[i], dz, dz, az) : 0.0;
    double c = 0.0;
    c = __dadd_rn(c, txp);
    c = __dadd_rn(c, txm);
    c = __dadd_rn(c, typ);
    c = __dadd_rn(c, tym);
    c = __dadd_rn(c, tzp);
    c = __dadd_rn(c, tzm);
    double bi = q ? q[i] : 0.0;
    for (int f = 0; f < F.n; ++f) {
      const int id = F.id[f];
      bool on = false;
      double t = 0.0;
      if (id == 0 && ix == 0) { on = true; t = tpfa_t(kx[i], bperm, dx, dx, axy); }
      if (id == 1 && ix == nx - 1) { on = true; t = tpfa_t(kx[i], bperm, dx, dx, axy); }
      if (id == 2 && iy == 0) { on = true; t = tpfa_t(ky[i], bperm, dy, dy, ayz); }
      if (id == 3 && iy == ny - 1) { on = true; t = tpfa_t(ky[i], bperm, dy, dy, ayz); }
      if (id == 4 && iz == 0) { on = true; t = tpfa_t(kz[i], bperm, dz, dz, az); }
      if (id == 5 && iz == nz - 1) { on = true; t = tpfa_t(kz[i], bperm, dz, dz, az); }
      if (on) {
        c = __dadd_rn(c, t);
        bi = __dadd_rn(bi, __dmul_rn(t, F.val[f]));
      }
    }
    if (c == 0.0) {  // sealed cell: identity row, zero right-hand side (testbed.py:200-205)
      c = 1.0;
      bi = 0.0;
    }
    // faces inside the grid hold -t (also -0.0 for a sealed face, as the host assembly does);
    // entries past the boundary stay +0.0
    dia[0 * n + i] = (nz > 1 && iz > 0) ? -tzm : 0.0;
    dia[1 * n + i] = (ny > 1 && iy > 0) ? -tym : 0.0;
    dia[2 * n + i] = (nx > 1 && ix > 0) ? -txm : 0.0;
    dia[3 * n + i] = c;
    dia[4 * n + i] = (nx > 1 && ix < nx - 1) ? -txp : 0.0;
    dia[5 * n + i] = (ny > 1 && iy < ny - 1) ? -typ : 0.0;
    dia[6 * n + i] = (nz > 1 && iz < nz - 1) ? -tzp : 0.0;
    b[i] = bi;
  }
}

int device_assemble_tpfa(int nx, int ny, int nz, double dx, double dy, double dz,
                         const double* kx, const double* ky, const double* kz, const double* q,
                         int nfaces, const int* face_ids, const double* face_values, double bperm,
                         double* diags_out, double* b_out, cudaStream_t s, std::string& err) {
  const long long n = (long long)nx * ny * nz;
  double *k = nullptr, *qq = nullptr, *dia = nullptr, *bb = nullptr;
  cudaError_t e = cudaSuccess;
  Faces F{};
  F.n = nfaces;
  for (int f = 0; f < nfaces && f < 6; ++f) {
    F.id[f] = face_ids[f];
    F.val[f] = face_values[f];
  }
#define DKS(x)              \
  do {                      \
    e = (x);                \
    if (e != cudaSuccess) { \
      err = #x;             \
      goto done;            \
    }                       \
  } while (0)
  DKS(cudaMallocAsync(&k, 3 * n * sizeof(double), s));
  DKS(cudaMallocAsync(&dia, 7 * n * sizeof(double), s));
  DKS(cudaMallocAsync(&bb, n * sizeof(double), s));
  DKS(cudaMemcpyAsync(k, kx, n * sizeof(double), cudaMemcpyDefault, s));
  DKS(cudaMemcpyAsync(k + n, ky, n * sizeof(double), cudaMemcpyDefault, s));
  DKS(cudaMemcpyAsync(k + 2 * n, kz, n * sizeof(double), cudaMemcpyDefault, s));
  if (q) {
    DKS(cudaMallocAsync(&qq, n * sizeof(double), s));
    DKS(cudaMemcpyAsync(qq, q, n * sizeof(double), cudaMemcpyDefault, s));
  }
  k_tpfa<<<num_sms() * 8, 256, 0, s>>>(nx, ny, nz, dx, dy, dz, k, k + n, k + 2 * n, qq, F, bperm, dia,
                                 bb);
  DKS(cudaGetLastError());
  DKS(cudaMemcpyAsync(diags_out, dia, 7 * n * sizeof(double), cudaMemcpyDefault, s));
  DKS(cudaMemcpyAsync(b_out, bb, n * sizeof(double), cudaMemcpyDefault, s));
  DKS(cudaStreamSynchronize(s));
done:
  void* bufs[] = {k, qq, dia, bb};
  for (void* p : bufs)
    if (p) cudaFreeAsync(p, s);
  cudaStreamSynchronize(s);
  return (int)e;
#undef DKS
}

}  // namespace dk
