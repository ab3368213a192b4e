// dk_labels.cpp — deflation-vector construction (host, native): 6-connected components of
// equal band inside each subdomain box, numbered by first occurrence in linear cell order.
//
// Reference semantics (physics.py): subdomain_partition boxes (:57-78, block sizes nc//p
// with the remainder added to the leading blocks), per (box, band) ndimage.label with the
// 6-neighbour structure (:119-141), then _relabel_by_first_occurrence (:44-54).  The
// reference's cost is O(n * boxes * bands); this is one union-find sweep, O(n alpha(n)).
// Linking every root to the smaller index keeps each root at its component's minimum
// linear index, so a single ascending sweep numbers components by first occurrence.
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/dk.h"

namespace {
thread_local std::string g_lab_err;

std::vector<int32_t> block_of(int64_t nc, int32_t p) {
  std::vector<int32_t> out(nc);
  const int64_t base = nc / p, rem = nc % p;
  int64_t start = 0;
  for (int32_t b = 0; b < p; ++b) {
    const int64_t size = base + (b < rem ? 1 : 0);
    for (int64_t i = start; i < start + size; ++i) out[i] = b;
    start += size;
  }
  return out;
}

template <typename Idx>
struct UnionFind {
  std::vector<Idx> parent;
  explicit UnionFind(int64_t n) : parent(n) {
    for (int64_t i = 0; i < n; ++i) parent[i] = (Idx)i;
  }
  Idx find(Idx a) {
    while (parent[a] != a) {
      parent[a] = parent[parent[a]];
      a = parent[a];
    }
    return a;
  }
  void unite(Idx a, Idx b) {
    Idx ra = find(a), rb = find(b);
    if (ra == rb) return;
    if (ra < rb) parent[rb] = ra;
    else parent[ra] = rb;
  }
};

template <typename Idx>
int label_impl(int64_t nx, int64_t ny, int64_t nz, const int64_t* band, int32_t px, int32_t py,
               int32_t pz, int64_t* labels, int64_t* ncomp, int64_t* comp_band) {
  const int64_t n = nx * ny * nz, nxy = nx * ny;
  const std::vector<int32_t> bx = block_of(nx, px), by = block_of(ny, py), bz = block_of(nz, pz);
  UnionFind<Idx> uf(n);
  for (int64_t iz = 0; iz < nz; ++iz) {
    for (int64_t iy = 0; iy < ny; ++iy) {
      const int64_t row = nx * (iy + ny * iz);
      for (int64_t ix = 0; ix < nx; ++ix) {
        const int64_t i = row + ix;
        const int64_t bi = band[i];
        if (ix + 1 < nx && bx[ix] == bx[ix + 1] && band[i + 1] == bi) uf.unite((Idx)i, (Idx)(i + 1));
        if (iy + 1 < ny && by[iy] == by[iy + 1] && band[i + nx] == bi)
          uf.unite((Idx)i, (Idx)(i + nx));
        if (iz + 1 < nz && bz[iz] == bz[iz + 1] && band[i + nxy] == bi)
          uf.unite((Idx)i, (Idx)(i + nxy));
      }
    }
  }
  int64_t next = 0;
  for (int64_t i = 0; i < n; ++i) {
    const Idx r = uf.find((Idx)i);
    if ((int64_t)r == i) {
      labels[i] = next;
      comp_band[next] = band[i];
      ++next;
    } else {
      labels[i] = labels[r];  // r < i is already numbered
    }
  }
  *ncomp = next;
  return DK_OK;
}
}  // namespace

extern "C" int dk_levelset_labels(int64_t nx, int64_t ny, int64_t nz, const int64_t* band,
                                  int32_t px, int32_t py, int32_t pz, int64_t* labels,
                                  int64_t* ncomp, int64_t* comp_band) {
  if (nx < 1 || ny < 1 || nz < 1) return DK_EINVAL;
  if (px < 1 || py < 1 || pz < 1 || px > nx || py > ny || pz > nz) return DK_EINVAL;
  if (!band || !labels || !ncomp || !comp_band) return DK_EINVAL;
  const int64_t n = nx * ny * nz;
  if (n < (int64_t)1 << 31)
    return label_impl<int32_t>(nx, ny, nz, band, px, py, pz, labels, ncomp, comp_band);
  return label_impl<int64_t>(nx, ny, nz, band, px, py, pz, labels, ncomp, comp_band);
}
