"""Coarse-matrix fill under a nested-dissection ordering of the labels (design probe).

Builds the label adjacency of a config's partition (E's pattern), orders it by geometric
nested dissection, and counts the 32 x 32 tiles of the row profile of L (= of W = L^-1) in
the natural and the ND order.  Usage: python tools/nd_probe.py [config]
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import paper_1510_02148_b200 as dk
from paper_1510_02148_b200 import configs

T = 32


def adjacency(grid, lab, d):
    L = lab.reshape(grid.nz, grid.ny, grid.nx)
    pairs = []
    for ax in range(3):
        a = np.moveaxis(L, ax, 0)
        u, v = a[:-1].ravel(), a[1:].ravel()
        k = (u != v) & (u >= 0) & (v >= 0)
        pairs.append(np.stack([u[k], v[k]]))
    p = np.concatenate(pairs, axis=1)
    p = np.concatenate([p, p[::-1]], axis=1)
    key = np.unique(p[0].astype(np.int64) * d + p[1])
    r, c = key // d, key % d
    ptr = np.searchsorted(r, np.arange(d + 1))
    return ptr, c


def centroids(grid, lab, d):
    iz, iy, ix = np.meshgrid(np.arange(grid.nz), np.arange(grid.ny), np.arange(grid.nx),
                             indexing="ij")
    k = lab >= 0
    cnt = np.bincount(lab[k], minlength=d)
    xyz = np.stack([np.bincount(lab[k], weights=a.ravel()[k], minlength=d) / cnt
                    for a in (ix * grid.dx, iy * grid.dy, iz * grid.dz)], axis=1)
    return xyz


def nested_dissection(ptr, col, xyz, leaf=64):
    d = len(ptr) - 1
    order = []
    side = np.zeros(d, np.int8)

    def rec(nodes):
        if len(nodes) <= leaf:
            order.extend(sorted(nodes.tolist()))
            return
        P = xyz[nodes]
        ax = int(np.argmax(P.max(0) - P.min(0)))
        med = np.median(P[:, ax])
        left = P[:, ax] <= med
        if left.all() or not left.any():
            left = np.arange(len(nodes)) < len(nodes) // 2
        A, B = nodes[left], nodes[~left]
        side[A] = 1
        side[B] = 2
        # separator: the vertices of the smaller side adjacent to the other side
        small, other = (A, 2) if len(A) <= len(B) else (B, 1)
        sep = np.array([v for v in small.tolist()
                        if (side[col[ptr[v]:ptr[v + 1]]] == other).any()], dtype=np.int64)
        side[nodes] = 0
        insep = np.zeros(d, bool)
        insep[sep] = True
        rec(A[~insep[A]])
        rec(B[~insep[B]])
        order.extend(sep.tolist())

    rec(np.arange(d))
    return np.array(order)


def profile_tiles(ptr, col, perm):
    """Row profile of the Cholesky factor of E permuted by perm (new = position in perm)."""
    d = len(perm)
    inv = np.empty(d, np.int64)
    inv[perm] = np.arange(d)
    first = np.arange(d)
    for v in range(d):
        nb = col[ptr[v]:ptr[v + 1]]
        if len(nb):
            i = inv[v]
            j = inv[nb].min()
            first[i] = min(first[i], j)
    # the envelope of L is E's; W = L^-1 closes it: g(i) = min(f(i), min_{f(i)<=k<i} g(k))
    g = first.copy()
    for i in range(d):
        if first[i] < i:
            g[i] = min(first[i], g[first[i]:i].min())
    nb = (d + T - 1) // T
    out = []
    for prof in (first, g):
        fb = np.array([prof[I * T:(I + 1) * T].min() // T for I in range(nb)])
        out.append(int(sum(I - fb[I] + 1 for I in range(nb))))
    return out, nb


def main():
    idx = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    c = configs.make_case(idx)
    px, py, pz = c.boxes
    part = dk.subdomain_levelset_partition(c.band_field, px, py, pz, c.jump_threshold,
                                           backend="host")
    lab = np.asarray(part.labels)
    d = part.d
    ptr, col = adjacency(c.grid, lab, d)
    print(f"config {idx}: d={d} nnz(E offdiag)={len(col)} avg deg {len(col)/d:.1f}")
    xyz = centroids(c.grid, lab, d)
    full = (d // T + 1) * (d // T + 2) // 2
    nat, nb = profile_tiles(ptr, col, np.arange(d))
    print(f"packed triangle tiles {full}; natural profile tiles L {nat[0]} W {nat[1]}")
    for leaf in (32, 64, 128, 256):
        t = time.time()
        perm = nested_dissection(ptr, col, xyz, leaf)
        assert len(np.unique(perm)) == d
        (ndl, ndw), _ = profile_tiles(ptr, col, perm)
        print(f"ND leaf {leaf}: profile tiles L {ndl} W {ndw} ({ndw/full:.3f} of packed; "
              f"W s + W^T t reads {2*ndw/full:.3f}x)  [{time.time()-t:.1f}s]")




def graph_nd(ptr, col, leaf=64):
    """Level-structure nested dissection (graph only, no geometry)."""
    from collections import deque
    d = len(ptr) - 1
    order = []
    active = np.zeros(d, bool)
    level = np.full(d, -1, np.int64)

    def bfs(src, nodes):
        for v in nodes:
            level[v] = -1
        level[src] = 0
        q = deque([src])
        seen = [src]
        while q:
            u = q.popleft()
            for w in col[ptr[u]:ptr[u + 1]]:
                if active[w] and level[w] < 0:
                    level[w] = level[u] + 1
                    q.append(w)
                    seen.append(w)
        return seen

    def rec(nodes):
        if len(nodes) <= leaf:
            order.extend(sorted(nodes))
            return
        for v in nodes:
            active[v] = True
        # components
        comps = []
        for v in nodes:
            level[v] = -1
        rem = set(nodes)
        while rem:
            s = min(rem)
            c = bfs(s, [])
            comps.append(c)
            rem -= set(c)
        if len(comps) > 1:
            for v in nodes:
                active[v] = False
            for c in comps:
                rec(c)
            return
        comp = comps[0]
        # pseudo-peripheral node
        src = min(comp, key=lambda v: ptr[v + 1] - ptr[v])
        ecc = -1
        while True:
            seen = bfs(src, comp)
            e = level[seen[-1]]
            if e <= ecc:
                break
            ecc = e
            last = [v for v in seen if level[v] == e]
            src = min(last, key=lambda v: ptr[v + 1] - ptr[v])
        seen = bfs(src, comp)
        lv = np.array([level[v] for v in seen])
        nl = lv.max() + 1
        cnt = np.bincount(lv, minlength=nl)
        cum = np.cumsum(cnt)
        n = len(seen)
        cands = [l for l in range(1, nl - 1) if 0.25 * n <= cum[l - 1] and cum[l] <= 0.75 * n]
        if not cands:
            cands = [int(np.searchsorted(cum, n / 2))]
        L = min(cands, key=lambda l: cnt[l])
        sep = [v for v in seen if level[v] == L
               and any(active[w] and level[w] == L + 1 for w in col[ptr[v]:ptr[v + 1]])]
        sset = set(sep)
        A = [v for v in seen if level[v] <= L and v not in sset]
        B = [v for v in seen if level[v] > L]
        for v in nodes:
            active[v] = False
        if not A or not B:
            order.extend(sorted(nodes))
            return
        rec(A)
        rec(B)
        order.extend(sep)

    rec(list(range(d)))
    return np.array(order)


def main2():
    idx = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    c = configs.make_case(idx)
    px, py, pz = c.boxes
    part = dk.subdomain_levelset_partition(c.band_field, px, py, pz, c.jump_threshold,
                                           backend="host")
    lab = np.asarray(part.labels)
    d = part.d
    ptr, col = adjacency(c.grid, lab, d)
    full = (d // T + 1) * (d // T + 2) // 2
    for leaf in (32, 64, 128):
        t = time.time()
        perm = graph_nd(ptr, col, leaf)
        assert len(np.unique(perm)) == d, (len(perm), d)
        (ndl, ndw), _ = profile_tiles(ptr, col, perm)
        print(f"graph ND leaf {leaf}: L {ndl} W {ndw} ({ndw/full:.3f}) [{time.time()-t:.1f}s]")


if __name__ == "__main__":
    main()
    main2()


def flops(ptr, col, perm):
    d = len(perm)
    inv = np.empty(d, np.int64)
    inv[perm] = np.arange(d)
    f = np.arange(d)
    for v in range(d):
        nb = col[ptr[v]:ptr[v + 1]]
        if len(nb):
            f[inv[v]] = min(f[inv[v]], inv[nb].min())
    g = f.copy()
    for i in range(d):
        if f[i] < i:
            g[i] = min(f[i], g[f[i]:i].min())
    out = []
    for prof in (f, g):
        # column counts: rows i >= j with prof(i) <= j
        cnt = np.zeros(d + 1, np.int64)
        np.add.at(cnt, prof, 1)
        np.add.at(cnt, np.arange(1, d + 1), -1)
        cc = np.cumsum(cnt)[:d]
        out.append(float((cc.astype(float) ** 2).sum()))
    return out


if __name__ == "__main__" and len(sys.argv) > 2:
    c = configs.make_case(int(sys.argv[1]))
    px, py, pz = c.boxes
    part = dk.subdomain_levelset_partition(c.band_field, px, py, pz, c.jump_threshold,
                                           backend="host")
    lab = np.asarray(part.labels)
    ptr, col = adjacency(c.grid, lab, part.d)
    perm = graph_nd(ptr, col, 64)
    fl, fw = flops(ptr, col, perm)
    d = part.d
    print(f"d={d} chol flops (envelope) {fl/1e9:.1f} GF, W flops ~{fw/1e9:.1f} GF; dense d^3/3 "
          f"{d**3/3/1e9:.0f} GF")
