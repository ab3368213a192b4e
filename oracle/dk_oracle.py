"""CPU ORACLE — test infrastructure only.

A numpy/scipy restatement of the reference `defkrylov` solver path, used as the checker by
tests/, by __graft_entry__.smoke() and as bench.py's CPU baseline ("port").  Nothing in the
product package imports this module.  Each function cites the reference code it restates
(paths relative to /root/reference/pkg/src/defkrylov/).

Pinned against the reference itself: tests/golden/make_golden.py runs the reference in the
build container and stores its outputs under tests/golden/; tests/test_oracle.py checks
this module against them (history, iterations, solutions, labels).

The deflation context is label-based (an indicator Z stored as one column id per cell):
    restriction  Z^T v      = bincount(labels, v)
    prolongation A_p Z y    = A_p @ y[labels]
    E = Z^T A_p Z           = sum of A_p's nonzeros grouped by (label_row, label_col)
which equals the reference's dense-Z context (deflation.py:71-89) up to rounding.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg
import scipy.sparse
from scipy import ndimage

REORTH_TOL = 1e-8       # krylov.py:18
BREAKDOWN_TOL = 1e-13   # krylov.py:19
PIVOT_FLOOR = 1e-300    # sparse.py:23


class OracleSingular(Exception):
    pass


# ---------------------------------------------------------------------------------------
# operator
# ---------------------------------------------------------------------------------------
def csr_from_dia(n, offsets, diags) -> scipy.sparse.csr_matrix:
    """CSR with exactly the reference's stored entries: nonzero off-diagonals + diagonal."""
    rows, cols, vals = [], [], []
    i = np.arange(n)
    for k, o in enumerate(offsets):
        ok = (i + o >= 0) & (i + o < n) & ((diags[k] != 0.0) | (o == 0))
        rows.append(i[ok])
        cols.append(i[ok] + o)
        vals.append(diags[k][ok])
    A = scipy.sparse.csr_matrix((np.concatenate(vals), (np.concatenate(rows),
                                                        np.concatenate(cols))), shape=(n, n))
    A.sort_indices()
    return A


def csr_from_dia_lean(n, offsets, diags) -> scipy.sparse.csr_matrix:
    """csr_from_dia without the O(nnz) int64 coordinate lists (BASELINE configs 4 and 5).

    Same stored entries in the same (sorted) column order: each row keeps its nonzero
    off-diagonals and its diagonal (testbed.py:160-211 stores exactly the couplings t > 0
    plus the diagonal).  Peak memory is the CSR itself plus one n-vector per pass.
    """
    order = np.argsort(np.asarray(offsets))
    offsets = np.asarray(offsets)[order]
    i = np.arange(n)
    keep = []
    for k, o in zip(order, offsets):
        ok = (i + o >= 0) & (i + o < n) & ((diags[k] != 0.0) | (o == 0))
        keep.append(ok)
    counts = np.zeros(n, dtype=np.int64)
    for ok in keep:
        counts += ok
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    nnz = int(indptr[-1])
    idx_t = np.int32 if nnz < 2**31 and n < 2**31 else np.int64
    indices = np.empty(nnz, dtype=idx_t)
    data = np.empty(nnz, dtype=np.float64)
    pos = indptr[:-1].copy()
    for (k, o), ok in zip(zip(order, offsets), keep):
        rows = np.flatnonzero(ok)
        p = pos[rows]
        indices[p] = (rows + o).astype(idx_t)
        data[p] = diags[k][rows]
        pos[rows] += 1
    A = scipy.sparse.csr_matrix((data, indices, indptr.astype(idx_t)), shape=(n, n))
    A.has_sorted_indices = True
    return A


def sketch(x, rows: int = 16, seed: int = 20251020, chunk: int = 1 << 22):
    """Johnson-Lindenstrauss sketch S x with S a seeded n-column Rademacher matrix (±1).

    For any vector e, mean((S e)_i^2) is an unbiased estimate of |e|_2^2 (rows = 16: the
    estimate is within a factor 2 with probability > 0.99), so |S(x - x_ref)| / sqrt(rows)
    estimates the full-vector 2-norm difference from 16 stored numbers when x_ref is too
    large to commit (BASELINE configs 4 and 5).  Chunked, so any n fits.
    """
    x = np.asarray(x, dtype=np.float64)
    out = np.zeros(rows)
    rng = np.random.default_rng(seed)
    for lo in range(0, len(x), chunk):
        xs = x[lo:lo + chunk]
        s = rng.integers(0, 2, size=(rows, len(xs)), dtype=np.int8).astype(np.float64)
        out += (2.0 * s - 1.0) @ xs
    return out


# ---------------------------------------------------------------------------------------
# deflation context (deflation.py:40-89, label form)
# ---------------------------------------------------------------------------------------
class LabelDeflation:
    def __init__(self, A, labels, d, b, inv_diag=None, ap="A"):
        self.A = A
        self.lab = np.asarray(labels, dtype=np.int64)
        self.d = int(d)
        self.keep = self.lab >= 0
        self.ap = ap
        self.inv = inv_diag
        # A_p = A or A M^-1 (deflation.py:50-51): column scaling by inv_diag
        Ap = A if ap == "A" else (A @ scipy.sparse.diags(inv_diag)).tocsr()
        self.Ap = Ap
        # E = Z^T (A_p Z) (deflation.py:84-85) with the row-wise product first, as the
        # reference's A_p @ Z forms it: q_i = (A_p Z)[i, lab(i)] sums row i's coefficients
        # into its own label in CSR (ascending column) order; E[L][L] = sum of q_i over the
        # cells of L in ascending order; E[L][L2] (L2 != L) = sum of the coupling
        # coefficients in (row, column) order.  Every sum is sequential (np.bincount adds in
        # input order), so the order is fully defined: the in-label couplings nearly cancel
        # on the diagonal and at a high coefficient contrast (BASELINE config 4) the order
        # fixes the last bits that the ill-conditioned coarse solve amplifies.  Row blocks
        # bound the memory; off-diagonal entries are collected in order and summed once.
        n = Ap.shape[0]
        q = np.zeros(n)
        okeys, ovals = [], []
        step = 1 << 22
        for r0 in range(0, n, step):
            blk = Ap[r0:min(n, r0 + step)].tocoo()  # row-major, columns ascending per row
            lr, lc = self.lab[blk.row + r0], self.lab[blk.col]
            own = (lr >= 0) & (lc == lr)
            q[r0:r0 + blk.shape[0]] = np.bincount(blk.row[own], weights=blk.data[own],
                                                  minlength=blk.shape[0])
            cross = (lr >= 0) & (lc >= 0) & (lc != lr)
            okeys.append(lr[cross].astype(np.int64) * self.d + lc[cross])
            ovals.append(blk.data[cross])
        E = np.bincount(np.concatenate(okeys), weights=np.concatenate(ovals),
                        minlength=self.d * self.d).reshape(self.d, self.d)
        diag = np.bincount(self.lab[self.keep], weights=q[self.keep], minlength=self.d)
        E[np.arange(self.d), np.arange(self.d)] = diag
        self.E = E
        # dense_lu (sparse.py:121-137)
        lu, piv = scipy.linalg.lu_factor(E, check_finite=True)
        if np.min(np.abs(np.diag(lu))) < PIVOT_FLOOR:
            raise OracleSingular("zero pivot in LU factorization")
        self.lu = (lu, piv)
        self.x_star = self.prolong_z(self.coarse(self.restrict(b)))

    def restrict(self, v):
        return np.bincount(self.lab[self.keep], weights=v[self.keep], minlength=self.d)

    def coarse(self, s):
        return scipy.linalg.lu_solve(self.lu, s, check_finite=False)

    def prolong_z(self, y):
        out = np.zeros(len(self.lab))
        out[self.keep] = y[self.lab[self.keep]]
        return out

    def apply_p1(self, v):
        """v - A_p Z E^-1 Z^T v (deflation.py:61-62)."""
        return v - self.Ap @ self.prolong_z(self.coarse(self.restrict(v)))

    def apply_p2(self, v):
        """v - Z E^-1 Z^T A_p v (deflation.py:64-65)."""
        return v - self.prolong_z(self.coarse(self.restrict(self.Ap @ v)))

    def reconstruct(self, xh):
        """x* + P2 xh (deflation.py:67-68)."""
        return self.x_star + self.apply_p2(xh)


class DenseDeflation(LabelDeflation):
    """The reference's dense-Z arithmetic (dense Zᵀ / AZ products), for small n."""

    def __init__(self, A, Z, b, inv_diag=None, ap="A"):
        self.A = A
        self.Z = np.asarray(Z, dtype=np.float64)
        self.inv = inv_diag
        self.ap = ap
        W = self.Z if ap == "A" else self.Z * inv_diag[:, None]
        self.AZ = np.column_stack([A @ W[:, j] for j in range(W.shape[1])])
        self.ZT = self.Z.T.copy()
        E = self.Z.T @ self.AZ
        self.E = E
        lu, piv = scipy.linalg.lu_factor(E, check_finite=True)
        if np.min(np.abs(np.diag(lu))) < PIVOT_FLOOR:
            raise OracleSingular("zero pivot in LU factorization")
        self.lu = (lu, piv)
        self.x_star = self.Z @ self.coarse(self.ZT @ b)

    def apply_p1(self, v):
        return v - self.AZ @ self.coarse(self.ZT @ v)

    def apply_p2(self, v):
        Apv = self.A @ v if self.ap == "A" else self.A @ (v * self.inv)
        return v - self.Z @ self.coarse(self.ZT @ Apv)


# ---------------------------------------------------------------------------------------
# restarted GMRES(m) (krylov.py:90-236)
# ---------------------------------------------------------------------------------------
def _rotate(col, cs, sn, g, j):
    """Apply rotations 0..j-1 to the new column, create rotation j (krylov.py:90-104)."""
    for i in range(j):
        a, b = col[i], col[i + 1]
        col[i] = cs[i] * a + sn[i] * b
        col[i + 1] = -sn[i] * a + cs[i] * b
    r = float(np.hypot(col[j], col[j + 1]))
    if r == 0.0:
        cs[j], sn[j] = 1.0, 0.0
    else:
        cs[j], sn[j] = col[j] / r, col[j + 1] / r
    col[j], col[j + 1] = r, 0.0
    g[j + 1] = -sn[j] * g[j]
    g[j] = cs[j] * g[j]


def run_cycles(A, b, x0=None, inv_diag=None, m=30, tol=1e-6, max_iters=300, min_iters=0,
               defl=None, max_cycles=None, gs="mgs"):
    """Restarted right-preconditioned GMRES(m) on P1 A M^-1 (krylov.py:107-236).

    gs="mgs" is the reference's modified Gram-Schmidt (krylov.py:163-166); gs="cgs" is the
    classical variant (all h_i = V_i . w from the same w, then one update) that the device
    path computes — used to separate the MGS-vs-CGS rounding spread from device error on
    ill-conditioned cases (config 4).  Returns a dict with the SolveReport fields the device
    path reports.
    """
    n = A.shape[0]
    pre = (lambda v: v) if inv_diag is None else (lambda v: v * inv_diag)
    x0 = np.zeros(n) if x0 is None else np.asarray(x0, dtype=np.float64)
    x = x0.copy()
    hist, rof = [], []
    its = cycle = 0
    converged = False
    warning = None
    denom = None
    prev_beta = None
    reorths = 0
    while its < max_iters and not converged:
        if max_cycles is not None and cycle >= max_cycles:
            break
        r = b - A @ x
        if defl is not None:
            r = defl.apply_p1(r)
        beta = float(np.linalg.norm(r))
        if denom is None:
            denom = beta if beta > 0 else 1.0
            hist.append(beta)
            rof.append(0)
        if beta == 0.0 or (beta <= tol * denom and its >= min_iters):
            converged = True
            break
        if prev_beta is not None and warning == "breakdown" and beta >= prev_beta * (1 - 1e-14):
            break
        prev_beta = beta
        V = np.zeros((m + 1, n))
        V[0] = r / beta
        H = np.zeros((m + 1, m))
        R = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        cols = 0
        for j in range(m):
            if its >= max_iters:
                break
            w = A @ pre(V[j])
            if defl is not None:
                w = defl.apply_p1(w)
            w0 = float(np.linalg.norm(w))
            if gs == "cgs":                 # classical Gram-Schmidt
                h = V[:j + 1] @ w
                H[:j + 1, j] = h
                w -= V[:j + 1].T @ h
            else:
                for i in range(j + 1):      # modified Gram-Schmidt
                    h = float(V[i] @ w)
                    H[i, j] = h
                    w -= h * V[i]
            c = V[:j + 1] @ w               # selective re-orthogonalisation
            if np.max(np.abs(c), initial=0.0) > REORTH_TOL * max(w0, 1e-300):
                w -= V[:j + 1].T @ c
                H[:j + 1, j] += c
                reorths += 1
            hn = float(np.linalg.norm(w))
            H[j + 1, j] = hn
            col = np.zeros(m + 1)
            col[:j + 2] = H[:j + 2, j]
            _rotate(col, cs, sn, g, j)
            R[:, j] = col
            cols = j + 1
            res = abs(g[j + 1])
            its += 1
            hist.append(res)
            rof.append(cycle)
            stop = False
            if res <= tol * denom and its >= min_iters:
                converged = stop = True
            elif hn <= BREAKDOWN_TOL * max(1.0, float(np.linalg.norm(H[:j + 2, j]))):
                warning = "breakdown"
                stop = True
            if stop:
                break
            V[j + 1] = w / hn
        if cols == 0:
            break
        while cols > 1 and abs(R[cols - 1, cols - 1]) < 1e-14 * abs(R[0, 0]):
            cols -= 1
        y = scipy.linalg.solve_triangular(R[:cols, :cols], g[:cols], check_finite=False)
        x = x + pre(V[:cols].T @ y)
        cycle += 1
    x_hat = x
    if defl is not None:
        x = defl.reconstruct(x)
    nr = float(np.linalg.norm(b - A @ x))
    n0 = float(np.linalg.norm(b - A @ x0))
    return {
        "x": x, "x_hat": x_hat, "converged": converged, "iterations": its, "restarts": max(cycle - 1, 0),
        "cycles": cycle, "history": np.array(hist), "restart_of": np.array(rof),
        "final_relres": nr / (n0 if n0 > 0 else 1.0), "warning": warning, "reorths": reorths,
    }


# ---------------------------------------------------------------------------------------
# deflation-vector construction (physics.py:44-180)
# ---------------------------------------------------------------------------------------
def box_blocks(nc, p):
    """Block index per cell index: sizes nc//p, remainder to the leading blocks."""
    sizes = np.full(p, nc // p)
    sizes[:nc % p] += 1
    return np.repeat(np.arange(p), sizes)


def band_ids(k, thr):
    """log10 gap clustering, zero band -1 (physics.py:81-93)."""
    k = np.asarray(k, dtype=np.float64)
    band = np.full(len(k), -1, dtype=np.int64)
    pos = k > 0
    if pos.any():
        lg = np.log10(k[pos])
        u = np.unique(lg)
        edges = u[:-1][np.diff(u) >= thr]
        band[pos] = np.searchsorted(edges, lg, side="left")
    return band


def subdomain_levelset_labels(kx, nx, ny, nz, px, py, pz, thr):
    """Labels by first occurrence of 6-connected (box, band) components (physics.py:119-143).

    Returns (labels int64, d, excluded ids).  Slow (one ndimage.label per (box, band)):
    oracle sizes only.
    """
    band = band_ids(kx, thr).reshape(nz, ny, nx)
    bz, by, bx = box_blocks(nz, pz), box_blocks(ny, py), box_blocks(nx, px)
    box = (bx[None, None, :] + px * (by[None, :, None] + py * bz[:, None, None]))
    raw = np.full((nz, ny, nx), -1, dtype=np.int64)
    zero = set()
    nxt = 0
    st = ndimage.generate_binary_structure(3, 1)
    for bid in range(px * py * pz):
        inb = box == bid
        for bnd in np.unique(band[inb]):
            comp, nc = ndimage.label(inb & (band == bnd), structure=st)
            for c in range(1, nc + 1):
                raw[comp == c] = nxt
                if bnd == -1:
                    zero.add(nxt)
                nxt += 1
    raw = raw.ravel()
    _, first = np.unique(raw, return_index=True)
    order = np.argsort(first)               # raw ids sorted by first occurrence
    rank = np.empty(len(order), dtype=np.int64)
    rank[order] = np.arange(len(order))
    ids = np.unique(raw)
    labels = rank[np.searchsorted(ids, raw)]
    excl = {int(rank[np.searchsorted(ids, z)]) for z in zero}
    return labels, len(ids), excl


def subdomain_levelset_labels_boxwise(kx, nx, ny, nz, px, py, pz, thr):
    """The same labels as subdomain_levelset_labels, one ndimage.label per box sub-volume.

    physics.py:119-143 labels `in_box & band == b` on the full grid; every component of that
    mask lies inside the box, so labelling the box's sub-volume finds the same components.
    A box is a product of index ranges, so its C-order ravel visits cells in increasing
    linear index: a component's first cell in the sub-volume is its minimum linear index,
    which is what _relabel_by_first_occurrence (physics.py:44-54) orders by.  Returns
    (labels int64, d, excluded ids).  O(n): seconds at BASELINE configs 4 and 5, where the
    full-grid form takes an hour.
    """
    band = band_ids(kx, thr).reshape(nz, ny, nx)
    st = ndimage.generate_binary_structure(3, 1)

    def bounds(nc, p):
        sizes = np.full(p, nc // p)
        sizes[:nc % p] += 1
        return np.concatenate([[0], np.cumsum(sizes)])

    bx, by, bz = bounds(nx, px), bounds(ny, py), bounds(nz, pz)
    comp = np.empty((nz, ny, nx), dtype=np.int64)     # global component id per cell
    first, zero = [], []                              # per component: min linear index, band
    lin_box = None
    nxt = 0
    for kz in range(pz):
        for ky in range(py):
            for kx_ in range(px):
                sl = np.s_[bz[kz]:bz[kz + 1], by[ky]:by[ky + 1], bx[kx_]:bx[kx_ + 1]]
                sub = band[sl]
                lin_box = (np.arange(bx[kx_], bx[kx_ + 1])[None, None, :]
                           + nx * (np.arange(by[ky], by[ky + 1])[None, :, None]
                                   + ny * np.arange(bz[kz], bz[kz + 1])[:, None, None]))
                out = np.empty(sub.shape, dtype=np.int64)
                for bnd in np.unique(sub):
                    lab, nc = ndimage.label(sub == bnd, structure=st)
                    if nc == 0:
                        continue
                    flat = lab.ravel()
                    sel = flat > 0
                    ids, idx = np.unique(flat[sel], return_index=True)
                    first.append(lin_box.ravel()[np.flatnonzero(sel)[idx]])
                    zero.append(np.full(nc, bnd == -1))
                    out[lab > 0] = lab[lab > 0] - 1 + nxt
                    nxt += nc
                comp[sl] = out
    first = np.concatenate(first)
    zero = np.concatenate(zero)
    rank = np.empty(nxt, dtype=np.int64)
    rank[np.argsort(first, kind="stable")] = np.arange(nxt)
    labels = rank[comp.ravel()]
    excl = {int(r) for r in rank[zero]}
    return labels, nxt, excl


def columns_from_labels(labels, d, exclude):
    """partition_to_basis column map (physics.py:167-180): kept labels in order, -1 else."""
    keep = np.ones(d, dtype=bool)
    for e in exclude:
        keep[e] = False
    col = np.full(d, -1, dtype=np.int64)
    col[keep] = np.arange(int(keep.sum()))
    return col[labels], int(keep.sum())


# ---------------------------------------------------------------------------------------
# the reference's own solver on a label-based context (bench.py's reference arm)
# ---------------------------------------------------------------------------------------
class ReferenceLabelContext:
    """Duck-typed deflation context for the REFERENCE's `_run_cycles`.

    `_run_cycles` (krylov.py:107-236) only calls ctx.apply_p1 and ctx.reconstruct; this
    context provides them in label form with the reference's own kernels — R.spmv
    (sparse.py:101-106), R.dense_lu / R.lu_solve (sparse.py:121-145) — where the shipped
    DeflationContext (deflation.py:40-68) would need a dense n x d Z (98 GB at BASELINE
    config 3).  Restriction Z^T v = bincount(labels, v); prolongation A Z y = spmv(A,
    y[labels]); E = Z^T A Z from A's nonzeros by label pair; x* = Z E^-1 Z^T b.
    """

    def __init__(self, R, A, col_labels, d, b):
        self.R = R
        self.A = A
        self.lab = np.asarray(col_labels, dtype=np.int64)
        self.keep = self.lab >= 0
        self.d = int(d)
        csr = scipy.sparse.csr_matrix((A.values, A.col_indices, A.row_offsets),
                                      shape=(A.n, A.n))
        E = np.zeros(self.d * self.d)
        step = 1 << 22
        for r0 in range(0, A.n, step):
            blk = csr[r0:min(A.n, r0 + step)].tocoo()
            lr, lc = self.lab[blk.row + r0], self.lab[blk.col]
            ok = (lr >= 0) & (lc >= 0)
            E += np.bincount(lr[ok] * self.d + lc[ok], weights=blk.data[ok],
                             minlength=self.d * self.d)
        self.E_lu = R.dense_lu(E.reshape(self.d, self.d))
        self.x_star = self._prolong(R.lu_solve(self.E_lu, self._restrict(b)))

    def _restrict(self, v):
        return np.bincount(self.lab[self.keep], weights=v[self.keep], minlength=self.d)

    def _prolong(self, y):
        out = np.zeros(len(self.lab))
        out[self.keep] = y[self.lab[self.keep]]
        return out

    def apply_p1(self, v):
        R = self.R
        return v - R.spmv(self.A, self._prolong(R.lu_solve(self.E_lu, self._restrict(v))))

    def apply_p2(self, v):
        R = self.R
        return v - self._prolong(R.lu_solve(self.E_lu, self._restrict(R.spmv(self.A, v))))

    def reconstruct(self, xh):
        return self.x_star + self.apply_p2(xh)
