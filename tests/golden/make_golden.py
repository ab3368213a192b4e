"""Generate the golden fixtures by running the REFERENCE implementation (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--big]

Writes tests/golden/*.npz.  Inputs are built with this repo's seeded generators (so the GPU
box can rebuild them without the reference); every output is produced by the reference's
own public API (defkrylov.pdgmres / gmres / assemble_pressure / subdomain_levelset_partition).
`--big` also runs config 2 (dense-Z reference, ~30 s, ~6 GB) and the config-3 partition;
`--labels 4 5` runs the reference partition of configs 4 and 5 (config5: about an hour).
"""
from __future__ import annotations

import sys
import time
import zlib
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import defkrylov as R  # noqa: E402  (the reference)

from paper_1510_02148_b200 import configs, testbed  # noqa: E402


def ref_matrix(A):
    """The reference SparseMatrix for one of our DIA-built operators (same CSR arrays)."""
    return R.SparseMatrix(A.n, A.row_offsets, A.col_indices, A.values)


def crc(a) -> int:
    return zlib.crc32(np.ascontiguousarray(a).tobytes())


def sandwich(sigma=1e6):
    g = R.Grid(7, 7, 3)
    f = R.make_layered_field(g, [((0, 1), sigma), ((1, 2), 1.0), ((2, 3), sigma)])
    q = np.zeros(g.n_cells)
    q[0], q[-1] = 1.0, -1.0
    p = R.diagonal_scale(R.assemble_pressure(f, R.BoundarySpec(), q))
    return g, f, q, p


def make_sandwich():
    out = {}
    g, f, q, p = sandwich()
    M = R.Preconditioner.jacobi(p.A)
    part = R.levelset_partition(f, 2.0)
    Z = R.partition_to_basis(part)
    rep = R.pdgmres(p.A, p.b, M=M, m=40, basis=Z, tol=1e-6, max_iters=300)
    plain = R.gmres(p.A, p.b, M=M, m=40, tol=1e-6, max_iters=300)
    # the reference's own golden CSV (frontend fixture) must agree with this run
    csv = Path("/root/reference/pkg/frontend/test/fixtures/convergence.pdgmres.csv")
    if csv.exists():
        rows = np.loadtxt(csv, delimiter=",", skiprows=1)
        assert np.array_equal(rows[:, 1], rep.residual_history), "frontend fixture mismatch"
        out["fixture_history"] = rows[:, 1]
    out.update(
        ro=p.A.row_offsets, ci=p.A.col_indices, va=p.A.values, b=p.b, q=q,
        labels=part.labels, d=part.d,
        pd_history=rep.residual_history, pd_x=rep.x, pd_iters=rep.iterations,
        pd_relres=rep.final_relres, pd_restart_of=rep.restart_of,
        gm_history=plain.residual_history, gm_x=plain.x, gm_iters=plain.iterations,
        gm_relres=plain.final_relres)
    np.savez_compressed(HERE / "sandwich.npz", **out)
    print("sandwich: pdgmres", rep.iterations, "gmres", plain.iterations)


def make_random_hetero():
    """Small heterogeneous field with zero-permeability cells, top Dirichlet and sources."""
    rng = np.random.default_rng(11)
    g = R.Grid(12, 10, 8, 2.0, 3.0, 0.5)
    n = g.n_cells
    kx = 10 ** rng.uniform(-4, 2, n)
    kx[rng.random(n) < 0.05] = 0.0
    ky = kx * 10 ** rng.uniform(-0.5, 0.5, n)
    kz = 0.1 * kx
    f = R.PermeabilityField(g, kx, ky, kz)
    q = np.zeros(n)
    q[5], q[n - 7] = 2.0, -2.0
    p = R.assemble_pressure(f, R.BoundarySpec(True, 1.5, 0.8), q)
    M = R.Preconditioner.jacobi(p.A)
    part = R.subdomain_levelset_partition(f, 3, 2, 2, 1.0)
    Z = R.partition_to_basis(part)
    rep = R.pdgmres(p.A, p.b, M=M, m=20, basis=Z, tol=1e-10, max_iters=2000)
    rep_am = R.pdgmres(p.A, p.b, M=M, m=20, basis=Z, tol=1e-10, max_iters=2000, A_p_choice="AM")
    plain = R.gmres(p.A, p.b, M=M, m=20, tol=1e-10, max_iters=2000)
    ctx = R.build_context(p.A, M, Z, p.b)
    v = rng.standard_normal(n)
    np.savez_compressed(
        HERE / "hetero.npz", kx=kx, ky=ky, kz=kz, q=q,
        ro=p.A.row_offsets, ci=p.A.col_indices, va=p.A.values, b=p.b,
        labels=part.labels, d=part.d, excl=np.array(sorted(part.default_exclude)),
        pd_history=rep.residual_history, pd_x=rep.x, pd_iters=rep.iterations,
        pd_relres=rep.final_relres,
        am_history=rep_am.residual_history, am_x=rep_am.x, am_iters=rep_am.iterations,
        gm_history=plain.residual_history, gm_x=plain.x, gm_iters=plain.iterations,
        v=v, p1v=ctx.apply_p1(v), p2v=ctx.apply_p2(v), rec=ctx.reconstruct(v),
        x_star=ctx.x_star, E=ctx.basis.Z.T @ ctx.AZ)
    print("hetero: pdgmres", rep.iterations, "AM", rep_am.iterations, "gmres", plain.iterations,
          "d", Z.d)


def make_config1():
    case = configs.config1()
    A, b = case.problem()
    Ar = ref_matrix(A)
    f = case.field
    fr = R.PermeabilityField(R.Grid(32, 32, 32), f.kx, f.ky, f.kz)
    part = R.subdomain_levelset_partition(fr, 2, 2, 2, 2.0)
    Z = R.partition_to_basis(part)
    M = R.Preconditioner.jacobi(Ar)
    t = time.time()
    rep = R.pdgmres(Ar, b, M=M, m=50, basis=Z, tol=1e-8, max_iters=20000)
    t_pd = time.time() - t
    t = time.time()
    plain = R.gmres(Ar, b, M=M, m=50, tol=1e-8, max_iters=20000)
    t_gm = time.time() - t
    np.savez_compressed(
        HERE / "config1.npz", labels=part.labels, d=part.d,
        pd_history=rep.residual_history, pd_x=rep.x, pd_iters=rep.iterations,
        pd_relres=rep.final_relres, gm_history=plain.residual_history, gm_x=plain.x,
        gm_iters=plain.iterations, gm_relres=plain.final_relres,
        a_crc=crc(A.values), b_crc=crc(b))
    print(f"config1: d={part.d} pdgmres {rep.iterations} it ({t_pd:.2f}s) "
          f"gmres {plain.iterations} it ({t_gm:.2f}s)")


def make_config2():
    case = configs.config2()
    A, b = case.problem()
    Ar = ref_matrix(A)
    f = case.field
    fr = R.PermeabilityField(R.Grid(128, 128, 64), f.kx, f.ky, f.kz)
    part = R.subdomain_levelset_partition(fr, 4, 4, 4, 1.0)
    Z = R.partition_to_basis(part)
    M = R.Preconditioner.jacobi(Ar)
    t = time.time()
    rep = R.pdgmres(Ar, b, M=M, m=50, basis=Z, tol=1e-8, max_iters=20000)
    t_pd = time.time() - t
    np.savez_compressed(
        HERE / "config2.npz", labels_crc=crc(part.labels.astype(np.int64)), d=part.d,
        pd_history=rep.residual_history, pd_x=rep.x, pd_x_sample=rep.x[::97],
        pd_x_norm=np.linalg.norm(rep.x),
        pd_iters=rep.iterations, pd_relres=rep.final_relres, seconds=t_pd)
    print(f"config2: d={part.d} pdgmres {rep.iterations} it ({t_pd:.1f}s)")


def make_config3_labels():
    case = configs.config3()
    fb = case.band_field
    fr = R.PermeabilityField(R.Grid(60, 220, 85, 20.0, 10.0, 2.0), fb.kx, fb.ky, fb.kz)
    t = time.time()
    part = R.subdomain_levelset_partition(fr, 6, 11, 5, 1.0)
    sec = time.time() - t
    np.savez_compressed(HERE / "config3_labels.npz", labels_crc=crc(part.labels.astype(np.int64)),
                        d=part.d, nexcl=len(part.default_exclude), seconds=sec,
                        sizes_head=np.bincount(part.labels)[:64])
    print(f"config3 labels: d={part.d} ({sec:.1f}s)")


def make_labels_big(idx):
    """Reference labels at BASELINE configs 4 and 5 (physics.py:119-143, run as shipped).

    The reference labels each (box, band) with ndimage.label on the full grid and renumbers
    in a Python loop over n cells: minutes at config 4, about an hour at config 5.  Stores
    the CRC of the int64 label vector, d, the excluded ids and every column's cell count.
    """
    case = configs.make_case(idx)
    fb = case.band_field
    g = case.grid
    fr = R.PermeabilityField(R.Grid(g.nx, g.ny, g.nz, g.dx, g.dy, g.dz), fb.kx, fb.ky, fb.kz)
    px, py, pz = case.boxes
    t = time.time()
    part = R.subdomain_levelset_partition(fr, px, py, pz, case.jump_threshold)
    sec = time.time() - t
    np.savez_compressed(HERE / f"config{idx}_labels.npz",
                        labels_crc=crc(part.labels.astype(np.int64)), d=part.d,
                        excl=np.array(sorted(part.default_exclude), dtype=np.int64),
                        nexcl=len(part.default_exclude), seconds=sec,
                        sizes=np.bincount(part.labels, minlength=part.d))
    print(f"config{idx} labels: d={part.d} excl={len(part.default_exclude)} ({sec:.1f}s)")


def make_harmonic():
    """RDGMRES, harmonic Ritz extraction and capture_ritz traces (harmonic.py, krylov.py)."""
    out = {}
    g, f, q, p = sandwich()
    M = R.Preconditioner.jacobi(p.A)
    for tag, kw in (("s3", dict(m=40, d=3, tol=1e-6)), ("s2", dict(m=40, d=2, tol=1e-8)),
                    ("s3j", dict(M=M, m=40, d=3, tol=1e-6))):
        rep = R.rdgmres(p.A, p.b, max_iters=300, **kw)
        out[f"{tag}_iters"] = rep.iterations
        out[f"{tag}_history"] = rep.residual_history
        out[f"{tag}_x"] = rep.x
        out[f"{tag}_flags"] = rep.deflated_flags
        out[f"{tag}_from"] = -1 if rep.deflated_from_cycle is None else rep.deflated_from_cycle
        out[f"{tag}_warning"] = rep.warning or ""
        out[f"{tag}_relres"] = rep.final_relres
    # hetero: Jacobi, A_p = A and AM, tight tolerance, several deflated cycles
    h = np.load(HERE / "hetero.npz")
    A = R.SparseMatrix(len(h["b"]), h["ro"], h["ci"], h["va"])
    Mh = R.Preconditioner.jacobi(A)
    for tag, ap in (("h", "A"), ("hAM", "AM")):
        rep = R.rdgmres(A, h["b"], M=Mh, m=20, d=4, tol=1e-10, max_iters=2000, A_p_choice=ap)
        out[f"{tag}_iters"] = rep.iterations
        out[f"{tag}_history"] = rep.residual_history
        out[f"{tag}_x"] = rep.x
        out[f"{tag}_flags"] = rep.deflated_flags
        out[f"{tag}_warning"] = rep.warning or ""
    # capture_ritz traces of plain GMRES(20) on hetero (three cycles)
    rep = R.gmres(A, h["b"], M=Mh, m=20, tol=1e-10, max_iters=60, capture_ritz=True)
    out["cr_iters"] = rep.iterations
    out["cr_cycles"] = np.array([len(t) for t in rep.ritz_trace])
    out["cr_trace"] = np.concatenate(rep.ritz_trace)
    out["cr_iter_trace"] = np.concatenate([np.asarray(t) for t in rep.ritz_iter_trace])
    # extraction on fixed cycle data (the reference's own Arnoldi output)
    data = rep.arnoldi
    out["ad_V"], out["ad_H"], out["ad_m"] = data.V, data.Hbar, data.m
    for d in (1, 4, 7):
        hb = R.harmonic_ritz_b(data, d)
        ha = R.harmonic_ritz_a(data, d)
        out[f"hb{d}_thetas"], out[f"hb{d}_Y"], out[f"hb{d}_Z"] = hb.thetas, hb.Y, hb.Zvecs
        out[f"ha{d}_thetas"], out[f"ha{d}_Y"] = ha.thetas, ha.Y
    # a dense (non-indicator) basis through pdgmres: 3 smooth random columns
    rng = np.random.default_rng(21)
    Zd = np.cumsum(rng.standard_normal((A.n, 3)), axis=0) / np.sqrt(A.n)
    basis = R.DeflationBasis(Zd)
    ctx = R.build_context(A, Mh, basis, h["b"])
    v = rng.standard_normal(A.n)
    rep = R.pdgmres(A, h["b"], M=Mh, m=20, basis=basis, tol=1e-10, max_iters=2000)
    out.update(dz_Z=Zd, dz_v=v, dz_p1v=ctx.apply_p1(v), dz_p2v=ctx.apply_p2(v),
               dz_xs=ctx.x_star, dz_E=Zd.T @ ctx.AZ, dz_iters=rep.iterations,
               dz_history=rep.residual_history, dz_x=rep.x)
    np.savez_compressed(HERE / "harmonic.npz", **out)
    print("harmonic:", {k: int(v) for k, v in out.items() if k.endswith("_iters")})


if __name__ == "__main__":
    if "--config2" in sys.argv:
        make_config2()
        sys.exit(0)
    if "--labels" in sys.argv:
        for i in sys.argv[sys.argv.index("--labels") + 1:]:
            make_labels_big(int(i))
        sys.exit(0)
    make_sandwich()
    make_random_hetero()
    make_config1()
    make_harmonic()
    if "--big" in sys.argv:
        make_config3_labels()
        make_config2()


# tests/golden/convergence.pdgmres.ref.csv is the reference CLI's own output for the sandwich
# case (`defkrylov compare`, GMRES(40), levelset d=3), copied from the reference frontend
# fixtures; make_sandwich() asserts that the reference run above reproduces its history.
