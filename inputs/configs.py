"""Seeded generators for BASELINE.json's five configs (SURVEY.md 8(d) recipes).

Every generator is deterministic: seed = 1000 + config number, numpy PCG64,
random draws taken in CSR (row, col) order of the stored entries they perturb.
The paper measures on SuiteSparse matrices (venkat50, the 100-matrix corpus,
af_shell); none is in the container and none is reproduced -- these synthetic
matrices stand in for them at the same scale.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .nd import grid_nd, expand_dof


@dataclass
class Problem:
    name: str
    n: int
    indptr: np.ndarray      # int64, original ordering
    indices: np.ndarray     # int32, sorted per row
    data: np.ndarray        # float64
    perm: np.ndarray        # int64, Ã = A(perm, perm)
    block_sizes: np.ndarray  # int32, initial partition of Ã
    tau: float
    block_part: np.ndarray  # int32 per block: top ND subtree id or -1 (separator)
    meta: dict

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])


def _csr_from_coo(n, rows, cols, vals):
    order = np.lexsort((cols, rows))
    rows = rows[order]
    cols = cols[order]
    vals = vals[order]
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(indptr, rows + 1, 1)
    indptr = np.cumsum(indptr)
    return indptr, cols.astype(np.int32), vals.astype(np.float64)


def _grid_offsets(kind):
    if kind == 7:
        return [(dx, dy, dz) for dx, dy, dz in
                [(-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)]]
    return [(dx, dy, dz) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)
            if (dx, dy, dz) != (0, 0, 0)]


def _stencil_pairs(nx, ny, nz, offsets):
    """All in-grid (i, j, offset-id) pairs for the given offsets."""
    X, Y, Z = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    X = X.ravel(); Y = Y.ravel(); Z = Z.ravel()
    I = X + nx * (Y + ny * Z)
    rows, cols, oid = [], [], []
    for k, (dx, dy, dz) in enumerate(offsets):
        x2, y2, z2 = X + dx, Y + dy, Z + dz
        ok = (x2 >= 0) & (x2 < nx) & (y2 >= 0) & (y2 < ny) & (z2 >= 0) & (z2 < nz)
        rows.append(I[ok])
        cols.append((x2 + nx * (y2 + ny * z2))[ok])
        oid.append(np.full(int(ok.sum()), k, dtype=np.int16))
    return np.concatenate(rows), np.concatenate(cols), np.concatenate(oid)


# --------------------------------------------------------------------------- c1
def config1(seed=1001, block=8):
    """2D 5-pt Laplacian 32x32, a_ii = 4, a_ij = -1 + U(-0.1, 0.1) iid per stored
    off-diagonal in CSR order; natural ordering; tau = 1e-2; uniform blocks of 8
    (the ILU(1,tau) estimator fallback of SURVEY.md 8(d))."""
    nx = ny = 32
    n = nx * ny
    rng = np.random.Generator(np.random.PCG64(seed))
    X, Y = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
    X = X.ravel(); Y = Y.ravel()
    I = X + nx * Y
    rows, cols = [I], [I]
    for dx, dy in [(-1, 0), (1, 0), (0, -1), (0, 1)]:
        x2, y2 = X + dx, Y + dy
        ok = (x2 >= 0) & (x2 < nx) & (y2 >= 0) & (y2 < ny)
        rows.append(I[ok]); cols.append((x2 + nx * y2)[ok])
    rows = np.concatenate(rows); cols = np.concatenate(cols)
    indptr, indices, _ = _csr_from_coo(n, rows, cols, np.zeros(len(rows)))
    rr = np.repeat(np.arange(n), np.diff(indptr))
    off = rr != indices
    data = np.where(off, 0.0, 4.0)
    data[off] = -1.0 + rng.uniform(-0.1, 0.1, size=int(off.sum()))
    sizes = np.full(n // block, block, dtype=np.int32)
    return Problem("c1", n, indptr, indices, data, np.arange(n, dtype=np.int64), sizes, 1e-2,
                   np.zeros(len(sizes), dtype=np.int32),
                   {"grid": (nx, ny), "ordering": "natural", "block": block, "seed": seed})


# --------------------------------------------------------------------------- c2
def config2(seed=1002, N=64, leaf=512, block=8, top_levels=0):
    """3D 7-pt convection-diffusion, N^3, h = 1/(N+1), beta = 10*(1, .5, .25):
    face off-diagonals -1, plus upwind -h*beta_d on the -e_d neighbour, each
    off-diagonal x (1 + 0.05 U(-1,1)) in CSR order; a_ii = sum |a_ij| over the full
    stencil (out-of-grid neighbours at their nominal value) -> irreducibly
    diagonally dominant M-matrix.  Geometric ND, tau = 1e-3."""
    n = N ** 3
    h = 1.0 / (N + 1)
    beta = 10.0 * np.array([1.0, 0.5, 0.25])
    offs = _grid_offsets(7)
    rows, cols, oid = _stencil_pairs(N, N, N, offs)
    nominal = np.array([-1.0 - h * beta[0], -1.0, -1.0 - h * beta[1], -1.0,
                        -1.0 - h * beta[2], -1.0])
    # CSR order of the off-diagonals
    order = np.lexsort((cols, rows))
    rows, cols, oid = rows[order], cols[order], oid[order]
    rng = np.random.Generator(np.random.PCG64(seed))
    vals = nominal[oid] * (1.0 + 0.05 * rng.uniform(-1.0, 1.0, size=len(rows)))
    diag = np.zeros(n)
    np.add.at(diag, rows, np.abs(vals))
    # out-of-grid neighbours (boundary rows): nominal magnitude
    cnt = np.zeros((n, 6))
    cnt[rows, oid] = 1.0
    diag += ((1.0 - cnt) * np.abs(nominal)[None, :]).sum(axis=1)
    allr = np.concatenate([rows, np.arange(n)])
    allc = np.concatenate([cols, np.arange(n)])
    allv = np.concatenate([vals, diag])
    indptr, indices, data = _csr_from_coo(n, allr, allc, allv)
    perm, sizes, parts = grid_nd(N, N, N, leaf=leaf, block=block, top_levels=top_levels)
    return Problem("c2", n, indptr, indices, data, perm, sizes, 1e-3, parts,
                   {"grid": (N, N, N), "ordering": "geometric ND", "leaf": leaf,
                    "block": block, "seed": seed})


# --------------------------------------------------------------------------- c3
def config3(seed=1003, N=48, dof=3, leaf=512, top_levels=1):
    """27-pt stencil on N^3 nodes with dof=3 unknowns/node: every node pair in the
    27-pt neighbourhood (incl. self) gets an iid N(0,1) 3x3 block ((p,q) and (q,p)
    independent), drawn in CSR order; then a_rr = 1.2 * sum_{c != r} |a_rc|.
    Nodal geometric ND, nodal 3x3 initial blocks, tau = 1e-3."""
    nn = N ** 3
    n = nn * dof
    offs = [(0, 0, 0)] + _grid_offsets(27)
    nr, nc, _ = _stencil_pairs(N, N, N, offs)
    rows = (nr[:, None, None] * dof + np.arange(dof)[None, :, None]).repeat(dof, axis=2).ravel()
    cols = (nc[:, None, None] * dof + np.arange(dof)[None, None, :]).repeat(dof, axis=1).ravel()
    indptr, indices, _ = _csr_from_coo(n, rows, cols, np.zeros(len(rows)))
    del rows, cols
    rng = np.random.Generator(np.random.PCG64(seed))
    data = rng.standard_normal(len(indices))
    rr = np.repeat(np.arange(n), np.diff(indptr))
    dmask = rr == indices
    offsum = np.bincount(rr, weights=np.abs(data) * (~dmask), minlength=n)
    data[dmask] = 1.2 * offsum[rr[dmask]]
    perm, sizes, parts = grid_nd(N, N, N, leaf=max(1, leaf // dof), block=1,
                                 top_levels=top_levels)
    perm, sizes, parts = expand_dof(perm, sizes, parts, dof)
    return Problem("c3", n, indptr, indices, data, perm, sizes, 1e-3, parts,
                   {"grid": (N, N, N), "dof": dof, "ordering": "nodal geometric ND",
                    "seed": seed})


# --------------------------------------------------------------------------- c4
def config4(seed=1004, nblocks=20000, bmin=16, bmax=64, per_row=12, dominance=1.5):
    """Random block-sparse unsymmetric matrix: nblocks dense diagonal blocks of size
    U{bmin..bmax}; per block row `per_row` distinct random column blocks != i; every
    stored block iid N(0,1) (drawn in CSR order); then a_rr = dominance *
    sum_{c != r} |a_rc| (diagonal block shifted to dominance).  Identity ordering,
    the generator's blocks as the initial partition, tau = 1e-4."""
    rng = np.random.Generator(np.random.PCG64(seed))
    bsz = rng.integers(bmin, bmax + 1, size=nblocks).astype(np.int64)
    bstart = np.concatenate([[0], np.cumsum(bsz)])
    n = int(bstart[-1])
    colblk = []
    for i in range(nblocks):
        c = rng.choice(nblocks - 1, size=min(per_row, nblocks - 1), replace=False)
        c = c + (c >= i)
        colblk.append(np.sort(np.concatenate([[i], c])))
    # row template of each block row, tiled over its rows
    rowlen = np.array([int(bsz[cb].sum()) for cb in colblk], dtype=np.int64)
    indptr = np.zeros(n + 1, dtype=np.int64)
    indptr[1:] = np.cumsum(np.repeat(rowlen, bsz))
    nnz = int(indptr[-1])
    indices = np.empty(nnz, dtype=np.int32)
    for i in range(nblocks):
        tmpl = np.concatenate([np.arange(bstart[c], bstart[c + 1], dtype=np.int32) for c in colblk[i]])
        a, b_ = indptr[bstart[i]], indptr[bstart[i + 1]]
        indices[a:b_] = np.tile(tmpl, int(bsz[i]))
    data = rng.standard_normal(nnz)
    rr = np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr))
    dmask = rr == indices
    offsum = np.bincount(rr, weights=np.abs(data) * (~dmask), minlength=n)
    data[dmask] = dominance * offsum[rr[dmask]]
    del rr, dmask
    return Problem("c4", n, indptr, indices, data, np.arange(n, dtype=np.int64), bsz.astype(np.int32), 1e-4,
                   np.zeros(nblocks, dtype=np.int32),
                   {"nblocks": nblocks, "bmin": bmin, "bmax": bmax, "per_row": per_row, "seed": seed,
                    "ordering": "identity"})


# --------------------------------------------------------------------------- c5
def config5(seed=1005, N=128, leaf=512, block=8, top_levels=3, peclet=50.0):
    """3D 27-pt convection-diffusion on N^3, h = 1/(N+1): node kappa ~ lognormal(0,1)
    (drawn in node order); off-diagonal -2 k_i k_j / (k_i + k_j) for all 26 neighbours;
    upwind -h*beta_d on the -e_d face neighbour, beta = Pe*(1, .5, .25); a_ii = sum
    |a_ij| over the full stencil (out-of-grid neighbours with k_j = k_i, nominal
    upwind) -> irreducibly diagonally dominant M-matrix.  Geometric ND with
    `top_levels` levels of top subtrees (8 for the multi-GPU partition), tau = 1e-3."""
    n = N ** 3
    h = 1.0 / (N + 1)
    beta = peclet * np.array([1.0, 0.5, 0.25])
    rng = np.random.Generator(np.random.PCG64(seed))
    kappa = rng.lognormal(0.0, 1.0, size=n)
    offs = _grid_offsets(27)
    rows, cols, oid = _stencil_pairs(N, N, N, offs)
    ki, kj = kappa[rows], kappa[cols]
    vals = -2.0 * ki * kj / (ki + kj)
    del ki, kj
    # upwind on the -e_d faces
    up = np.zeros(len(offs))
    for d, e in enumerate([(-1, 0, 0), (0, -1, 0), (0, 0, -1)]):
        up[offs.index(e)] = -h * beta[d]
    vals += up[oid]
    diag = np.bincount(rows, weights=np.abs(vals), minlength=n)
    # out-of-grid neighbours: k_j = k_i -> -k_i (+ upwind), counted into the diagonal
    present = np.bincount(rows, minlength=n)
    full = np.zeros(n)
    for k in range(len(offs)):
        full += np.abs(-kappa + up[k])
    present_sum = np.zeros(n)
    np.add.at(present_sum, rows, np.abs(-kappa[rows] + up[oid]))
    diag += full - present_sum
    del present
    allr = np.concatenate([rows, np.arange(n)])
    allc = np.concatenate([cols, np.arange(n)])
    allv = np.concatenate([vals, diag])
    del rows, cols, vals, oid
    indptr, indices, data = _csr_from_coo(n, allr, allc, allv)
    perm, sizes, parts = grid_nd(N, N, N, leaf=leaf, block=block, top_levels=top_levels)
    return Problem("c5", n, indptr, indices, data, perm, sizes, 1e-3, parts,
                   {"grid": (N, N, N), "ordering": "geometric ND", "leaf": leaf, "block": block,
                    "top_levels": top_levels, "peclet": peclet, "seed": seed})


CONFIGS = {"c1": config1, "c2": config2, "c3": config3, "c4": config4, "c5": config5}


def make_config(name, **kw) -> Problem:
    return CONFIGS[name](**kw)


# ------------------------------------------------------------------ test inputs
def random_dd(n, density=0.1, seed=0, dominance=1.5, sym_pattern=False):
    """Random sparse matrix with a nonzero diagonal, N(0,1) off-diagonals and
    a_ii = dominance * sum_{j != i} |a_ij| * (random sign) -> strictly row
    diagonally dominant (nonsingular, every principal block nonsingular)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    M = rng.random((n, n)) < density
    if sym_pattern:
        M = M | M.T
    np.fill_diagonal(M, False)
    A = np.where(M, rng.standard_normal((n, n)), 0.0)
    sgn = np.where(rng.random(n) < 0.5, -1.0, 1.0)
    d = dominance * np.abs(A).sum(axis=1)
    d[d == 0] = 1.0
    A[np.arange(n), np.arange(n)] = sgn * d
    return A


def wide_range_matrix(n=300_000, nfar=40, seed=7):
    """Tridiagonal, plus `nfar` symmetric couplings between the first and the last 4000
    unknowns, uniform(-1,1) entries, row-dominant diagonal: candidate key ranges wider
    than 2^18 (the pos-map path of the factor kernel) at a cost the oracle finishes fast."""
    rng = np.random.default_rng(seed)
    i = np.arange(n)
    a = rng.integers(0, 4000, nfar)
    b = rng.integers(n - 4000, n, nfar)
    r = np.concatenate([i, i[1:], i[:-1], a, b])
    c = np.concatenate([i, i[:-1], i[1:], b, a])
    key = np.unique(r.astype(np.int64) * n + c)
    r, c = key // n, key % n
    v = rng.uniform(-1, 1, len(r))
    ip, ix, dv = _csr_from_coo(n, r, c, v)
    rr = np.repeat(np.arange(n), np.diff(ip))
    d = rr == ix
    off = np.bincount(rr, weights=np.abs(dv) * (~d), minlength=n)
    dv[d] = 1.5 * off[rr[d]] + 1.0
    return ip, ix, dv


def dense_to_csr(A):
    n = A.shape[0]
    rows, cols = np.nonzero(A)
    return _csr_from_coo(n, rows, cols, A[rows, cols])
