"""Generators (SURVEY.md 8(d) recipes) and the GMRES harness, pinned on CPU."""
import numpy as np
import scipy.sparse as sp

from harness.gmres import gmres
from inputs.configs import config1, config2, config3
from inputs.nd import grid_nd


def test_c1_shape_and_m_matrix_margin():
    """c1: 32x32 5-pt, nnz = 5*1024 - 4*32 = 4992; seed 1001 is an M-matrix
    (4 - rho(4I - A) = 0.0100), so no pivot block is singular."""
    P = config1()
    assert P.n == 1024 and P.nnz == 4992
    A = sp.csr_matrix((P.data, P.indices, P.indptr), shape=(P.n, P.n)).toarray()
    off = A - np.diag(np.diag(A))
    assert np.all(np.diag(A) == 4.0) and np.all(off <= 0)
    assert np.all(np.abs(off[off != 0] + 1.0) <= 0.1)
    rho = np.abs(np.linalg.eigvals(4.0 * np.eye(P.n) - A)).max()
    assert 4.0 - rho > 0.009
    assert P.block_sizes.sum() == P.n and P.block_sizes.max() == 8


def test_c2_shape_dominance_and_nd():
    """c2: 64^3 7-pt, nnz = N^3 + 6 N^2 (N-1) = 1,810,432; rows diagonally dominant
    (strictly on the boundary) Z-matrix; ND permutation is a bijection; blocks <= 8."""
    P = config2()
    assert P.n == 262144 and P.nnz == 1810432
    A = sp.csr_matrix((P.data, P.indices, P.indptr), shape=(P.n, P.n))
    d = A.diagonal()
    off = A - sp.diags(d)
    assert off.max() <= 0.0
    rowsum = np.asarray(abs(off).sum(axis=1)).ravel()
    assert np.all(d >= rowsum - 1e-12) and np.any(d > rowsum + 1e-3)
    assert np.array_equal(np.sort(P.perm), np.arange(P.n))
    assert P.block_sizes.sum() == P.n and P.block_sizes.max() <= 8
    # unsymmetric values (upwind convection)
    assert abs(A - A.T).max() > 0.1


def test_c3_small_version_shape():
    """c3 recipe at N=6: nnz = 9 (3N-2)^3, a_rr = 1.2 * sum_{c != r} |a_rc|, nodal 3x3 blocks."""
    P = config3(N=6)
    assert P.n == 3 * 216 and P.nnz == 9 * 16 ** 3
    A = sp.csr_matrix((P.data, P.indices, P.indptr), shape=(P.n, P.n))
    d = A.diagonal()
    off = np.asarray(abs(A - sp.diags(d)).sum(axis=1)).ravel()
    np.testing.assert_allclose(d, 1.2 * off, rtol=1e-12)
    assert np.all(P.block_sizes == 3)


def test_grid_nd_separators_decouple_subtrees():
    """In the ND ordering, the two halves of every dissection are not coupled by the
    7-pt stencil: the first leaf block never connects to the last leaf of the other side."""
    perm, sizes, parts = grid_nd(8, 8, 8, leaf=16, block=4, top_levels=1)
    assert len(perm) == 512 and sizes.sum() == 512
    assert set(parts.tolist()) == {-1, 0, 1}
    iperm = np.empty(512, int); iperm[perm] = np.arange(512)
    st = np.concatenate([[0], np.cumsum(sizes)])
    blk = np.repeat(np.arange(len(sizes)), sizes)
    # nodes of subtree 0 and subtree 1 are never 7-pt neighbours
    part_of = parts[blk[iperm]]
    for v in range(512):
        x, y, z = v % 8, (v // 8) % 8, v // 64
        for dx, dy, dz in [(1, 0, 0), (0, 1, 0), (0, 0, 1)]:
            if x + dx < 8 and y + dy < 8 and z + dz < 8:
                w = (x + dx) + 8 * ((y + dy) + 8 * (z + dz))
                a, b = part_of[v], part_of[w]
                assert not (a >= 0 and b >= 0 and a != b)


def test_gmres_diag_polynomial_exactness():
    """Unpreconditioned GMRES on diag(1..k), k <= restart, converges in <= k steps."""
    k = 12
    D = np.arange(1, k + 1, dtype=float)
    x, its, ok, _ = gmres(lambda v: D * v, np.ones(k), tol=1e-12)
    assert ok and its <= k
    np.testing.assert_allclose(x, 1.0 / D, rtol=1e-10)


def test_gmres_exact_preconditioner_one_step():
    rng = np.random.default_rng(0)
    A = rng.standard_normal((40, 40)) + 10 * np.eye(40)
    Ainv = np.linalg.inv(A)
    x, its, ok, _ = gmres(lambda v: A @ v, np.ones(40), precond=lambda v: Ainv @ v, tol=1e-8)
    assert ok and its == 1


def test_gmres_restarts():
    rng = np.random.default_rng(1)
    n = 200
    A = np.diag(np.linspace(1, 1000, n)) + 0.1 * rng.standard_normal((n, n))
    x, its, ok, hist = gmres(lambda v: A @ v, np.ones(n), restart=10, tol=1e-8, max_restarts=500)
    assert ok and its > 10
    assert np.linalg.norm(A @ x - 1.0) / np.sqrt(n) <= 1e-8 * 1.01


def test_config4_recipe_small():
    from inputs.configs import config4
    P = config4(nblocks=50, per_row=5)
    Q = config4(nblocks=50, per_row=5)
    assert np.array_equal(P.data, Q.data) and np.array_equal(P.indices, Q.indices)
    bs = P.block_sizes
    assert bs.min() >= 16 and bs.max() <= 64 and bs.sum() == P.n
    # every block row: the diagonal block + 5 distinct off-diagonal blocks, all dense
    bst = np.concatenate([[0], np.cumsum(bs)])
    r0 = np.diff(P.indptr)[bst[:-1]]
    for i in range(50):
        rows = np.arange(bst[i], bst[i + 1])
        assert np.all(np.diff(P.indptr)[rows] == r0[i])
    import scipy.sparse as sp
    A = sp.csr_matrix((P.data, P.indices, P.indptr), shape=(P.n, P.n))
    d = np.abs(A.diagonal()); off = np.abs(A).sum(axis=1).A1 - d
    np.testing.assert_allclose(d / off, 1.5, rtol=1e-12)


def test_config5_recipe_small():
    from inputs.configs import config5
    N = 12
    P = config5(N=N, top_levels=1)
    assert P.nnz == (3 * N - 2) ** 3          # 27-pt stencil incl. self
    import scipy.sparse as sp
    A = sp.csr_matrix((P.data, P.indices, P.indptr), shape=(P.n, P.n)).tocoo()
    off = A.row != A.col
    assert np.all(A.data[off] < 0)            # Z-matrix
    d = sp.csr_matrix(A).diagonal()
    s = np.bincount(A.row[off], weights=-A.data[off], minlength=P.n)
    assert np.all(d >= s * (1 - 1e-14))       # diagonally dominant (strict on the boundary)
    assert np.any(d > s * (1 + 1e-6))
    assert sorted(P.perm.tolist()) == list(range(P.n))
    assert set(np.unique(P.block_part)) == {-1, 0, 1}
