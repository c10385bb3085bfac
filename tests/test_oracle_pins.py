"""Pins of the CPU oracle to things other than itself (run without a GPU).

Each test names what fixes the expected value: a worked example of the paper /
SPEC, a closed form, a library routine, a mathematical identity, or a literal
transcription of Alg. 1 on tiny inputs.
"""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla

import oracle
from inputs.configs import dense_to_csr, random_dd
from tests.parity import dense_LPU

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def fac(A, bs, tau, agg=False, max_block=128):
    ip, ix, dv = dense_to_csr(A)
    return oracle.factor(ip, ix, dv, bs, tau, aggregate=agg, max_block=max_block)


def random_partition(n, rng, maxb=8):
    out = []
    while sum(out) < n:
        out.append(int(min(rng.integers(1, maxb + 1), n - sum(out))))
    return out


# ------------------------------------------------------------ worked examples
def test_spec_2x2_worked_example():
    """[[2,1],[1,2]], tau=0 -> L=[[1,0],[.5,1]], pivots diag(2,1.5), U=[[1,.5],[0,1]]."""
    g = json.load(open(os.path.join(GOLD, "spec_2x2.json")))
    A = np.array(g["A"])
    f = fac(A, g["block_sizes"], g["tau"])
    L, P, U = dense_LPU(f, 2)
    np.testing.assert_allclose(L, g["L"], atol=1e-15)
    np.testing.assert_allclose(P, g["pivots"], atol=1e-15)
    np.testing.assert_allclose(U, g["U"], atol=1e-15)
    # D stores the inverted pivots
    np.testing.assert_allclose(f.block(1)[6], [[1 / 1.5]], atol=1e-15)


def test_spec_forced_merge_gives_inverse():
    """merging the two scalar blocks of [[2,1],[1,2]] gives one 2x2 block, D = A^{-1}."""
    A = np.array([[2.0, 1.0], [1.0, 2.0]])
    f = fac(A, [1, 1], 0.0, agg=True)
    assert f.nblk == 1 and f.n_merges == 1
    np.testing.assert_allclose(f.block(0)[6], np.linalg.inv(A), atol=1e-15)


def test_aggregate_test_worked_examples():
    g = json.load(open(os.path.join(GOLD, "aggregate_test.json")))
    for c in g["cases"]:
        p, q, r, s, t, r2, s2, t2, u, v = c["args"]
        mu = p * (p + r + s + r2 + s2) + q * (q + t + t2)
        nu = (p + q) * (p + q + u + v)
        assert (mu, nu) == (c["mu"], c["nu"])
        assert oracle.aggregate_test(*c["args"]) == c["merge"]
    # max_block caps the merge (R9)
    assert oracle.aggregate_test(1, 1, 0, 0, 0, 0, 0, 0, 0, 0, max_block=2)
    assert not oracle.aggregate_test(1, 1, 0, 0, 0, 0, 0, 0, 0, 0, max_block=1)


def test_identity_chain_merges_to_one_block():
    """SPEC.md:396 / PAPER.md:1436-1440: decoupled scalars merge step by step into one block."""
    f = fac(np.eye(4), [1, 1, 1, 1], 1e-2, agg=True)
    assert f.nblk == 1 and f.n_merges == 3
    np.testing.assert_allclose(f.block(0)[6], np.eye(4), atol=0)


# ------------------------------------------------------------ closed forms
@pytest.mark.parametrize("seed", range(6))
def test_tau0_is_exact_block_LDU(seed):
    """tau = 0 keeps every nonzero row: L P U = A to rounding (BASELINE north_star)."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(10, 80))
    A = random_dd(n, 0.15, seed)
    bs = random_partition(n, rng)
    f = fac(A, bs, 0.0)
    L, P, U = dense_LPU(f, n)
    assert np.abs(L @ P @ U - A).max() <= 1e-12 * np.abs(A).max()


def test_tau0_matches_scipy_lu_without_pivoting():
    """Library routine: a column-diagonally-dominant matrix needs no row swaps in
    LAPACK getrf, so A = L_s U_s with L_s unit lower; the scalar BILU at tau=0 gives
    the same L, pivots diag(U_s) and unit U = diag(U_s)^{-1} U_s."""
    A = random_dd(30, 0.3, 7).T.copy()            # column dominant
    Pm, Ls, Us = sla.lu(A)
    assert np.array_equal(Pm, np.eye(30))
    f = fac(A, [1] * 30, 0.0)
    L, P, U = dense_LPU(f, 30)
    np.testing.assert_allclose(L, Ls, atol=1e-13)
    np.testing.assert_allclose(np.diag(P), np.diag(Us), rtol=1e-13)
    np.testing.assert_allclose(U, np.diag(1 / np.diag(Us)) @ Us, atol=1e-13)


def test_tridiagonal_thomas_closed_form():
    """No fill on a tridiagonal matrix: p_1 = a_11, p_i = a_ii - a_{i,i-1} a_{i-1,i} / p_{i-1},
    l_{i,i-1} = a_{i,i-1}/p_{i-1}, Ũ_{i-1,i} = a_{i-1,i} (ILU(0)-pattern results are exact)."""
    rng = np.random.default_rng(3)
    n = 50
    sub, sup = rng.uniform(-1, 1, n - 1), rng.uniform(-1, 1, n - 1)
    dia = 3.0 + rng.uniform(0, 1, n)
    A = np.diag(dia) + np.diag(sub, -1) + np.diag(sup, 1)
    f = fac(A, [1] * n, 1e-6)
    p = np.zeros(n)
    p[0] = dia[0]
    for i in range(1, n):
        p[i] = dia[i] - sub[i - 1] * sup[i - 1] / p[i - 1]
    for K in range(n):
        s, e, rows, L, cols, Ut, D = f.block(K)
        np.testing.assert_allclose(D, [[1 / p[K]]], rtol=1e-14)
        if K < n - 1:
            assert list(rows) == [K + 1] and list(cols) == [K + 1]
            np.testing.assert_allclose(L[0, 0], sub[K] / p[K], rtol=1e-14)
            np.testing.assert_allclose(Ut[0, 0], sup[K], rtol=1e-14)


def test_block_tridiagonal_aligned_partition_is_exact():
    """Block Thomas: P_1 = A_11, P_i = A_ii - A_{i,i-1} P_{i-1}^{-1} A_{i-1,i}; fill stays
    inside the dense diagonal blocks, so BILU with tau=0 reproduces it."""
    rng = np.random.default_rng(5)
    bs = [3, 5, 2, 4, 6]
    st = np.concatenate([[0], np.cumsum(bs)])
    n = st[-1]
    A = np.zeros((n, n))
    for i in range(len(bs)):
        A[st[i]:st[i + 1], st[i]:st[i + 1]] = rng.standard_normal((bs[i], bs[i])) + 8 * np.eye(bs[i])
        if i:
            A[st[i]:st[i + 1], st[i - 1]:st[i]] = rng.standard_normal((bs[i], bs[i - 1]))
            A[st[i - 1]:st[i], st[i]:st[i + 1]] = rng.standard_normal((bs[i - 1], bs[i]))
    f = fac(A, bs, 0.0)
    Pprev = None
    for i in range(len(bs)):
        Aii = A[st[i]:st[i + 1], st[i]:st[i + 1]]
        if i == 0:
            Pi = Aii
        else:
            Pi = Aii - A[st[i]:st[i + 1], st[i - 1]:st[i]] @ np.linalg.solve(Pprev, A[st[i - 1]:st[i], st[i]:st[i + 1]])
        np.testing.assert_allclose(np.linalg.inv(f.block(i)[6]), Pi, rtol=1e-12, atol=1e-12)
        Pprev = Pi


def test_tau_infinite_is_block_jacobi():
    """tau = 1e300 drops every off-diagonal row/col: L = U = I, D_K = Ã_KK^{-1}."""
    A = random_dd(40, 0.2, 11)
    bs = [3, 5, 2, 4, 6, 1, 3, 8, 4, 4]
    f = fac(A, bs, 1e300)
    st = np.concatenate([[0], np.cumsum(bs)])
    assert len(f.Li) == 0 and len(f.Ui) == 0
    for K in range(len(bs)):
        np.testing.assert_allclose(f.block(K)[6], np.linalg.inv(A[st[K]:st[K + 1], st[K]:st[K + 1]]),
                                   rtol=1e-12, atol=1e-14)


def test_single_block_is_the_inverse():
    A = random_dd(17, 0.5, 2)
    f = fac(A, [17], 0.3)
    np.testing.assert_allclose(f.block(0)[6], np.linalg.inv(A), rtol=1e-12, atol=1e-14)


# ------------------------------------------------------- residual characterisation
def residual_check(A, f, tau, slack=1e-12):
    """R = A - L P U vanishes on every kept position and on the diagonal blocks; a
    dropped L row / U column equals the unscaled dropped entries and its scaled form
    is <= tau; a kept one is > tau.  These equations
    determine the factors uniquely, given the partition."""
    n = A.shape[0]
    L, P, U = dense_LPU(f, n)
    R = A - L @ P @ U
    scale = np.abs(A).max()
    for K in range(f.nblk):
        s, e, rows, Lp, cols, Ut, D = f.block(K)
        assert np.abs(R[s:e, s:e]).max() <= slack * scale
        kept = set(int(r) for r in rows)
        for i in range(e, n):
            Ri = R[i, s:e]
            if i in kept:
                assert np.abs(Ri).max() <= slack * scale
                assert np.abs(L[i, s:e]).max() > tau
            else:
                assert np.abs(Ri @ D).max() <= tau * (1 + 1e-10) + slack
        keptc = set(int(c) for c in cols)
        for j in range(e, n):
            Rj = R[s:e, j]
            if j in keptc:
                assert np.abs(Rj).max() <= slack * scale
                assert np.abs(D @ Ut[:, list(cols).index(j)]).max() > tau
            else:
                assert np.abs(D @ Rj).max() <= tau * (1 + 1e-10) + slack


@pytest.mark.parametrize("seed,tau", [(0, 1e-3), (1, 1e-2), (2, 5e-2), (3, 0.3), (4, 0.0)])
def test_residual_characterisation(seed, tau):
    rng = np.random.default_rng(100 + seed)
    n = 60
    A = random_dd(n, 0.12, 100 + seed, dominance=1.3)
    bs = random_partition(n, rng)
    f = fac(A, bs, tau)
    residual_check(A, f, tau)


def test_residual_characterisation_scalar_tridiag_plus_fill():
    A = random_dd(45, 0.08, 42, dominance=1.1)
    f = fac(A, [1] * 45, 2e-2)
    residual_check(A, f, 2e-2)


# ------------------------------------------------------------ aggregation identity
@pytest.mark.parametrize("seed,tau", [(0, 1e-3), (1, 1e-2), (2, 0.0)])
def test_merge_leaves_operator_unchanged(seed, tau):
    """merging k-1 and k rewrites L D^{-1} U without changing it,
    so L P U with aggregation equals L P U without (and the merged diagonal blocks are
    the inverses of the merged pivots)."""
    rng = np.random.default_rng(200 + seed)
    n = 70
    A = random_dd(n, 0.1, 200 + seed)
    bs = random_partition(n, rng, maxb=4)
    f0 = fac(A, bs, tau, agg=False)
    f1 = fac(A, bs, tau, agg=True)
    assert f1.n_merges > 0
    L0, P0, U0 = dense_LPU(f0, n)
    L1, P1, U1 = dense_LPU(f1, n)
    assert np.abs(L0 @ P0 @ U0 - L1 @ P1 @ U1).max() <= 1e-12 * np.abs(A).max()
    # unit triangularity of the merged factors
    for K in range(f1.nblk):
        s, e, rows, Lp, cols, Ut, D = f1.block(K)
        assert np.all(np.asarray(rows) >= e) and np.all(np.asarray(cols) >= e)


def test_merge_sizes_respect_max_block():
    A = random_dd(120, 0.3, 9)
    f = fac(A, [4] * 30, 1e-3, agg=True, max_block=16)
    assert np.diff(f.bstart).max() <= 16


# ------------------------------------------------------------ Alg. 1 transcription
def crout_ilu_alg1(A, tau):
    """Literal transcription of Alg. 1, dense loops, n <= 60.
    Returns L (unit lower, scaled) and U (upper, unscaled incl. the diagonal)."""
    n = A.shape[0]
    L = np.zeros((n, n))
    U = np.zeros((n, n))
    for k in range(n):
        l = A[:, k].copy()                      # l_ik <- a_ik, i >= k
        l[:k] = 0.0
        for j in range(k):
            if U[j, k] != 0.0:
                for i in range(k, n):
                    if L[i, j] != 0.0:
                        l[i] -= L[i, j] * U[j, k]
        u = A[k, :].copy()                      # u_ki <- a_ki, i >= k
        u[:k] = 0.0
        for j in range(k):
            if L[k, j] != 0.0:
                for i in range(k, n):
                    if U[j, i] != 0.0:
                        u[i] -= L[k, j] * U[j, i]
        lkk = l[k]
        for i in range(k + 1, n):               # drop |l_ik| <= tau |l_kk|, then scale
            if abs(l[i]) <= tau * abs(lkk):
                l[i] = 0.0
        L[k:, k] = l[k:] / lkk
        for i in range(k + 1, n):               # drop |u_ki| <= tau |u_kk|
            if abs(u[i]) <= tau * abs(u[k]):
                u[i] = 0.0
        U[k, k:] = u[k:]
    return L, U


@pytest.mark.parametrize("seed,tau", [(0, 1e-2), (1, 5e-2), (2, 1e-3)])
def test_scalar_partition_is_alg1(seed, tau):
    """BILU(---) reduces to the scalar Crout ILU."""
    A = random_dd(40, 0.12, 300 + seed, dominance=1.2)
    Lr, Ur = crout_ilu_alg1(A, tau)
    f = fac(A, [1] * 40, tau)
    L, P, U = dense_LPU(f, 40)
    np.testing.assert_allclose(L, Lr, atol=1e-12)
    np.testing.assert_allclose(P @ U, Ur, atol=1e-12)


# ------------------------------------------------------------ apply
def test_apply_solves_LPU():
    A = random_dd(50, 0.1, 77)
    bs = [5] * 10
    for agg in (False, True):
        f = fac(A, bs, 1e-2, agg=agg)
        L, P, U = dense_LPU(f, 50)
        x = np.random.default_rng(1).standard_normal(50)
        y = oracle.apply(f, x)
        np.testing.assert_allclose(L @ P @ U @ y, x, atol=1e-12 * np.abs(x).max())


def test_breakdown_is_reported():
    A = np.array([[1.0, 1.0, 0.0], [1.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
    with pytest.raises(oracle.OracleError, match="breakdown in block 0"):
        fac(A, [2, 1], 0.0)


def test_decision_override_replays():
    """Decision replay (SURVEY.md 8(c) reading 15): a forced keep of a dropped row."""
    A = np.array([[2.0, 0.0], [0.02, 1.0]])
    f = fac(A, [1, 1], 0.01)                     # l = 0.01 == tau -> dropped (ties drop, R2)
    assert len(f.Li) == 0 and f.n_near == 1 and f.min_margin == 0.0
    ip, ix, dv = dense_to_csr(A)
    g = oracle.factor(ip, ix, dv, [1, 1], 0.01, aggregate=False, overrides=[(0, 0, 1, 1)])
    assert list(g.Li) == [1] and g.n_override_applied == 1


def test_decision_override_guard():
    """Replay is bounded (R15): an override of a decision far from tau (here l = 0.5, margin
    49 at tau = 0.01) is refused with an error instead of being copied into the oracle;
    an override naming no decision is not applied."""
    A = np.array([[2.0, 0.0], [1.0, 1.0]])
    ip, ix, dv = dense_to_csr(A)
    with pytest.raises(oracle.OracleError, match="override refused"):
        oracle.factor(ip, ix, dv, [1, 1], 0.01, aggregate=False, overrides=[(0, 0, 1, 0)])
    g = oracle.factor(ip, ix, dv, [1, 1], 0.01, aggregate=False, overrides=[(1, 0, 5, 1)])
    assert g.n_override_applied == 0 and list(g.Li) == [1]


def test_aggregation_segments_reading_r18():
    """seg (R18): one segment == no segments; all-distinct segments == no
    aggregation; piecewise segments: merged blocks never straddle a segment boundary and
    the operator L P U equals the unmerged one."""
    from inputs.configs import config5
    P = config5(N=10, top_levels=1)
    ip, ix, dv = oracle.permute_csr(P.indptr, P.indices, P.data, P.perm)
    bs = P.block_sizes
    nb = len(bs)
    a = oracle.factor(ip, ix, dv, bs, P.tau)
    b = oracle.factor(ip, ix, dv, bs, P.tau, seg=np.zeros(nb, np.int32))
    assert np.array_equal(a.bstart, b.bstart) and np.array_equal(a.Lv, b.Lv)
    c = oracle.factor(ip, ix, dv, bs, P.tau, seg=np.arange(nb, dtype=np.int32))
    d = oracle.factor(ip, ix, dv, bs, P.tau, aggregate=False)
    assert c.n_merges == 0 and np.array_equal(c.bstart, d.bstart)
    seg = np.where(P.block_part >= 0, P.block_part, -1).astype(np.int32)
    e = oracle.factor(ip, ix, dv, bs, P.tau, seg=seg)
    assert 0 < e.n_merges < a.n_merges + 1
    bst = np.concatenate([[0], np.cumsum(bs)])
    seg_of_row = np.repeat(seg, bs)
    for K in range(e.nblk):
        s0, s1 = int(e.bstart[K]), int(e.bstart[K + 1])
        assert len(np.unique(seg_of_row[s0:s1])) == 1
    from tests.parity import dense_LPU
    L1, P1, U1 = dense_LPU(e, P.n)
    L0, P0, U0 = dense_LPU(d, P.n)
    M1, M0 = L1 @ P1 @ U1, L0 @ P0 @ U0
    assert np.abs(M1 - M0).max() <= 1e-12 * np.abs(M0).max()


# ---------------- Sec. 3.6 diagonal-block perturbation (R19) ----------------
PT = (1e-2, 1e-1, 1e12)          # tau_p, rho, cond_max (SPEC default)


def test_perturbation_inactive_on_well_conditioned_blocks():
    """Strictly dominant input: no pivot block is singular or ill-conditioned, so the
    factors with the perturbation enabled are those without it."""
    A = random_dd(120, 0.1, 11, dominance=1.5)
    ip, ix, dv = dense_to_csr(A)
    bs = [4] * 30
    a = oracle.factor(ip, ix, dv, bs, 1e-2)
    b = oracle.factor(ip, ix, dv, bs, 1e-2, perturb=PT)
    assert b.n_perturbed == 0
    assert np.array_equal(a.Lv, b.Lv) and np.array_equal(a.Dv, b.Dv) and np.array_equal(a.Uv, b.Uv)


def test_perturbation_zero_column_closed_form():
    """Pivot block [[2, 0], [1, 0]] (zero column, "if d = 0"): its largest entry is
    the diagonal zero, which becomes 0 (1 + rho 0) + sign(0) tau_p alpha = tau_p alpha;
    rows are then nonzero.  D = [[2, 0], [1, t]]^{-1} = [[1/2, 0], [-1/(2t), 1/t]]."""
    A = np.array([[2.0, 0.0, 0.5], [1.0, 0.0, 0.0], [0.0, 0.0, 4.0]])
    ip, ix, dv = dense_to_csr(A)
    with pytest.raises(oracle.OracleError):
        oracle.factor(ip, ix, dv, [2, 1], 0.0, aggregate=False)
    f = oracle.factor(ip, ix, dv, [2, 1], 0.0, aggregate=False, perturb=PT)
    t = PT[0] * 4.0                                   # alpha = max |a_ij| = 4
    D0 = f.block(0)[6]
    np.testing.assert_allclose(D0, [[0.5, 0.0], [-1.0 / (2 * t), 1.0 / t]], rtol=1e-14)
    assert f.n_perturbed == 1


def test_perturbation_singular_block_bounded_modification():
    """A singular pivot block ([[1, 1], [1, 1]] inside a dominant matrix) is perturbed and the
    factorization completes; with tau = 0 (no dropping) L P U - Ã is zero except on the
    perturbed diagonal block, where each entry moved by at most rho |p| delta + tau_p alpha
    per perturbation pass (SPEC: a bounded modification)."""
    rng = np.random.default_rng(5)
    n = 12
    A = np.zeros((n, n))
    A[np.arange(n), np.arange(n)] = 6.0
    A[np.arange(n - 1), np.arange(1, n)] = rng.uniform(-1, 1, n - 1)
    A[np.arange(1, n), np.arange(n - 1)] = rng.uniform(-1, 1, n - 1)
    A[4:6, 4:6] = [[1.0, 1.0], [1.0, 1.0]]            # singular diagonal block of block 2
    A[4, 3] = A[5, 6] = A[3, 4] = A[6, 5] = 0.0         # decouple -> its Schur block stays singular
    ip, ix, dv = dense_to_csr(A)
    bs = [2] * 6
    with pytest.raises(oracle.OracleError):
        oracle.factor(ip, ix, dv, bs, 0.0, aggregate=False)
    f = oracle.factor(ip, ix, dv, bs, 0.0, aggregate=False, perturb=PT)
    assert f.n_perturbed == 1
    from tests.parity import dense_LPU
    L, P, U = dense_LPU(f, n)
    E = L @ P @ U - A
    mask = np.zeros((n, n), bool); mask[4:6, 4:6] = True
    assert np.abs(E[~mask]).max() <= 1e-13 * np.abs(A).max()
    alpha, (tp, rho, _) = np.abs(A).max(), PT
    pmax = np.abs(L @ P @ U)[4:6, 4:6].max()
    assert np.abs(E[mask]).max() > 0
    assert np.abs(E[mask]).max() <= 3 * (rho * pmax * pmax + tp * alpha)


# ------------------------------------------------------------ ILU(1,tau) block estimate (Sec. 3.4)
def _csr(D):
    import scipy.sparse as sp
    A = sp.csr_matrix(np.asarray(D, dtype=np.float64))
    A.sort_indices()
    return A.indptr, A.indices, A.data


def test_ilu1_sets_hand_trace():
    """Hand trace of PAPER.md:1178-1198 on a 4x4 unsymmetric matrix (tests/golden/ilu1_hand_4x4.json).

    tau=0.5: I~_1 = {2} only through the ILU(1) fill a_21 = -a_20 a_01 / a_00 (|5*1| >= .5|2*4|);
    the direct a_31 = .1 < .5*4 is dropped.  J~_2 = {3} only through the fill of row 2 via i=0
    (|a_20 a_03| = 5 >= .5|a_00 a_22|).  tau=0.625 sits exactly on |5| = tau*8 (kept, ">="), and
    J~_0 loses a_01 = a_03 = 1 < 1.25.  tau=0.63 drops the fill.  tau=0.01 keeps a_31.
    Using a_kj instead of a_jk in the fill (a transposed operand) gives I~_1 = {} at tau=0.5."""
    g = json.load(open(os.path.join(GOLD, "ilu1_hand_4x4.json")))
    ip, ix, dv = _csr(g["A"])
    for c in g["cases"]:
        for k in range(4):
            assert list(oracle.ilu1_set(ip, ix, dv, c["tau"], k, True)) == c["I"][k], (c["tau"], k)
            assert list(oracle.ilu1_set(ip, ix, dv, c["tau"], k, False)) == c["J"][k], (c["tau"], k)
        if "blocks_max8" in c:
            # k0=0: t=1 f=8,c'=7 (24<=28); t=2 f=12,c'=9 (36<=36); t=3 f=16 <= c'+16 = 26
            assert list(oracle.ilu1_blocks(ip, ix, dv, c["tau"], 8)) == c["blocks_max8"]
            assert list(oracle.ilu1_blocks(ip, ix, dv, c["tau"], 2)) == c["blocks_max2"]


def test_ilu1_identity_blocks_of_five():
    """Identity: f_{l+1} = (l+1)^2, c' = l+1, so l+1 <= 5 (SURVEY S:303 / §8c: f6 = 36 > 6+24)."""
    n = 23
    ip, ix, dv = np.arange(n + 1), np.arange(n), np.ones(n)
    assert list(oracle.ilu1_blocks(ip, ix, dv, 1e-2, 128)) == [5, 5, 5, 5, 3]
    assert list(oracle.ilu1_blocks(ip, ix, dv, 1e-2, 3)) == [3] * 7 + [2]      # the max_size cap
    assert list(oracle.ilu1_blocks(ip, ix, dv, 1e-2, 1)) == [1] * n


def test_ilu1_tridiagonal_hand_trace():
    """Tridiagonal(-1, 4, -1), n=8, tau=.1: I~_k = J~_k = {k+1}.  From k0=0 the block keeps r=s=1:
    f = 8,15,24,35 against c' = 6,9,12,15 (4/3 test or c'+4(l+1)) -> l=5; t=5: f=48 > 18+24.
    From k0=5: f=8 <= 4/3*6, then r=s=0, f=9 <= 4/3*7 -> [5, 3].  Not removing the in-block
    entries from r, s would stop the first block at 2 (t=2: f=27 > 9+12)."""
    import scipy.sparse as sp
    T = sp.diags([-np.ones(7), 4 * np.ones(8), -np.ones(7)], [-1, 0, 1]).tocsr()
    T.sort_indices()
    assert list(oracle.ilu1_blocks(T.indptr, T.indices, T.data, 0.1, 8)) == [5, 3]


def test_ilu1_star_fill_path_theorem():
    """Dense first row/column + diagonal (a star eliminated centre-first): every fill path has one
    intermediate vertex (0), so with tau=0 the ILU(1) estimate is the exact LU pattern: I~_k =
    J~_k = {k+1..n-1} (fill-path theorem, Rose-Tarjan)."""
    rng = np.random.default_rng(3)
    n = 9
    D = np.diag(rng.uniform(5, 6, n))
    D[0, 1:] = rng.uniform(0.5, 1, n - 1)
    D[1:, 0] = rng.uniform(0.5, 1, n - 1)
    ip, ix, dv = _csr(D)
    for k in range(n):
        assert list(oracle.ilu1_set(ip, ix, dv, 0.0, k, True)) == list(range(k + 1, n))
        assert list(oracle.ilu1_set(ip, ix, dv, 0.0, k, False)) == list(range(k + 1, n))


def test_ilu1_sets_inside_exact_lu_pattern_and_monotone():
    """tau=0: pattern(A) below/right of k  <=  I~_k, J~_k  <=  pattern of the exact (no pivoting) LU
    factors (generic values: no cancellation); the sets shrink as tau grows."""
    rng = np.random.default_rng(11)
    n = 40
    M = (rng.random((n, n)) < 0.08) * rng.uniform(-1, 1, (n, n))
    M += np.diag(np.abs(M).sum(1) + 1.0)
    P, Lf, Uf = sla.lu(M)
    assert np.allclose(P, np.eye(n))          # diagonally dominant: no row exchanges
    ip, ix, dv = _csr(M)
    for k in range(n):
        lo = set(oracle.ilu1_set(ip, ix, dv, 0.0, k, True))
        up = set(oracle.ilu1_set(ip, ix, dv, 0.0, k, False))
        assert set(np.nonzero(M[k + 1:, k])[0] + k + 1) <= lo <= set(np.nonzero(np.abs(Lf[k + 1:, k]) > 0)[0] + k + 1)
        assert set(np.nonzero(M[k, k + 1:])[0] + k + 1) <= up <= set(np.nonzero(np.abs(Uf[k, k + 1:]) > 0)[0] + k + 1)
        prev_lo, prev_up = lo, up
        for tau in (1e-3, 1e-2, 1e-1, 1.0):
            lo_t = set(oracle.ilu1_set(ip, ix, dv, tau, k, True))
            up_t = set(oracle.ilu1_set(ip, ix, dv, tau, k, False))
            assert lo_t <= prev_lo and up_t <= prev_up
            prev_lo, prev_up = lo_t, up_t
    b = oracle.ilu1_blocks(ip, ix, dv, 1e-2, 8)
    assert b.sum() == n and b.min() >= 1 and b.max() <= 8


# ------------------------------------------------------------ cosine-based blocking (Sec. 3.2)
def _pattern_csr(rows, n):
    ip = np.zeros(n + 1, dtype=np.int64)
    for i, r in enumerate(rows):
        ip[i + 1] = ip[i] + len(r)
    return ip, np.concatenate([np.asarray(sorted(r), dtype=np.int32) for r in rows])


def test_cosine_hand_trace():
    """Hand trace of PAPER.md:934-947 on a 6x6 pattern (tests/golden/cosine_hand_6x6.json).
    No row/column exceeds mu + 2 sigma (rows: mu=3, 4 sigma^2 = 240/36; columns: 48/36).
    tau=.8: row 0 (nz 4) takes row 2 on the equality 4^2 = .8*4*5 but not row 1 (3^2 < 9.6);
    rows 3,4: 2^2 < .8*2*3.  tau=.75: 3^2 >= .75*12 also takes row 1.  max_size=2 stops the
    first group after row 1, and row 2 (with rows 3, 4: 1 < 7.5, 4 < 11.25) stays alone.
    Grouping columns instead of rows (a transposed operand) gives {0,1,2} at tau=.8."""
    g = json.load(open(os.path.join(GOLD, "cosine_hand_6x6.json")))
    ip, ix = _pattern_csr(g["rows"], 6)
    for c in g["cases"]:
        q, s = oracle.cosine_blocks(ip, ix, c["tau"], c["max_size"])
        assert list(q) == c["q"] and list(s) == c["sizes"], c


def test_cosine_ignores_dense_rows_and_columns():
    """Arrow pattern (dense row 0 and column 0 + diagonal), n=10, tau=.2: row/column 0 have
    10 > mu + 2 sigma nonzeros (mu = 2.8, sigma = 2.4) and are ignored; the other rows then share
    no kept column, so every group is a singleton.  Keeping column 0 would put rows 1.. together
    (1^2 >= .2*2*2)."""
    n = 10
    rows = [list(range(n))] + [[0, i] for i in range(1, n)]
    ip, ix = _pattern_csr(rows, n)
    q, s = oracle.cosine_blocks(ip, ix, 0.2, 128)
    assert list(s) == [1] * n and list(q) == list(range(n))


def test_cosine_cap_identical_rows():
    """Identical rows (sigma = 0, nothing ignored): the first row takes the next ones up to max_size."""
    n = 10
    ip, ix = _pattern_csr([list(range(n))] * n, n)
    q, s = oracle.cosine_blocks(ip, ix, 0.8, 4)
    assert list(s) == [4, 4, 2] and list(q) == list(range(n))


def test_cosine_recovers_permuted_block_diagonal():
    """Dense diagonal blocks [3,1,4,2,5] under a random symmetric permutation: rows of one block
    have identical patterns (cosine 1) and rows of different blocks share no column, so the
    groups are exactly the blocks, in the order of their first row."""
    sizes = [3, 1, 4, 2, 5]
    n = sum(sizes)
    lab = np.repeat(np.arange(len(sizes)), sizes)
    perm = np.random.default_rng(4).permutation(n)          # new row r = old row perm[r]
    lab_new = lab[perm]
    rows = [list(np.nonzero(lab_new == lab_new[r])[0]) for r in range(n)]
    ip, ix = _pattern_csr(rows, n)
    q, s = oracle.cosine_blocks(ip, ix, 0.8, 128)
    groups, seen = [], set()
    for r in range(n):
        if lab_new[r] not in seen:
            seen.add(lab_new[r])
            groups.append(list(np.nonzero(lab_new == lab_new[r])[0]))
    assert list(s) == [len(g) for g in groups]
    assert list(q) == [x for g in groups for x in g]


# ------------------------------------------------------------ maximum weight matching (Sec. 3.1)
def test_mwm_hand_2x2():
    """[[1,3],[2,1]]: the transversal {a01, a10} (product 6) beats the diagonal (1).  Column maxima
    (2, 3); the scaled matrix has 1 on the matching: D_l = I, D_r = diag(1/2, 1/3)."""
    A = np.array([[1.0, 3.0], [2.0, 1.0]])
    ip, ix, dv = dense_to_csr(A)
    sigma, dl, dr = oracle.mwm(ip, ix, dv)
    assert list(sigma) == [1, 0]
    S = dl[:, None] * A * dr[None, :]
    np.testing.assert_allclose(S, [[0.5, 1.0], [1.0, 1.0 / 3.0]], rtol=1e-14)


def _mwm_random(n, seed):
    rng = np.random.default_rng(seed)
    A = (rng.random((n, n)) < 0.08) * rng.standard_normal((n, n)) * np.exp(rng.uniform(-4, 4, (n, n)))
    A[np.arange(n), rng.permutation(n)] += rng.uniform(0.1, 1.0, n)    # a perfect matching exists
    return A


@pytest.mark.parametrize("seed", range(4))
def test_mwm_optimum_matches_linear_sum_assignment(seed):
    """The transversal's objective equals scipy's linear_sum_assignment (an independent solver)
    on the costs c_ij = log(cmax_j) - log|a_ij| (missing entries excluded by a prohibitive cost),
    and the scalings satisfy |d_l a d_r| <= 1 with equality on the matching."""
    from scipy.optimize import linear_sum_assignment
    n = 60
    A = _mwm_random(n, seed)
    ip, ix, dv = dense_to_csr(A)
    sigma, dl, dr = oracle.mwm(ip, ix, dv)
    assert sorted(sigma) == list(range(n)) and np.all(A[np.arange(n), sigma] != 0)
    cmax = np.abs(A).max(axis=0)
    with np.errstate(divide="ignore"):
        C = np.where(A != 0, np.log(cmax)[None, :] - np.log(np.abs(A)), 1e6)
    r, c = linear_sum_assignment(C)
    assert abs(C[np.arange(n), sigma].sum() - C[r, c].sum()) < 1e-9
    S = np.abs(dl[:, None] * A * dr[None, :])
    assert S.max() <= 1 + 1e-12
    np.testing.assert_allclose(S[np.arange(n), sigma], 1.0, rtol=1e-12)


def test_mwm_permuted_diagonal_and_singular():
    """One entry per row and column: the matching is forced and every scaled entry is 1.  A
    structurally singular pattern (an empty column) has no perfect matching."""
    rng = np.random.default_rng(2)
    n = 25
    perm = rng.permutation(n)
    A = np.zeros((n, n))
    A[np.arange(n), perm] = rng.uniform(-5, 5, n)
    ip, ix, dv = dense_to_csr(A)
    sigma, dl, dr = oracle.mwm(ip, ix, dv)
    assert list(sigma) == list(perm)
    np.testing.assert_allclose(np.abs(dl * A[np.arange(n), perm] * dr[perm]), 1.0, rtol=1e-13)
    B = _mwm_random(20, 9)
    B[:, 3] = 0.0
    ipb, ixb, dvb = dense_to_csr(B)
    with pytest.raises(oracle.OracleError):
        oracle.mwm(ipb, ixb, dvb)


# ---------------- aggregation counts (Sec. 3.5) pinned by a hand trace ----------------
def _trace_matrix(g):
    n = g["n"]
    L0 = np.eye(n)
    U0 = np.eye(n)
    for i, k, v in g["L0"]:
        L0[i, k] = v
    for k, j, v in g["U0"]:
        U0[k, j] = v
    return L0 @ np.diag(g["pivots"]) @ U0


def test_aggregation_counts_hand_trace():
    """tests/golden/aggregate_trace.json: a 7x7 A = L0 P0 U0 with scalar initial blocks whose
    factor patterns are known by construction; the counts r,s,t,r',s',t',u,v of every merge
    test were traced by hand from those patterns.  The trace's merge
    decisions, and hence the final partition [1,1,5], differ from what a sum instead of a
    union for u or v, counting the rows of L_{k-1} inside block k in u, dropping r or t'
    from mu, or strict inequalities would give (the mutants listed in the file)."""
    g = json.load(open(os.path.join(GOLD, "aggregate_trace.json")))
    A = _trace_matrix(g)
    f = fac(A, g["block_sizes"], g["tau"])            # no aggregation: the patterns of L0, U0
    for K in range(g["n"]):
        _, _, rows, _, cols, _, _ = f.block(K)
        assert list(rows) == g["L_rows_per_block"][K] and list(cols) == g["U_cols_per_block"][K]
    for st in g["steps"]:
        p, q = st["p"], st["q"]
        assert st["r"] + st["s"] + st["t"] >= st["u"] >= max(st["s"], st["t"])
        assert st["u"] == len(st["u_rows"]) and st["v"] == len(st["v_cols"])
        mu = p * (p + st["r"] + st["s"] + st["r2"] + st["s2"]) + q * (q + st["t"] + st["t2"])
        nu = (p + q) * (p + q + st["u"] + st["v"])
        assert (mu, nu) == (st["mu"], st["nu"])
        assert oracle.aggregate_test(p, q, st["r"], st["s"], st["t"], st["r2"], st["s2"], st["t2"],
                                     st["u"], st["v"]) == st["merge"]
    h = fac(A, g["block_sizes"], g["tau"], agg=True)
    assert list(np.diff(h.bstart)) == g["final_block_sizes"] and h.n_merges == g["n_merges"]
    # max_block = 3 (R9) stops the run at p + q = 4 (step k = 5); block 5 alone then meets
    # block 6: p = q = 1, r = 1 (row 6 of L_5), s = t = r' = s' = t' = u = v = 0, mu = 3,
    # nu = 4 <= mu + 2(p+q) = 7 -> merge: partition [1, 1, 3, 2]
    m = fac(A, g["block_sizes"], g["tau"], agg=True, max_block=3)
    assert list(np.diff(m.bstart)) == [1, 1, 3, 2] and m.n_merges == 3
    # the merged factors represent the same operator
    L, P, U = dense_LPU(h, g["n"])
    np.testing.assert_allclose(L @ P @ U, A, atol=1e-13 * np.abs(A).max())


def test_perturbation_ill_conditioned_nonsingular_block():
    """Sec. 3.6: a pivot block that is nonsingular but ill-conditioned is
    perturbed.  P = [[1, 1], [1, 1 + 1e-13]] has kappa_1 = ||P||_1 ||P^{-1}||_1 ~ 4e13 >
    cond_max = 1e12 (R19), so every column, then every row, gets its largest entry (the
    diagonal, preferred when 2|d_jj| >= |d_kj|) moved to d (1 + rho delta) + sign(d) tau_p
    alpha; with cond_max = 1e20 the same block is inverted unperturbed."""
    eps = 1e-13
    A = np.array([[1.0, 1.0], [1.0, 1.0 + eps]])
    ip, ix, dv = dense_to_csr(A)
    tp, rho, _ = PT
    f = oracle.factor(ip, ix, dv, [2], 0.0, aggregate=False, perturb=PT)
    assert f.n_perturbed == 1
    alpha = 1.0 + eps
    Pp = A.copy()
    for j in range(2):                                  # columns: delta_j = max_i |p_ij|
        d = np.abs(Pp[:, j]).max()
        Pp[j, j] = Pp[j, j] * (1 + rho * d) + tp * alpha
    for i in range(2):                                  # then rows
        d = np.abs(Pp[i, :]).max()
        Pp[i, i] = Pp[i, i] * (1 + rho * d) + tp * alpha
    np.testing.assert_allclose(f.block(0)[6], np.linalg.inv(Pp), rtol=1e-12)
    kappa = np.abs(Pp).sum(0).max() * np.abs(np.linalg.inv(Pp)).sum(0).max()
    assert kappa < 1e12
    g = oracle.factor(ip, ix, dv, [2], 0.0, aggregate=False, perturb=(PT[0], PT[1], 1e20))
    assert g.n_perturbed == 0
    np.testing.assert_allclose(g.block(0)[6], np.linalg.inv(A), rtol=1e-3)
