"""CUDA path (through the C-ABI) vs the CPU oracle on the same seeded inputs.

Bar (BASELINE north_star):
  - kept/dropped pattern identical after replaying the GPU's near-threshold
    decisions (|max/tau - 1| <= 1e-8) in the oracle,
  - factor values within 1e-10 normwise per L row / Ũ column / D block,
  - preconditioned GMRES(30) iteration counts to 1e-8 within +-1.
"""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from harness.gmres import gmres
from inputs.configs import config1, config2, config3, dense_to_csr, random_dd
from tests.parity import compare_factors, dense_LPU, oracle_replay, overrides_from_near

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_1908_10169_b200.build import build
    build()


def run_pair(ip, ix, dv, bs, tau, agg=True, perm=None, max_block=128, **kw):
    from paper_1908_10169_b200 import BILU
    g = BILU(ip, ix, dv, bs, perm=perm, aggregate=int(agg), max_block=max_block, **kw)
    st = g.factor(tau)
    gf = g.export()
    if perm is not None:
        pip, pix, pdv = oracle.permute_csr(ip, ix, dv, perm)
    else:
        pip, pix, pdv = ip, ix, dv
    of = oracle_replay(pip, pix, pdv, bs, tau, aggregate=agg, max_block=max_block,
                       overrides=overrides_from_near(gf.near))
    return g, st, gf, of


def assert_parity(gf, of, tol=TOL):
    r = compare_factors(gf, of, tol)
    assert not r["problems"], r["problems"][:5]
    return r


def partition(n, rng, maxb):
    out = []
    while sum(out) < n:
        out.append(int(min(rng.integers(1, maxb + 1), n - sum(out))))
    return np.array(out)


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("tau", [0.0, 1e-3, 3e-2])
@pytest.mark.parametrize("agg", [False, True])
def test_random_small(seed, tau, agg):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(30, 260))
    A = random_dd(n, float(rng.uniform(0.02, 0.2)), 500 + seed, dominance=float(rng.uniform(1.05, 2.0)))
    ip, ix, dv = dense_to_csr(A)
    bs = partition(n, rng, int(rng.integers(1, 17)))
    g, st, gf, of = run_pair(ip, ix, dv, bs, tau, agg)
    assert_parity(gf, of)
    if agg:
        assert st["n_blocks_final"] == of.nblk
    g.close()


def test_edge_single_unknown():
    g, st, gf, of = run_pair([0, 1], [0], [3.0], [1], 1e-2)
    assert_parity(gf, of)
    np.testing.assert_allclose(gf.Dv, [1 / 3.0])


def test_edge_one_block_of_max_size():
    A = random_dd(128, 0.3, 1)
    ip, ix, dv = dense_to_csr(A)
    g, st, gf, of = run_pair(ip, ix, dv, [128], 1e-2)
    assert_parity(gf, of)
    np.testing.assert_allclose(gf.block(0)[6], np.linalg.inv(A), rtol=1e-9, atol=1e-13)


def test_edge_scalar_blocks_and_large_blocks_mixed():
    A = random_dd(300, 0.05, 2, dominance=1.2)
    ip, ix, dv = dense_to_csr(A)
    bs = np.array([1] * 50 + [64, 64] + [2] * 61)
    assert bs.sum() == 300
    g, st, gf, of = run_pair(ip, ix, dv, bs, 1e-3)
    assert_parity(gf, of)


def test_edge_tau_infinite_block_jacobi():
    A = random_dd(100, 0.1, 3)
    ip, ix, dv = dense_to_csr(A)
    g, st, gf, of = run_pair(ip, ix, dv, [10] * 10, 1e300, agg=False)
    assert len(gf.Li) == 0 and len(gf.Ui) == 0
    assert_parity(gf, of)


def test_edge_identity():
    n = 64
    ip = np.arange(n + 1)
    g, st, gf, of = run_pair(ip, np.arange(n), np.ones(n), [8] * 8, 1e-2, agg=True)
    assert_parity(gf, of)


def test_breakdown_reports_block():
    from paper_1908_10169_b200 import BILU, BiluError
    A = np.array([[4.0, 1, 0, 0], [1, 4, 0, 0], [0, 0, 1, 1], [0, 0, 1, 1]])
    ip, ix, dv = dense_to_csr(A)
    g = BILU(ip, ix, dv, [2, 2], aggregate=0)
    with pytest.raises(BiluError) as ei:
        g.factor(0.0)
    assert ei.value.status == 2 and ei.value.breakdown_block == 1


def test_near_threshold_decision_is_logged_and_replayed():
    """l_21 = 0.02 / 2 = 0.01 = tau exactly: a tie (dropped, R2) with margin 0."""
    A = np.array([[2.0, 0.0], [0.02, 1.0]])
    ip, ix, dv = dense_to_csr(A)
    g, st, gf, of = run_pair(ip, ix, dv, [1, 1], 0.01, agg=False)
    assert st["n_near"] == 1 and gf.near.shape == (1, 4)
    assert tuple(gf.near[0]) == (0, 0, 1, 0)
    assert_parity(gf, of)


def test_refactor_new_values_and_tau():
    A = random_dd(150, 0.08, 4)
    ip, ix, dv = dense_to_csr(A)
    bs = [5] * 30
    from paper_1908_10169_b200 import BILU
    g = BILU(ip, ix, dv, bs)
    g.factor(1e-2)
    dv2 = dv * np.random.default_rng(0).uniform(0.9, 1.1, len(dv))
    g.set_values(dv2)
    g.factor(3e-3)
    gf = g.export()
    of = oracle_replay(ip, ix, dv2, bs, 3e-3, overrides=overrides_from_near(gf.near))
    assert_parity(gf, of)


def test_apply_matches_oracle_apply():
    import torch
    A = random_dd(200, 0.05, 5)
    ip, ix, dv = dense_to_csr(A)
    rng = np.random.default_rng(0)
    perm = rng.permutation(200)
    g, st, gf, of = run_pair(ip, ix, dv, [4] * 50, 1e-2, perm=perm)
    x = rng.standard_normal(200)
    y = g.apply_tensor(torch.tensor(x, device="cuda")).cpu().numpy()
    yo_p = oracle.apply(of, x[perm])
    yo = np.empty(200); yo[perm] = yo_p
    np.testing.assert_allclose(y, yo, rtol=1e-11, atol=1e-13 * np.abs(yo).max())
    # and it inverts L P U in the original ordering
    L, P, U = dense_LPU(of, 200)
    M = np.zeros((200, 200)); M[np.ix_(perm, perm)] = L @ P @ U
    np.testing.assert_allclose(M @ y, x, atol=1e-10 * np.abs(x).max())


def _gmres_counts(prob, g, of):
    import torch
    A = sp.csr_matrix((prob.data, prob.indices, prob.indptr), shape=(prob.n, prob.n))
    perm = prob.perm
    b = np.ones(prob.n)

    def m_gpu(v):
        return g.apply_tensor(torch.tensor(v, device="cuda")).cpu().numpy()

    def m_orc(v):
        y = oracle.apply(of, v[perm])
        out = np.empty_like(y); out[perm] = y
        return out
    _, it_g, ok_g, _ = gmres(A.dot, b, precond=m_gpu, restart=30, tol=1e-8)
    _, it_o, ok_o, _ = gmres(A.dot, b, precond=m_orc, restart=30, tol=1e-8)
    return it_g, ok_g, it_o, ok_o


def test_c1_full_parity_and_gmres():
    P = config1()
    g, st, gf, of = run_pair(P.indptr, P.indices, P.data, P.block_sizes, P.tau, True, P.perm)
    assert_parity(gf, of)
    it_g, ok_g, it_o, ok_o = _gmres_counts(P, g, of)
    assert ok_g and ok_o and abs(it_g - it_o) <= 1


def test_c2_reduced_parity():
    P = config2(N=24, leaf=128)
    g, st, gf, of = run_pair(P.indptr, P.indices, P.data, P.block_sizes, P.tau, True, P.perm)
    assert_parity(gf, of)


def test_c2_full_parity_and_gmres():
    """BASELINE configs[1] at full size, in the bench.py launch configuration."""
    P = config2()
    g, st, gf, of = run_pair(P.indptr, P.indices, P.data, P.block_sizes, P.tau, True, P.perm)
    assert st["n_blocks_init"] == 33111
    assert_parity(gf, of)
    assert st["n_merges"] == of.n_merges
    it_g, ok_g, it_o, ok_o = _gmres_counts(P, g, of)
    assert ok_g and ok_o and abs(it_g - it_o) <= 1


def test_c3_reduced_parity_nodal_blocks():
    P = config3(N=10)
    g, st, gf, of = run_pair(P.indptr, P.indices, P.data, P.block_sizes, P.tau, True, P.perm)
    assert_parity(gf, of)


def test_small_max_block_merges():
    A = random_dd(400, 0.02, 6, dominance=1.3)
    ip, ix, dv = dense_to_csr(A)
    g, st, gf, of = run_pair(ip, ix, dv, [2] * 200, 1e-3, True, max_block=16)
    assert_parity(gf, of)
    assert np.diff(gf.bstart).max() <= 16


def test_c4_reduced_parity_wide_blocks():
    """BASELINE configs[3] recipe at reduced size: dense blocks of 16-64 (the DMMA
    Schur-update and scaling paths), random block pattern, tau = 1e-4."""
    from inputs.configs import config4
    P = config4(nblocks=80, per_row=4)
    g, st, gf, of = run_pair(P.indptr, P.indices, P.data, P.block_sizes, P.tau, True, P.perm)
    assert_parity(gf, of)
    assert st["n_blocks_final"] == of.nblk


def test_c4_reduced_gmres():
    from inputs.configs import config4
    P = config4(nblocks=60, per_row=3)
    g, st, gf, of = run_pair(P.indptr, P.indices, P.data, P.block_sizes, P.tau, True, P.perm)
    assert_parity(gf, of)
    it_g, ok_g, it_o, ok_o = _gmres_counts(P, g, of)
    assert ok_g and ok_o and abs(it_g - it_o) <= 1


def test_c5_reduced_parity_and_gmres():
    """BASELINE configs[4] recipe at reduced size (27-pt, lognormal kappa, Pe 50, ND)."""
    from inputs.configs import config5
    P = config5(N=20, top_levels=1)
    g, st, gf, of = run_pair(P.indptr, P.indices, P.data, P.block_sizes, P.tau, True, P.perm)
    assert_parity(gf, of)
    assert st["n_merges"] == of.n_merges
    it_g, ok_g, it_o, ok_o = _gmres_counts(P, g, of)
    assert ok_g and ok_o and abs(it_g - it_o) <= 1


@pytest.mark.parametrize("zone", ["none", "partial", "full"])
@pytest.mark.parametrize("cfg", ["c2r", "c5r"])
def test_zone_coverage_parity(cfg, zone):
    """Dense zone: the factors must not depend on how much of the block
    elimination tree keeps pushed per-block panels -- none (contributor lists only), a
    budget-limited top of the tree, or every block (panels over each block's etree path)."""
    from inputs.configs import config5
    P = config2(N=24, leaf=128) if cfg == "c2r" else config5(N=20, top_levels=1)
    nb = len(P.block_sizes)
    zb = {"none": -1, "partial": 6 << 20, "full": 0}[zone]
    g, st, gf, of = run_pair(P.indptr, P.indices, P.data, P.block_sizes, P.tau, True, P.perm, zone_bytes=zb)
    assert_parity(gf, of)
    assert st["n_merges"] == of.n_merges
    if zone == "none":
        assert st["zone_blocks"] == 0
    elif zone == "full":
        assert st["zone_blocks"] == nb and st["zone_unknowns"] == P.n
    else:
        assert 2 <= st["zone_blocks"] < nb
    # refactor with new values: the zone buffers are all zero again after a factorization
    st2 = g.factor(P.tau)
    gf2 = g.export()
    assert st2["n_blocks_final"] == st["n_blocks_final"]
    assert np.array_equal(np.asarray(gf2.Lv), np.asarray(gf.Lv)) or compare_factors(gf2, of, TOL)["problems"] == []


@pytest.mark.parametrize("agg", [False, True])
def test_edge_wide_key_range_posmap(agg):
    """Candidate key ranges wider than 2^18 unknowns (the per-CTA pos-map path of a-3
    instead of the shared-memory bitmap): n = 300,000 with couplings between the
    first and the last 4000 unknowns."""
    from inputs.configs import wide_range_matrix
    ip, ix, dv = wide_range_matrix()
    bs = np.full(300_000 // 8, 8)
    g, st, gf, of = run_pair(ip, ix, dv, bs, 1e-3, agg)
    assert_parity(gf, of)


@pytest.mark.parametrize("zone_gib", [None, 120])
def test_c3_full_parity(zone_gib):
    """BASELINE configs[2] at full size (48^3 nodes x 3 dof, n = 331,776, 25.8M nnz), with the
    library's default dense-zone budget and with the one bench.py passes for c3 (ZONE_GIB)."""
    import torch
    opts = {}
    if zone_gib is not None:
        if torch.cuda.mem_get_info()[0] < (zone_gib + 40) << 30:
            pytest.skip("needs %d GiB of free HBM" % (zone_gib + 40))
        opts["zone_bytes"] = zone_gib << 30
    P = config3()
    g, st, gf, of = run_pair(P.indptr, P.indices, P.data, P.block_sizes, P.tau, True, P.perm, **opts)
    assert st["n_blocks_init"] == 110592
    if zone_gib is not None:
        assert st["zone_blocks"] > 60000
    assert_parity(gf, of)
    assert st["n_merges"] == of.n_merges


def test_c5_full_parity_and_gmres():
    """BASELINE configs[4] at full size (27-pt 128^3, n = 2,097,152, 55.7M nnz; the
    oracle takes a few minutes single-threaded)."""
    from inputs.configs import config5
    P = config5()
    g, st, gf, of = run_pair(P.indptr, P.indices, P.data, P.block_sizes, P.tau, True, P.perm)
    assert P.nnz == 55742968
    assert_parity(gf, of)
    assert st["n_merges"] == of.n_merges
    it_g, ok_g, it_o, ok_o = _gmres_counts(P, g, of)
    assert ok_g and ok_o and abs(it_g - it_o) <= 1


def test_c4_full_parity():
    """BASELINE configs[3] at full size (20,000 dense blocks of 16-64, n = 802,382, 422M nnz),
    in the bench.py launch configuration; the oracle takes a few minutes single-threaded."""
    from inputs.configs import config4
    P = config4()
    assert P.nnz == 422328517
    g, st, gf, of = run_pair(P.indptr, P.indices, P.data, P.block_sizes, P.tau, True, P.perm)
    assert st["n_blocks_init"] == 20000 and st["n_blocks_final"] == of.nblk
    r = assert_parity(gf, of)
    assert r["max_rel"] <= TOL


def test_c4_2000_blocks_parity():
    """BASELINE configs[3] recipe with 2,000 of its 20,000 blocks (n ~ 80k, nnz ~ 43M): the
    split wide-block path (contributor-range GEMM parts, scaling parts) at scale."""
    from inputs.configs import config4
    P = config4(nblocks=2000)
    g, st, gf, of = run_pair(P.indptr, P.indices, P.data, P.block_sizes, P.tau, True, P.perm)
    assert_parity(gf, of)
    assert st["n_blocks_final"] == of.nblk


# ---------------- Sec. 3.6 perturbation (R19) ----------------
PT = (1e-2, 1e-1, 1e12)


def run_pair_pt(ip, ix, dv, bs, tau, agg=True):
    from paper_1908_10169_b200 import BILU
    g = BILU(ip, ix, dv, bs, aggregate=int(agg), perturb=1, perturb_tau=PT[0], perturb_rho=PT[1],
             cond_max=PT[2])
    st = g.factor(tau)
    gf = g.export()
    of = oracle_replay(ip, ix, dv, bs, tau, aggregate=agg, perturb=PT, overrides=overrides_from_near(gf.near))
    return g, st, gf, of


def test_perturbation_zero_column_block():
    A = np.array([[2.0, 0.0, 0.5], [1.0, 0.0, 0.0], [0.0, 0.0, 4.0]])
    ip, ix, dv = dense_to_csr(A)
    g, st, gf, of = run_pair_pt(ip, ix, dv, [2, 1], 0.0, agg=False)
    assert st["n_perturbed"] == 1 == of.n_perturbed
    assert_parity(gf, of)


def _singular_blocks_matrix(n, nsing, seed, bsz=2):
    rng = np.random.default_rng(seed)
    A = random_dd(n, 0.08, seed, dominance=1.6)
    starts = rng.choice(np.arange(1, n // bsz - 1), nsing, replace=False) * bsz
    for s0 in starts:
        A[s0:s0 + bsz, :] = 0.0
        A[:, s0:s0 + bsz] = 0.0
        A[s0:s0 + bsz, s0:s0 + bsz] = rng.uniform(0.5, 1.5) * np.ones((bsz, bsz))   # rank 1, decoupled
    return A


@pytest.mark.parametrize("agg", [False, True])
def test_perturbation_singular_blocks_match_oracle(agg):
    A = _singular_blocks_matrix(160, 6, 21)
    ip, ix, dv = dense_to_csr(A)
    bs = [2] * 80
    g, st, gf, of = run_pair_pt(ip, ix, dv, bs, 1e-3, agg)
    assert st["n_perturbed"] == of.n_perturbed >= 6
    assert_parity(gf, of)


def test_perturbation_wide_singular_block():
    """A rank-deficient 24 x 24 pivot block (multi-warp Gauss-Jordan path)."""
    A = _singular_blocks_matrix(240, 2, 23, bsz=24)
    ip, ix, dv = dense_to_csr(A)
    bs = [24] * 10
    g, st, gf, of = run_pair_pt(ip, ix, dv, bs, 1e-3, False)
    assert st["n_perturbed"] == of.n_perturbed >= 2
    assert_parity(gf, of)


def test_perturbation_inactive_on_c2_reduced():
    P = config2(N=16, leaf=64)
    pip, pix, pdv = oracle.permute_csr(P.indptr, P.indices, P.data, P.perm)
    g, st, gf, of = run_pair_pt(pip, pix, pdv, P.block_sizes, P.tau, True)
    assert st["n_perturbed"] == 0 == of.n_perturbed
    assert_parity(gf, of)


# ---------------- device GMRES (bilu_gmres) ----------------
@pytest.mark.parametrize("cfg", ["c1", "c2s", "c5s"])
def test_device_gmres_matches_host_gmres(cfg):
    """bilu_gmres (device vectors, MGS coefficients on the device) against the host
    harness GMRES(30) driven by the same preconditioner: iteration counts within +-1
    (BASELINE), both converged to 1e-8 on the true residual, the same solution."""
    import torch
    from inputs.configs import config1, config5
    from paper_1908_10169_b200 import BILU
    P = {"c1": lambda: config1(), "c2s": lambda: config2(N=24, leaf=128), "c5s": lambda: config5(N=20, top_levels=1)}[cfg]()
    g = BILU(P.indptr, P.indices, P.data, P.block_sizes, perm=P.perm)
    g.factor(P.tau)
    b = torch.ones(P.n, dtype=torch.float64, device="cuda")
    x, st = g.gmres(b, restart=30, tol=1e-8)
    assert st["converged"] == 1 and st["rel_residual"] <= 1e-8
    A = sp.csr_matrix((P.data, P.indices, P.indptr), shape=(P.n, P.n))
    xs = x.cpu().numpy()
    assert np.linalg.norm(np.ones(P.n) - A @ xs) <= 1e-8 * np.sqrt(P.n) * 1.0000001

    def m_gpu(v):
        return g.apply_tensor(torch.tensor(v, device="cuda")).cpu().numpy()
    xh, it_h, ok_h, _ = gmres(A.dot, np.ones(P.n), precond=m_gpu, restart=30, tol=1e-8)
    assert ok_h and abs(st["iterations"] - it_h) <= 1
    assert np.abs(xs - xh).max() <= 1e-6 * np.abs(xh).max()


@pytest.mark.parametrize("agg", [False, True])
def test_apply_heavy_blocks_split_over_warps(agg):
    """Blocks with wide panels (b >= 32, >= 16K panel entries) are applied by several warps of
    a CTA (forward: 64-row parts pushing into w; backward: 128-column parts accumulating into
    the owner's z).  Block 0 (b=64) couples densely to all 2000 later rows/columns, a middle
    block (b=48) to everything after it; the apply must match the oracle's (L P U)^{-1} x."""
    import torch
    rng = np.random.default_rng(17)
    n0, nmid, nrest = 64, 48, 2000
    n = n0 + nrest
    A = sp.random(n, n, density=3.0 / n, random_state=17, format="lil")
    A[:n0, n0:] = rng.uniform(-0.1, 0.1, (n0, nrest))
    A[n0:, :n0] = rng.uniform(-0.1, 0.1, (nrest, n0))
    m0 = n0 + 1000
    A[m0:m0 + nmid, m0 + nmid:] = rng.uniform(-0.1, 0.1, (nmid, n - m0 - nmid))
    A[m0 + nmid:, m0:m0 + nmid] = rng.uniform(-0.1, 0.1, (n - m0 - nmid, nmid))
    A = A.tocsr()
    A.setdiag(0.0)
    A.eliminate_zeros()
    A = (A + sp.diags(1.5 * np.asarray(abs(A).sum(axis=1)).ravel() + 1.0)).tocsr()
    A.sort_indices()
    bs = [n0] + [8] * (1000 // 8) + [nmid] + [8] * ((nrest - 1000 - nmid) // 8)
    assert sum(bs) == n
    g, st, gf, of = run_pair(A.indptr, A.indices, A.data, bs, 1e-5, agg)
    Lm = np.diff(gf.Lp)
    b = np.diff(gf.bstart)
    assert ((b >= 32) & (Lm * b >= 16384)).sum() >= 2          # the split paths are exercised
    for x in (np.ones(n), rng.standard_normal(n)):
        y = g.apply_tensor(torch.tensor(x, device="cuda")).cpu().numpy()
        yo = oracle.apply(of, x)
        np.testing.assert_allclose(y, yo, rtol=1e-11, atol=1e-12 * np.abs(yo).max())


@pytest.mark.parametrize("cfg", ["c2r", "c4r", "rand"])
def test_flop_count_matches_oracle_without_aggregation(cfg):
    """The GFLOP/s numerator (bilu_factor_stats.flops) equals the oracle's count
    of the same executed structure: with aggregate = False both count 2 b_J m c per
    contributor side and 2b^3 + 2b^2(|R_K| + |C_K|) per block over identical candidate
    sets (integer-valued sums, exact in fp64)."""
    from inputs.configs import config4
    if cfg == "c2r":
        P = config2(N=24, leaf=128)
        args = (P.indptr, P.indices, P.data, P.block_sizes, P.tau, False, P.perm)
    elif cfg == "c4r":
        P = config4(nblocks=80, per_row=4)
        args = (P.indptr, P.indices, P.data, P.block_sizes, P.tau, False, P.perm)
    else:
        A = random_dd(300, 0.05, 9, dominance=1.3)
        ip, ix, dv = dense_to_csr(A)
        args = (ip, ix, dv, partition(300, np.random.default_rng(9), 12), 1e-3, False)
    g, st, gf, of = run_pair(*args)
    assert_parity(gf, of)
    assert st["flops"] == of.flops, (st["flops"], of.flops)
    g.close()
