"""Device ILU(1,tau) initial blocking (bilu_ilu1_blocks, Sec. 3.4) vs the oracle's estimate.

The partition is integer output decided by fp64 comparisons that both sides evaluate with the
same products (R20), so the bar is bit-exact equality of the block sizes.  Cases:
the hand-traced pins, ragged sizes around the chain chunk (256), the warp-table and the
global-table (overflow) paths, max_size in {1, 3, 8, 128}, tau in {0, large}, full-size c2, c3
and c5, and factorizations that start from the estimated partition.
"""
import numpy as np
import pytest
import scipy.sparse as sp

import oracle
from inputs.configs import config1, config2, config3, config4, config5, dense_to_csr, random_dd
from tests.parity import compare_factors, oracle_replay, overrides_from_near

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_1908_10169_b200.build import build
    build()


def both(ip, ix, dv, tau, max_size, perm=None):
    from paper_1908_10169_b200 import ilu1_blocks
    g, launches = ilu1_blocks(ip, ix, dv, tau, max_size, perm=perm)
    if perm is not None:
        ip, ix, dv = oracle.permute_csr(ip, ix, dv, perm)
    o = oracle.ilu1_blocks(ip, ix, dv, tau, max_size)
    assert launches > 0
    return g, o


def assert_same(g, o, n):
    assert g.sum() == n
    assert len(g) == len(o) and np.array_equal(g, o), (len(g), len(o), np.nonzero(g[: min(len(g), len(o))] != o[: min(len(g), len(o))])[0][:5])


def test_identity_and_tridiagonal_pins():
    n = 23
    ip, ix, dv = np.arange(n + 1), np.arange(n), np.ones(n)
    g, o = both(ip, ix, dv, 1e-2, 128)
    assert list(g) == [5, 5, 5, 5, 3]
    T = sp.diags([-np.ones(7), 4 * np.ones(8), -np.ones(7)], [-1, 0, 1]).tocsr()
    g, o = both(T.indptr, T.indices, T.data, 0.1, 8)
    assert list(g) == [5, 3]


def test_hand_4x4():
    A = np.array([[2, 1, 0, 1], [0, 4, 0, 3], [5, 0, 1, 0], [0, 0.1, 0, 8.0]])
    ip, ix, dv = dense_to_csr(A)
    for tau, ms, want in ((0.5, 8, [4]), (0.5, 2, [2, 2])):
        g, o = both(ip, ix, dv, tau, ms)
        assert list(g) == want == list(o)


@pytest.mark.parametrize("n", [1, 2, 255, 256, 257, 1000, 5000])
@pytest.mark.parametrize("max_size", [1, 3, 8, 128])
def test_ragged_random(n, max_size):
    A = sp.random(n, n, density=min(1.0, 6.0 / n), random_state=n, format="csr") + sp.eye(n) * 3
    A = A.tocsr()
    A.sum_duplicates()
    A.sort_indices()
    for tau in (0.0, 1e-2, 0.3):
        g, o = both(A.indptr, A.indices, A.data, tau, max_size)
        assert_same(g, o, n)
        assert g.max() <= max_size


def test_missing_diagonal_and_empty_rows():
    """a_kk absent counts as 0 (R20): every nonzero passes the direct test."""
    rng = np.random.default_rng(5)
    n = 600
    A = sp.random(n, n, density=0.01, random_state=5, format="lil")
    for k in rng.choice(n, 100, replace=False):
        A[k, k] = 0
        A[k, :] = 0                     # some empty rows
    A = A.tocsr()
    A.eliminate_zeros()
    A.sort_indices()
    g, o = both(A.indptr, A.indices, A.data, 1e-2, 8)
    assert_same(g, o, n)


def test_overflow_tables_block_matrix():
    """Dense block rows (c4 recipe, 150 blocks of 16..64): candidate bounds exceed both
    shared-memory tables, so every step runs on the global-table kernels."""
    P = config4(nblocks=150)
    for ms in (8, 64):
        g, o = both(P.indptr, P.indices, P.data, P.tau, ms)
        assert_same(g, o, P.n)


def test_perm_applied():
    A = random_dd(700, 0.01, 9, dominance=1.2)
    ip, ix, dv = dense_to_csr(A)
    perm = np.random.default_rng(9).permutation(700)
    g, o = both(ip, ix, dv, 1e-2, 8, perm=perm)
    assert_same(g, o, 700)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c5"])
def test_full_configs(name):
    P = {"c1": config1, "c2": config2, "c3": config3, "c5": config5}[name]()
    g, o = both(P.indptr, P.indices, P.data, P.tau, 8, perm=P.perm)
    assert_same(g, o, P.n)
    if name == "c3":
        assert np.bincount(g)[3] > 0.8 * len(g)     # recovers the nodal 3x3 blocks


def test_bad_arguments():
    from paper_1908_10169_b200 import BiluError, ilu1_blocks
    ip, ix, dv = np.arange(4), np.arange(3), np.ones(3)
    with pytest.raises(BiluError):
        ilu1_blocks(ip, ix, dv, 1e-2, 0)
    with pytest.raises(BiluError):
        ilu1_blocks(ip, ix, dv, -1.0, 8)
    with pytest.raises(BiluError):
        ilu1_blocks(ip, ix, dv, 1e-2, 8, perm=[0, 0, 1])
    with pytest.raises(BiluError):
        ilu1_blocks(np.array([0, 2, 2, 3]), np.array([1, 0, 2]), dv, 1e-2, 8)   # row 0 unsorted


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_factor_from_estimated_blocks(name):
    """The estimate feeds bilu_analyze: the factorization from it matches the oracle's."""
    from paper_1908_10169_b200 import BILU, ilu1_blocks
    P = config1() if name == "c1" else config2()
    bs, _ = ilu1_blocks(P.indptr, P.indices, P.data, P.tau, 8, perm=P.perm)
    g = BILU(P.indptr, P.indices, P.data, bs, perm=P.perm)
    st = g.factor(P.tau)
    gf = g.export()
    pip, pix, pdv = oracle.permute_csr(P.indptr, P.indices, P.data, P.perm) if P.perm is not None else (
        P.indptr, P.indices, P.data)
    of = oracle_replay(pip, pix, pdv, bs, P.tau, aggregate=True, overrides=overrides_from_near(gf.near))
    assert st["n_blocks_init"] == len(bs)
    r = compare_factors(gf, of, 1e-10)
    assert not r["problems"], r["problems"][:5]


# ------------------------------------------------------------ cosine-based blocking (Sec. 3.2)
def cos_both(ip, ix, tau=0.8, max_size=128):
    from paper_1908_10169_b200 import cosine_blocks
    q, s, nl = cosine_blocks(ip, ix, tau, max_size)
    oq, os_ = oracle.cosine_blocks(ip, ix, tau, max_size)
    assert nl > 0
    assert np.array_equal(np.sort(q), np.arange(len(ip) - 1))
    assert len(s) == len(os_) and np.array_equal(s, os_), (len(s), len(os_))
    assert np.array_equal(q, oq)
    return q, s


def _rows_csr(rows, n):
    ip = np.zeros(n + 1, dtype=np.int64)
    for i, r in enumerate(rows):
        ip[i + 1] = ip[i] + len(r)
    return ip, np.concatenate([np.asarray(sorted(set(r)), dtype=np.int32) for r in rows])


def test_cosine_pins():
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cosine_hand_6x6.json")))
    ip, ix = _rows_csr(g["rows"], 6)
    for c in g["cases"]:
        q, s = cos_both(ip, ix, c["tau"], c["max_size"])
        assert list(q) == c["q"] and list(s) == c["sizes"]
    n = 10
    ip, ix = _rows_csr([list(range(n))] + [[0, i] for i in range(1, n)], n)
    q, s = cos_both(ip, ix, 0.2)
    assert list(s) == [1] * n
    ip, ix = _rows_csr([list(range(n))] * n, n)
    q, s = cos_both(ip, ix, 0.8, 4)
    assert list(s) == [4, 4, 2]


def _dup_pattern(n, seed, deg=6, dup=0.6, noise=0.3):
    """rows copied (with noise) from a few earlier rows: groups of similar rows"""
    rng = np.random.default_rng(seed)
    rows = []
    for i in range(n):
        if i > 0 and rng.random() < dup:
            src = rows[max(0, i - int(rng.integers(1, 4)))]
            r = [c for c in src if rng.random() > noise * 0.3]
            if rng.random() < noise:
                r.append(int(rng.integers(0, n)))
        else:
            r = list(rng.integers(0, n, size=int(rng.integers(1, deg + 1))))
        rows.append(sorted(set(r + [i])))
    return _rows_csr(rows, n)


@pytest.mark.parametrize("n", [1, 2, 255, 257, 1000, 5000])
@pytest.mark.parametrize("max_size", [1, 2, 4, 128])
def test_cosine_ragged_random(n, max_size):
    ip, ix = _dup_pattern(n, n + max_size)
    for tau in (0.3, 0.5, 0.8):
        cos_both(ip, ix, tau, max_size)


def test_cosine_band_long_chain():
    """Band of half-width 6: consecutive rows share 12 of 13 columns, so the greedy's dependency
    chain runs through the whole matrix (exercises the in-order sweep after the rounds stall)."""
    n, w = 3000, 6
    rows = [list(range(max(0, i - w), min(n, i + w + 1))) for i in range(n)]
    ip, ix = _rows_csr(rows, n)
    for ms in (3, 128):
        cos_both(ip, ix, 0.8, ms)


def test_cosine_overflow_block_rows():
    P = config4(nblocks=150)
    q, s = cos_both(P.indptr, P.indices, 0.8, 128)


@pytest.mark.parametrize("name", ["c2", "c3", "c5"])
def test_cosine_full_configs(name):
    P = {"c2": config2, "c3": config3, "c5": config5}[name]()
    q, s = cos_both(P.indptr, P.indices, 0.8, 128)
    if name == "c3":
        assert len(s) == P.n // 3 and set(s) == {3}      # the nodal 3x3 blocks (PAPER.md Ex. 3.2's role)


def test_cosine_bad_arguments():
    from paper_1908_10169_b200 import BiluError, cosine_blocks
    ip, ix = np.arange(4), np.arange(3)
    with pytest.raises(BiluError):
        cosine_blocks(ip, ix, 1.5, 8)
    with pytest.raises(BiluError):
        cosine_blocks(ip, ix, 0.8, 0)
    with pytest.raises(BiluError):
        cosine_blocks(np.array([0, 2, 2, 3]), np.array([1, 0, 2]), 0.8, 8)


def test_factor_from_cosine_blocks():
    """Q and the groups feed bilu_analyze (perm = Q): parity with the oracle on the same input."""
    from paper_1908_10169_b200 import BILU, cosine_blocks
    P = config3(N=10)
    q, s, _ = cosine_blocks(P.indptr, P.indices, 0.8, 128)
    g = BILU(P.indptr, P.indices, P.data, s, perm=q)
    st = g.factor(P.tau)
    gf = g.export()
    pip, pix, pdv = oracle.permute_csr(P.indptr, P.indices, P.data, q)
    of = oracle_replay(pip, pix, pdv, s, P.tau, aggregate=True, overrides=overrides_from_near(gf.near))
    r = compare_factors(gf, of, 1e-10)
    assert not r["problems"], r["problems"][:5]
