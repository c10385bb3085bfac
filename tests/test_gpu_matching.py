"""Device matching + scaling of Sec. 3.1 (bilu_mwm; R22) vs the
oracle's Hungarian method (orc_mwm) and scipy's linear_sum_assignment."""
import numpy as np
import pytest

import oracle
from inputs.configs import dense_to_csr

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    from paper_1908_10169_b200.build import build
    build()


def _costs(A):
    cmax = np.abs(A).max(axis=0)
    with np.errstate(divide="ignore"):
        return np.where(A != 0, np.log(cmax)[None, :] - np.log(np.abs(A)), np.inf)


def _check_scaling(A, sigma, dl, dr, tol=1e-9):
    n = A.shape[0]
    assert sorted(sigma) == list(range(n))
    assert np.all(A[np.arange(n), sigma] != 0)
    S = np.abs(dl[:, None] * A * dr[None, :])
    assert S.max() <= 1 + tol
    np.testing.assert_allclose(S[np.arange(n), sigma], 1.0, rtol=tol)


def _random(n, seed, density=0.08):
    rng = np.random.default_rng(seed)
    A = (rng.random((n, n)) < density) * rng.standard_normal((n, n)) * np.exp(rng.uniform(-4, 4, (n, n)))
    A[np.arange(n), rng.permutation(n)] += rng.uniform(0.1, 1.0, n)
    return A


def test_mwm_hand_2x2():
    from paper_1908_10169_b200 import mwm
    A = np.array([[1.0, 3.0], [2.0, 1.0]])
    sigma, dl, dr, _ = mwm(*dense_to_csr(A))
    assert list(sigma) == [1, 0]
    np.testing.assert_allclose(np.abs(dl[:, None] * A * dr[None, :]), [[0.5, 1.0], [1.0, 1.0 / 3.0]], rtol=1e-9)


@pytest.mark.parametrize("seed", range(6))
def test_mwm_matches_oracle_objective(seed):
    from paper_1908_10169_b200 import mwm
    n = [60, 61, 150, 257, 300, 33][seed]
    A = _random(n, 100 + seed)
    ip, ix, dv = dense_to_csr(A)
    sigma, dl, dr, launches = mwm(ip, ix, dv)
    so, _, _ = oracle.mwm(ip, ix, dv)
    C = _costs(A)
    obj, objo = C[np.arange(n), sigma].sum(), C[np.arange(n), so].sum()
    assert abs(obj - objo) <= 1e-8 * max(1.0, abs(objo)), (obj, objo)
    _check_scaling(A, sigma, dl, dr)
    assert launches > 0


def test_mwm_large_vs_linear_sum_assignment():
    from scipy.optimize import linear_sum_assignment
    from paper_1908_10169_b200 import mwm
    n = 2000
    A = _random(n, 7, density=0.004)
    ip, ix, dv = dense_to_csr(A)
    sigma, dl, dr, _ = mwm(ip, ix, dv)
    C = _costs(A)
    Cf = np.where(np.isfinite(C), C, 1e9)
    r, c = linear_sum_assignment(Cf)
    assert abs(C[np.arange(n), sigma].sum() - Cf[r, c].sum()) <= 1e-7 * max(1.0, Cf[r, c].sum())
    _check_scaling(A, sigma, dl, dr)


def test_mwm_forced_and_singular():
    from paper_1908_10169_b200 import BiluError, mwm
    rng = np.random.default_rng(3)
    n = 40
    perm = rng.permutation(n)
    A = np.zeros((n, n))
    A[np.arange(n), perm] = rng.uniform(-5, 5, n)
    sigma, dl, dr, _ = mwm(*dense_to_csr(A))
    assert list(sigma) == list(perm)
    _check_scaling(A, sigma, dl, dr)
    B = _random(30, 9)
    B[:, 4] = 0.0
    with pytest.raises(BiluError):
        mwm(*dense_to_csr(B))


def test_mwm_c2_full_size():
    """BASELINE configs[1] (n = 262,144): a transversal at least as good as the identity (which
    is one), with the scaling property."""
    import scipy.sparse as sp
    from inputs.configs import config2
    from paper_1908_10169_b200 import mwm
    P = config2()
    sigma, dl, dr, _ = mwm(P.indptr, P.indices, P.data)
    A = sp.csr_matrix((P.data, P.indices, P.indptr), shape=(P.n, P.n))
    assert np.array_equal(np.sort(sigma), np.arange(P.n))
    cmax = abs(A).max(axis=0).toarray().ravel()
    matched = np.abs(np.asarray(A[np.arange(P.n), sigma]).ravel())
    diag = np.abs(A.diagonal())
    obj = np.sum(np.log(cmax[sigma]) - np.log(matched))
    obj_id = np.sum(np.log(cmax) - np.log(diag))
    assert obj <= obj_id + 1e-8 * max(1.0, abs(obj_id))
    S = sp.diags(dl) @ abs(A) @ sp.diags(dr)
    assert S.max() <= 1 + 1e-9
    np.testing.assert_allclose(dl * matched * dr[sigma], 1.0, rtol=1e-9)
