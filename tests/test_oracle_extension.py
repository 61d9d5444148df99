"""Oracle pins: the extension operators of PAPER.md §"A few signal extensions".

The displayed matrices are instantiated at N = 5, L' = 2 in tests/golden/extension_n5.txt;
(E^dagger)* is also checked against numpy's pseudoinverse (brute force), including the
N < 2L' regime where "some of the 1/2 terms become 1/3" (reading R10).
"""
import numpy as np
import pytest

from golden_io import load


def test_displayed_extension_matrices(oracle_lib):
    O = oracle_lib
    g = load("extension_n5.txt")
    y = np.arange(1.0, 6.0)
    np.testing.assert_array_equal(O.extend([1.0, 2.0, 3.0], 2, "zero"), g["E_zpd_n3"])
    np.testing.assert_array_equal(O.extend(y, 2, "symmetric"), g["E_sym"])
    np.testing.assert_array_equal(O.extend(y, 2, "periodic"), g["E_per"])
    np.testing.assert_allclose(O.extend_pinv_adjoint(y, 2, "symmetric"), g["E_sym_pinv_adj"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(O.extend_pinv_adjoint(y, 2, "periodic"), g["E_per_pinv_adj"], rtol=0, atol=1e-15)
    np.testing.assert_array_equal(O.extend_adjoint(O.extend(y, 2, "symmetric"), 5, 2, "symmetric"), g["E_symT_E_sym"])


def _dense(fn, n, m):
    return np.stack([fn(np.eye(n)[i]) for i in range(n)], axis=1).reshape(m, n)


@pytest.mark.parametrize("kind", ["zero", "symmetric", "periodic"])
@pytest.mark.parametrize("n,Lp", [(5, 2), (8, 3), (3, 2), (4, 2), (2, 2), (16, 15), (9, 7)])
def test_pinv_adjoint_matches_numpy_pinv(oracle_lib, kind, n, Lp):
    O = oracle_lib
    if kind == "symmetric" and n < Lp:
        pytest.skip("E_sym needs n >= L'")
    E = _dense(lambda e: O.extend(e, Lp, kind), n, n + 2 * Lp)
    P = _dense(lambda e: O.extend_pinv_adjoint(e, Lp, kind), n, n + 2 * Lp)
    np.testing.assert_allclose(P, np.linalg.pinv(E).T, rtol=0, atol=1e-14)
    # E^T and E^dagger from the adjoint routine
    ET = np.stack([O.extend_adjoint(np.eye(n + 2 * Lp)[t], n, Lp, kind) for t in range(n + 2 * Lp)], axis=1)
    np.testing.assert_array_equal(ET, E.T)
    Ed = np.stack([O.extend_adjoint(np.eye(n + 2 * Lp)[t], n, Lp, kind, pinv=True) for t in range(n + 2 * Lp)], axis=1)
    np.testing.assert_allclose(Ed @ E, np.eye(n), atol=1e-14)


def test_one_third_regime(oracle_lib):
    """for N <= 2L' some 1/2 weights become 1/3 (they do for N < 2L'; reading R10)."""
    O = oracle_lib
    w = O.extend_pinv_adjoint(np.ones(3), 2, "symmetric")      # counts [2, 3, 2]
    assert np.isclose(w, 1.0 / 3.0).sum() == 3 and np.isclose(w, 0.5).sum() == 4
    w4 = O.extend_pinv_adjoint(np.ones(4), 2, "symmetric")     # n = 2L': still all 1/2
    assert np.allclose(w4, 0.5)


def test_zpd_orthonormal_columns(oracle_lib):
    """E_zpd has orthonormal columns, E_zpd^dagger E_zpd = E_zpd^* E_zpd = I."""
    O = oracle_lib
    E = _dense(lambda e: O.extend(e, 4, "zero"), 7, 15)
    np.testing.assert_array_equal(E.T @ E, np.eye(7))
    np.testing.assert_allclose(np.linalg.pinv(E), E.T, atol=1e-15)
