"""Oracle pins for Example 2, blind channel estimation.

Pinned by what the paper and mathematics fix, not by the oracle itself:
  * the paper's K=3, N=5 worked example: the matrices H (x_est = H s), S (x_est = S h) and S*
    displayed at P:216-236, transcribed in tests/golden/bce_conv_k3_n5.txt, against the dense
    matrices assembled column by column from the oracle with distinct prime entries;
  * the library routes the paper itself names: MATLAB conv(h, s, 'full') and
    conv(r, conj(s(end:-1:1)), 'valid'), as numpy.convolve with the same modes;
  * adjoint identities <S h, r> = <h, S* r>, <H s, r> = <s, H* r>;
  * Huber closed-form values and continuity at |z| = delta;
  * the gradient of Eq. (6): central finite differences (K=5, N=9, two channels, all weights
    nonzero), zero at a noiseless exact solution with the TV weight 0, and the dense 2 S^T r.
"""
import os

import numpy as np
import pytest

from oracle import bce as B

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "bce_conv_k3_n5.txt")


def _golden():
    mats, cur = {}, None
    with open(GOLDEN) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            if line.startswith("["):
                cur = line[1:-1]
                mats[cur] = []
                continue
            mats[cur].append(line.split())
    return mats


def _value(tok, h, s):
    if tok == ".":
        return 0.0
    return float((h if tok[0] == "h" else s)[int(tok[1:])])


def test_worked_example_matrices():
    h = np.array([2.0, 3.0, 5.0])
    s = np.array([7.0, 11.0, 13.0, 17.0, 19.0])
    K, N, M = 3, 5, 7
    g = _golden()
    Hm = np.array([[_value(t, h, s) for t in row] for row in g["H"]])
    Sm = np.array([[_value(t, h, s) for t in row] for row in g["S"]])
    SA = np.array([[_value(t, h, s) for t in row] for row in g["SADJ"]])
    # dense matrices of the oracle, column by column
    H_or = np.stack([B.conv_full(h, e) for e in np.eye(N)], 1)
    S_or = np.stack([B.conv_full(e, s) for e in np.eye(K)], 1)
    SA_or = np.stack([B.conv_adjoint_h(s, e, K) for e in np.eye(M)], 1)
    HA_or = np.stack([B.conv_adjoint_s(h, e, N) for e in np.eye(M)], 1)
    np.testing.assert_array_equal(H_or, Hm)
    np.testing.assert_array_equal(S_or, Sm)
    np.testing.assert_array_equal(SA_or, SA)
    np.testing.assert_array_equal(SA_or, Sm.T)          # S* = S^T for real s
    np.testing.assert_array_equal(HA_or, Hm.T)
    np.testing.assert_array_equal(B.conv_full(h, s), Hm @ s)


@pytest.mark.parametrize("K,N", [(1, 1), (1, 7), (6, 1), (3, 5), (17, 40), (64, 33)])
def test_against_matlab_routes(K, N):
    rng = np.random.default_rng(K * 100 + N)
    h, s, r = rng.standard_normal(K), rng.standard_normal(N), rng.standard_normal(K + N - 1)
    np.testing.assert_allclose(B.conv_full(h, s), np.convolve(h, s, "full"), rtol=0, atol=1e-13)
    np.testing.assert_allclose(B.conv_adjoint_h(s, r, K), np.convolve(r, s[::-1], "valid"), rtol=0, atol=1e-13)
    np.testing.assert_allclose(B.conv_adjoint_s(h, r, N), np.convolve(r, h[::-1], "valid"), rtol=0, atol=1e-13)


def test_adjoint_identities_batched():
    rng = np.random.default_rng(1)
    K, N = 13, 29
    h, s, r = rng.standard_normal((4, K)), rng.standard_normal((4, N)), rng.standard_normal((4, K + N - 1))
    lhs = np.sum(B.conv_full(h, s) * r, axis=-1)
    np.testing.assert_allclose(lhs, np.sum(h * B.conv_adjoint_h(s, r, K), axis=-1), rtol=1e-13)
    np.testing.assert_allclose(lhs, np.sum(s * B.conv_adjoint_s(h, r, N), axis=-1), rtol=1e-13)


def test_huber_closed_form():
    d = 0.1
    z = np.array([-0.5, -0.1, -0.05, 0.0, 0.02, 0.1, 0.3])
    np.testing.assert_allclose(B.huber(z, d), [0.1 * 0.45, 0.005, 0.00125, 0.0, 0.0002, 0.005, 0.1 * 0.25],
                               rtol=1e-15)
    np.testing.assert_allclose(B.huber_grad(z, d), [-0.1, -0.1, -0.05, 0.0, 0.02, 0.1, 0.1], rtol=1e-15)
    e = 1e-9
    assert abs(B.huber(d + e, d) - B.huber(d - e, d)) < 1e-9          # C^1 at the kink


def test_diff_adjoint_is_transpose():
    K = 7
    D = np.stack([B.diff(e) for e in np.eye(K)], 1)                      # (K-1, K)
    DT = np.stack([B.diff_adjoint(e) for e in np.eye(K - 1)], 1)         # (K, K-1)
    np.testing.assert_array_equal(DT, D.T)
    np.testing.assert_array_equal(D, np.eye(K - 1, K, 1) - np.eye(K - 1, K))


def test_gradient_finite_differences():
    rng = np.random.default_rng(2)
    C, K, N = 2, 5, 9
    h, s = rng.standard_normal((C, K)), rng.standard_normal(N)
    x = rng.standard_normal((C, K + N - 1))
    lam, delta = 0.3, 0.4       # delta comparable to the differences: both Huber branches active
    F, gh, gs = B.bce_smooth(h, s, x, lam, delta)
    eps = 1e-6
    for idx in np.ndindex(h.shape):
        hp, hm = h.copy(), h.copy()
        hp[idx] += eps
        hm[idx] -= eps
        fd = (B.bce_smooth(hp, s, x, lam, delta)[0] - B.bce_smooth(hm, s, x, lam, delta)[0]) / (2 * eps)
        assert abs(fd - gh[idx]) <= 1e-6 * max(1.0, abs(gh[idx]))
    for i in range(N):
        sp, sm = s.copy(), s.copy()
        sp[i] += eps
        sm[i] -= eps
        fd = (B.bce_smooth(h, sp, x, lam, delta)[0] - B.bce_smooth(h, sm, x, lam, delta)[0]) / (2 * eps)
        assert abs(fd - gs[i]) <= 1e-6 * max(1.0, abs(gs[i]))


def test_gradient_zero_at_noiseless_solution_and_dense_factor_two():
    rng = np.random.default_rng(3)
    C, K, N = 2, 6, 9
    h, s = rng.standard_normal((C, K)), rng.standard_normal(N)
    x = np.stack([np.convolve(h[i], s) for i in range(C)])
    F, gh, gs = B.bce_smooth(h, s, x, 0.0, 0.1)
    assert abs(F) < 1e-24
    assert np.abs(gh).max() < 1e-12 and np.abs(gs).max() < 1e-12
    # away from the solution: 2 S^T r with the dense S of the K=3, N=5 display generalised
    x2 = rng.standard_normal((C, K + N - 1))
    _, gh2, gs2 = B.bce_smooth(h, s, x2, 0.0, 0.1)
    for i in range(C):
        S = np.array([[s[m - k] if 0 <= m - k < N else 0.0 for k in range(K)] for m in range(K + N - 1)])
        r = S @ h[i] - x2[i]
        np.testing.assert_allclose(gh2[i], 2 * S.T @ r, rtol=1e-12, atol=1e-12)
    r_all = [np.convolve(h[i], s) - x2[i] for i in range(C)]
    gs_dense = sum(2 * np.array([[h[i][m - k] if 0 <= m - k < K else 0.0 for k in range(N)]
                                 for m in range(K + N - 1)]).T @ r_all[i] for i in range(C))
    np.testing.assert_allclose(gs2, gs_dense, rtol=1e-12, atol=1e-12)
