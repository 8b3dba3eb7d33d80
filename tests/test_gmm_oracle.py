"""CPU: pin the fp64 ADBench GMM restatement (oracle/gmm.py), which is the
parity oracle of the GMM kernel class (the reference language cannot express
GMM: no exp/log, ir.hpp:121-124 -- parity unpinned by the reference)."""
import math

import numpy as np
import pytest

from oracle import gmm as G


def _small(n=6, d=3, k=4, seed=1):
    a, mu, icf, x = G.gmm_inputs(n, d, k, seed=seed)
    return a.astype(np.float64), mu.astype(np.float64), icf.astype(np.float64), x.astype(np.float64)


def test_vectorised_matches_loop_transcription():
    for seed in range(3):
        a, mu, icf, x = _small(seed=seed)
        for gamma, m in ((1.0, 0), (0.5, 3)):
            assert abs(G.gmm_objective(a, mu, icf, x, gamma, m) - G.gmm_objective_loops(a, mu, icf, x, gamma, m)) < 1e-10


def test_closed_form_1d():
    """d = 1, K = 1: sum of scalar Gaussian log-densities with precision e^q,
    plus the Wishart prior 0.5 e^{2q} - C (gamma = 1, m = 0)."""
    xs = np.array([[0.3], [-1.2], [2.0]])
    q, m0, al = 0.4, 0.5, 0.7
    e = G.gmm_objective(np.array([al]), np.array([[m0]]), np.array([[q]]), xs, 1.0, 0)
    s = math.exp(q)
    ll = sum(-0.5 * math.log(2 * math.pi) + q - 0.5 * (s * (v - m0)) ** 2 for v in xs[:, 0])
    C = 2 * 1 * (0 - 0.5 * math.log(2)) - math.lgamma(1.0)
    assert abs(e - (ll + 0.5 * s * s - C)) < 1e-12


@pytest.mark.parametrize("gamma,m", [(1.0, 0), (0.6, 2)])
def test_fd_gradient(gamma, m):
    a, mu, icf, x = _small(n=5, d=3, k=3, seed=4)
    err, da, dm, di = G.gmm_objective_grad(a, mu, icf, x, gamma, m)
    assert abs(err - G.gmm_objective(a, mu, icf, x, gamma, m)) < 1e-10
    h = 1e-6
    for arr, g in ((a, da), (mu, dm), (icf, di)):
        it = np.nditer(arr, flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            arr[idx] += h
            ep = G.gmm_objective(a, mu, icf, x, gamma, m)
            arr[idx] -= 2 * h
            em = G.gmm_objective(a, mu, icf, x, gamma, m)
            arr[idx] += h
            assert abs((ep - em) / (2 * h) - g[idx]) < 1e-5 * (1 + abs(g[idx]))


def test_tril_layout_is_column_packed():
    """ADBench Qtimesx: icf[d:] fills L column by column (i < j -> L[j][i])."""
    r, c = G.tril_index(4)
    assert list(zip(r.tolist(), c.tolist())) == [(1, 0), (2, 0), (3, 0), (2, 1), (3, 1), (3, 2)]


def test_blocked_equals_unblocked():
    a, mu, icf, x = G.gmm_inputs(300, 8, 5, seed=9)
    e1 = G.gmm_objective_grad(a, mu, icf, x, block=64)
    e2 = G.gmm_objective_grad(a, mu, icf, x, block=1 << 14)
    assert abs(e1[0] - e2[0]) < 1e-8 * abs(e2[0])
    for u, v in zip(e1[1:], e2[1:]):
        assert np.allclose(u, v, rtol=1e-10, atol=1e-10)
