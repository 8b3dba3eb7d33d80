"""ORACLE / TEST INFRASTRUCTURE ONLY: fp64 restatement of the ADBench GMM
objective and its gradient (BASELINE.json configs[2]).

Parity status: **unpinned by the reference.**  The reference language has no
`exp`/`log` (/root/reference/proj/include/dexlet/ir.hpp:121-124), so the GMM
objective cannot be written as a dexlet program, and no GMM code exists under
/root/reference.  The algorithm restated here is the one ADBench publishes
(microsoft/ADBench, `src/cpp/shared/gmm.h`: `gmm_objective`, `Qtimesx`,
`preprocess_qs`, `log_wishart_prior`, `log_gamma_distrib`, `logsumexp`; the
dependency is not vendored anywhere in this image).  It is pinned instead by

* a closed form: d = 1, K = 1 reduces to a scalar Gaussian log-likelihood
  (tests/test_gmm_oracle.py::test_closed_form_1d);
* central finite differences of :func:`gmm_objective` for every parameter
  block of :func:`gmm_objective_grad` (test_gmm_oracle.py::test_fd_gradient);
* agreement of the vectorised objective with a literal per-point loop
  transcription of ADBench's C++ (:func:`gmm_objective_loops`).

Parameter layout (ADBench): alphas [K], means [K][d], icf [K][d(d+1)/2] where
icf[k][:d] are the log-diagonal of Q_k and icf[k][d:] the strictly lower
triangle of Q_k packed column by column (Qtimesx: for i < j, L[j][i] in
order i-major).  The gradient is returned in the same layout.
"""
from __future__ import annotations

import math

import numpy as np


def icf_size(d: int) -> int:
    return d * (d + 1) // 2


def tril_index(d: int):
    """(rows, cols) of the packed strictly-lower entries, in ADBench order
    (column i ascending, then row j = i+1 .. d-1)."""
    rows, cols = [], []
    for i in range(d):
        for j in range(i + 1, d):
            rows.append(j)
            cols.append(i)
    return np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64)


def q_matrices(icf: np.ndarray, d: int) -> np.ndarray:
    """Q_k = diag(exp(icf[k,:d])) + L_k (lower triangular), [K][d][d] fp64."""
    icf = np.asarray(icf, dtype=np.float64)
    K = icf.shape[0]
    Q = np.zeros((K, d, d))
    r, c = tril_index(d)
    Q[:, r, c] = icf[:, d:]
    Q[:, np.arange(d), np.arange(d)] = np.exp(icf[:, :d])
    return Q


def logsumexp(v: np.ndarray, axis=-1) -> np.ndarray:
    m = np.max(v, axis=axis, keepdims=True)
    return (np.log(np.sum(np.exp(v - m), axis=axis, keepdims=True)) + m).squeeze(axis)


def log_gamma_distrib(a: float, p: int) -> float:
    out = 0.25 * p * (p - 1) * math.log(math.pi)
    for j in range(1, p + 1):
        out += math.lgamma(a + 0.5 * (1 - j))
    return out


def log_wishart_prior(icf: np.ndarray, d: int, gamma: float, m: int) -> float:
    icf = np.asarray(icf, dtype=np.float64)
    K = icf.shape[0]
    n = d + m + 1
    C = n * d * (math.log(gamma) - 0.5 * math.log(2)) - log_gamma_distrib(0.5 * n, d)
    sum_qs = icf[:, :d].sum(1)
    frob = (np.exp(icf[:, :d]) ** 2).sum(1) + (icf[:, d:] ** 2).sum(1)
    return float((0.5 * gamma * gamma * frob - m * sum_qs).sum() - K * C)


def _main_terms(alphas, means, Q, sum_qs, xb):
    """beta[i,k] = alpha_k + sum_qs_k - 0.5 ||Q_k (x_i - mu_k)||^2 for a block of points."""
    K = means.shape[0]
    beta = np.empty((xb.shape[0], K))
    for k in range(K):
        y = (xb - means[k]) @ Q[k].T
        beta[:, k] = alphas[k] + sum_qs[k] - 0.5 * np.einsum("ij,ij->i", y, y)
    return beta


def gmm_objective(alphas, means, icf, x, gamma: float = 1.0, m: int = 0, block: int = 1 << 14) -> float:
    """ADBench gmm_objective (fp64)."""
    x = np.asarray(x, dtype=np.float64)
    alphas = np.asarray(alphas, dtype=np.float64)
    means = np.asarray(means, dtype=np.float64)
    icf = np.asarray(icf, dtype=np.float64)
    n, d = x.shape
    Q = q_matrices(icf, d)
    sum_qs = icf[:, :d].sum(1)
    slse = 0.0
    for s in range(0, n, block):
        slse += float(logsumexp(_main_terms(alphas, means, Q, sum_qs, x[s:s + block]), axis=1).sum())
    const = -n * d * 0.5 * math.log(2 * math.pi)
    return const + slse - n * float(logsumexp(alphas)) + log_wishart_prior(icf, d, gamma, m)


def gmm_objective_loops(alphas, means, icf, x, gamma: float = 1.0, m: int = 0) -> float:
    """Literal transcription of ADBench's per-point C++ loops (small sizes only):
    Qtimesx applies diag(exp(q)) then the column-packed lower triangle."""
    x = np.asarray(x, dtype=np.float64)
    n, d = x.shape
    K = len(alphas)
    slse = 0.0
    for ix in range(n):
        main = []
        for ik in range(K):
            xc = [x[ix, j] - means[ik][j] for j in range(d)]
            out = [math.exp(icf[ik][j]) * xc[j] for j in range(d)]
            li = 0
            for i in range(d):
                for j in range(i + 1, d):
                    out[j] += icf[ik][d + li] * xc[i]
                    li += 1
            main.append(alphas[ik] + sum(icf[ik][:d]) - 0.5 * sum(v * v for v in out))
        mx = max(main)
        slse += math.log(sum(math.exp(v - mx) for v in main)) + mx
    mx = max(alphas)
    lse_a = math.log(sum(math.exp(a - mx) for a in alphas)) + mx
    const = -n * d * 0.5 * math.log(2 * math.pi)
    return const + slse - n * lse_a + log_wishart_prior(np.asarray(icf), d, gamma, m)


def gmm_objective_grad(alphas, means, icf, x, gamma: float = 1.0, m: int = 0, block: int = 1 << 14):
    """(err, d_alphas [K], d_means [K][d], d_icf [K][d(d+1)/2]) in fp64.

    With g_ik = softmax_k(beta_i), y_ik = Q_k (x_i - mu_k):
      d alpha_k = sum_i g_ik - n softmax(alpha)_k
      d mu_k    = Q_k^T sum_i g_ik y_ik
      d Q_k     = -sum_i g_ik y_ik (x_i - mu_k)^T     (lower triangle used)
      d icf diag_j = dQ_k[j,j] exp(q_kj) + sum_i g_ik + gamma^2 exp(2 q_kj) - m
      d icf L      = dQ_k[r,c] + gamma^2 L_k[r,c]"""
    x = np.asarray(x, dtype=np.float64)
    alphas = np.asarray(alphas, dtype=np.float64)
    means = np.asarray(means, dtype=np.float64)
    icf = np.asarray(icf, dtype=np.float64)
    n, d = x.shape
    K = means.shape[0]
    Q = q_matrices(icf, d)
    sum_qs = icf[:, :d].sum(1)
    slse = 0.0
    W = np.zeros(K)
    gy = np.zeros((K, d))
    dQ = np.zeros((K, d, d))
    for s in range(0, n, block):
        xb = x[s:s + block]
        beta = _main_terms(alphas, means, Q, sum_qs, xb)
        lse = logsumexp(beta, axis=1)
        slse += float(lse.sum())
        g = np.exp(beta - lse[:, None])
        W += g.sum(0)
        for k in range(K):
            xc = xb - means[k]
            y = xc @ Q[k].T
            gyk = g[:, k:k + 1] * y
            gy[k] += gyk.sum(0)
            dQ[k] -= gyk.T @ xc
    const = -n * d * 0.5 * math.log(2 * math.pi)
    lse_a = float(logsumexp(alphas))
    err = const + slse - n * lse_a + log_wishart_prior(icf, d, gamma, m)
    d_alphas = W - n * np.exp(alphas - lse_a)
    d_means = np.einsum("kji,kj->ki", Q, gy)
    d_icf = np.zeros_like(icf)
    diag = np.arange(d)
    qd = np.exp(icf[:, :d])
    d_icf[:, :d] = dQ[:, diag, diag] * qd + W[:, None] + gamma * gamma * qd * qd - m
    r, c = tril_index(d)
    d_icf[:, d:] = dQ[:, r, c] + gamma * gamma * icf[:, d:]
    return err, d_alphas, d_means, d_icf


# Seeded input generator shared with the product bench (pure numpy, no
# library load): lives with the other workload generators.
from paper_2104_05372_b200.programs import gmm_inputs  # noqa: E402,F401
