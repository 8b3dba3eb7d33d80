"""Dev tool: how close can ANY fp32 evaluation get to the fp64 reference at the
BASELINE sizes?  Runs the MLP (configs[4]) and GMM (configs[2]) gradients with
numpy float32 (BLAS sgemm, fp32 intermediates) and compares them elementwise
(the reference's rtMaxRelDiff, eval.cpp:758-763) and normwise against the fp64
restatements in oracle/.  Output is committed under profiles/ as the measured
basis of the tolerances in tests/test_gpu_full.py and tests/test_gpu_gmm.py."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import gmm as G
from oracle import restate
from paper_2104_05372_b200 import programs as P

f4, f8 = np.float32, np.float64


def rel(a, b):
    a = np.asarray(a, f8).ravel()
    b = np.asarray(b, f8).ravel()
    return float(np.max(np.abs(a - b) / (1 + np.maximum(np.abs(a), np.abs(b)))))


def normrel(a, b):
    a = np.asarray(a, f8).ravel()
    b = np.asarray(b, f8).ravel()
    return float(np.max(np.abs(a - b)) / max(1.0, float(np.max(np.abs(b)))))


def mlp(b=8192, i=1024, h=1024, o=1024):
    x, w1, w2 = P.mlp_inputs(b, i, h, o)
    rl, r1, r2 = restate.mlp_grad(x, w1, w2)
    z = x @ w1
    hh = z * z
    y = hh @ w2
    dy = 2 * y
    d2 = hh.T @ dy
    dz = 2 * z * (dy @ w2.T)
    d1 = x.T @ dz
    print(f"MLP {b}x{i}x{h}x{o} numpy-fp32: dW1 rel {rel(d1, r1):.2e} norm {normrel(d1, r1):.2e}; "
          f"dW2 rel {rel(d2, r2):.2e} norm {normrel(d2, r2):.2e}", flush=True)


def gmm32(alphas, means, icf, x, block=1 << 14):
    """oracle/gmm.py's gradient with every array and product in float32."""
    n, d = x.shape
    K = means.shape[0]
    Q = G.q_matrices(icf, d).astype(f4)
    sum_qs = icf[:, :d].sum(1).astype(f4)
    W = np.zeros(K, f4)
    gy = np.zeros((K, d), f4)
    dQ = np.zeros((K, d, d), f4)
    for s in range(0, n, block):
        xb = x[s:s + block]
        beta = np.empty((xb.shape[0], K), f4)
        for k in range(K):
            y = (xb - means[k]) @ Q[k].T
            beta[:, k] = alphas[k] + sum_qs[k] - f4(0.5) * np.einsum("ij,ij->i", y, y)
        m = beta.max(1, keepdims=True)
        g = np.exp(beta - m)
        g /= g.sum(1, keepdims=True)
        W += g.sum(0)
        for k in range(K):
            xc = xb - means[k]
            gyk = g[:, k:k + 1] * (xc @ Q[k].T)
            gy[k] += gyk.sum(0)
            dQ[k] -= gyk.T @ xc
    lse_a = float(G.logsumexp(alphas.astype(f8)))
    d_alphas = W - n * np.exp(alphas - lse_a)
    d_means = np.einsum("kji,kj->ki", Q, gy)
    d_icf = np.zeros_like(icf)
    diag = np.arange(d)
    qd = np.exp(icf[:, :d])
    d_icf[:, :d] = dQ[:, diag, diag] * qd + W[:, None] + qd * qd
    r, c = G.tril_index(d)
    d_icf[:, d:] = dQ[:, r, c] + icf[:, d:]
    return d_alphas, d_means, d_icf


def gmm(n, k=200):
    a, mu, icf, x = G.gmm_inputs(n, 64, k)
    t = time.time()
    want = G.gmm_objective_grad(a, mu, icf, x)[1:]
    t1 = time.time()
    got = gmm32(a, mu, icf, x)
    t2 = time.time()
    print(f"GMM n={n} K={k} numpy-fp32 (f64 oracle {t1 - t:.0f} s, fp32 {t2 - t1:.0f} s): " +
          "; ".join(f"{nm} rel {rel(g, w):.2e} norm {normrel(g, w):.2e}"
                    for nm, g, w in zip(("d_alphas", "d_means", "d_icf"), got, want)), flush=True)


if __name__ == "__main__":
    mlp()
    mlp(3200, 64, 1024, 64)
    for n in [int(v) for v in (sys.argv[1:] or ["20000", "100000"])]:
        gmm(n)
