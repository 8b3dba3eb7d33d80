"""ORACLE / TEST INFRASTRUCTURE ONLY: fp64 numpy restatements of the benchmark
programs, for full-size parity checks where the reference evaluator is too
slow (its transposed `sum` is O(n^2)).  Each restatement follows
the IR the reference emits for the program in paper_2104_05372_b200/programs.py
and is pinned against the reference evaluator at small sizes in
tests/test_oracle.py.
"""
import numpy as np


def kmeans_cost_grad(pts, asg, cs):
    """cost = sum_i sum_j (pts[i,j] - cs[asg[i],j])^2 ; dC = d cost / d cs.
    Reference IR (optimized): tape e = pts.i.j - c.(asg.i).j, cost = sum e*e,
    transposed scatter r!(asg.b)!b2 += -(e*ct + ct*e) with ct = 1."""
    p = np.asarray(pts, dtype=np.float64)
    c = np.asarray(cs, dtype=np.float64)
    a = np.asarray(asg, dtype=np.int64)
    e = p - c[a]
    cost = float((e * e).sum())
    g = np.zeros_like(c)
    np.add.at(g, a, -2.0 * e)
    return cost, g


def histogram(keys, k):
    """h!(p.i) += 1.0 over every i: exact integer counts."""
    return np.bincount(np.asarray(keys, dtype=np.int64), minlength=k).astype(np.float64)


def matmul_fwd(x, y):
    return np.asarray(x, np.float64) @ np.asarray(y, np.float64)


def contraction(x, y, x_kmajor=True, y_kmajor=False):
    """C[i][l] = sum_j x(i,j) y(j,l) in fp64 (programs.contraction)."""
    a = np.asarray(x, np.float64) if x_kmajor else np.asarray(x, np.float64).T
    b = np.asarray(y, np.float64).T if y_kmajor else np.asarray(y, np.float64)
    return a @ b


def matmul_grad(x, y):
    """loss = sum(x . y); d loss / d x = ones . y^T."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    loss = float((x @ y).sum())
    return loss, np.ones_like(x) @ y.T


def mlp_grad(x, w1, w2):
    """h = (x w1)^2, y = h w2, loss = sum y^2; grads over (w1, w2)."""
    x = np.asarray(x, np.float64)
    w1 = np.asarray(w1, np.float64)
    w2 = np.asarray(w2, np.float64)
    z = x @ w1
    h = z * z
    y = h @ w2
    loss = float((y * y).sum())
    dy = 2.0 * y
    dw2 = h.T @ dy
    dh = dy @ w2.T
    dz = dh * 2.0 * z
    dw1 = x.T @ dz
    return loss, dw1, dw2
