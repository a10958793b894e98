"""Seeded synthetic inputs for the BASELINE.json configs (bench / test input
generation; not part of the product path).

The paper's datasets are not available here; BASELINE.json's synthetic
configs stand in for them:

  C1  N=10k, d=50, 10 equal isotropic clusters, centres ~ N(0, 25 I)
  C2  N=100k 2-D embedding: 20 blobs, centres U[-40,40]^2, std 1.5, Dirichlet sizes
  C3  N=1.3M, d=50, 40 clusters, anisotropic covariances (eigenvalues
      log-uniform in [0.1, 10], random rotations), power-law sizes (exp. 1.5)
  C4  N=10M 2-D, 100 blobs in [-100,100]^2, random kNN-like P (90/row)
  C5  N=1M, d=50, 30 clusters (1-D embedding)

Affinities follow the reference pipeline's definitions (exact kNN, per-row
perplexity bisection on sigma as in affinities.py:228-285, symmetrisation
p_ij = (p_j|i + p_i|j) / 2N as in affinities.py:294-316), computed with torch
on the GPU (or CPU for small N) because the reference's numpy kNN is
infeasible at 1.3M points.
"""

from __future__ import annotations

import math

import numpy as np
import torch


def mixture(n, d, k, seed, *, centre_std=5.0, anisotropic=False, power=None, device="cpu"):
    """Gaussian mixture; returns X (n, d) float32 torch on `device` and labels."""
    rng = np.random.default_rng(seed)
    if power is None:
        sizes = np.full(k, n // k)
        sizes[: n - sizes.sum()] += 1
    else:
        w = np.arange(1, k + 1, dtype=float) ** (-power)
        w /= w.sum()
        sizes = np.floor(w * n).astype(int)
        sizes[: n - sizes.sum()] += 1
    centres = rng.normal(0.0, centre_std, (k, d))
    g = torch.Generator(device="cpu").manual_seed(int(seed))
    parts, labels = [], []
    for c in range(k):
        z = torch.randn(int(sizes[c]), d, generator=g, dtype=torch.float32)
        if anisotropic:
            lam = np.exp(rng.uniform(np.log(0.1), np.log(10.0), d))
            q, _ = np.linalg.qr(rng.standard_normal((d, d)))
            a = torch.from_numpy((q * np.sqrt(lam)[None, :]).T.astype(np.float32))
            z = z @ a
        parts.append(z + torch.from_numpy(centres[c].astype(np.float32)))
        labels.append(np.full(int(sizes[c]), c))
    X = torch.cat(parts).to(device)
    return X, np.concatenate(labels)


@torch.no_grad()
def knn(X, k, block=4096):
    """Exact k nearest neighbours (squared Euclidean), self excluded."""
    n = X.shape[0]
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    sq = (X * X).sum(1)
    idx = torch.empty((n, k), dtype=torch.int64, device=X.device)
    dist = torch.empty((n, k), dtype=torch.float32, device=X.device)
    for a in range(0, n, block):
        b = min(a + block, n)
        d2 = sq[a:b, None] + sq[None, :] - 2.0 * (X[a:b] @ X.T)
        d2.clamp_(min=0.0)
        r = torch.arange(a, b, device=X.device)
        d2[r - a, r] = float("inf")
        v, j = torch.topk(d2, k, dim=1, largest=False, sorted=True)
        idx[a:b] = j
        dist[a:b] = v
    torch.backends.cuda.matmul.allow_tf32 = old
    return idx, dist


@torch.no_grad()
def calibrate(d2, perplexity, tol=1e-4, max_iters=200):
    """Per-row sigma bisection to the target perplexity (affinities.py:228-285)."""
    d2 = d2.to(torch.float64)
    n, k = d2.shape
    lo = torch.full((n,), 1e-20, dtype=torch.float64, device=d2.device)
    hi = torch.full((n,), 1e20, dtype=torch.float64, device=d2.device)

    def perp(sigma):
        t = d2 / (2.0 * sigma[:, None] ** 2)
        t = t - t.min(dim=1, keepdim=True).values
        e = torch.exp(-t)
        s = e.sum(1)
        cond = e / s[:, None]
        ent = torch.log(s) + (t * e).sum(1) / s
        return torch.exp(ent), cond

    sigma = torch.sqrt(lo * hi)
    for _ in range(max_iters):
        p, cond = perp(sigma)
        err = p - perplexity
        if bool((err.abs() <= tol).all()):
            break
        hi = torch.where(err > 0, sigma, hi)
        lo = torch.where(err < 0, sigma, lo)
        sigma = torch.sqrt(lo * hi)
    _, cond = perp(sigma)
    return cond


@torch.no_grad()
def symmetrize(cond, idx):
    """Upper-triangle COO of p_ij = (p_j|i + p_i|j) / 2N (affinities.py:294-316)."""
    n, k = idx.shape
    i = torch.arange(n, device=idx.device).repeat_interleave(k)
    j = idx.reshape(-1)
    v = cond.reshape(-1).to(torch.float64)
    lo = torch.minimum(i, j)
    hi = torch.maximum(i, j)
    key = lo * n + hi
    uk, inv = torch.unique(key, return_inverse=True)
    vals = torch.zeros(uk.numel(), dtype=torch.float64, device=idx.device)
    vals.index_add_(0, inv, v)
    vals /= 2.0 * n
    rows = uk // n
    cols = uk % n
    return rows, cols, vals


def affinities(X, k=90, perplexity=30.0, block=4096):
    idx, d = knn(X, k, block)
    cond = calibrate(d, perplexity)
    return symmetrize(cond, idx)


def pca2(X, scale_to=100.0, dims=2):
    """Top principal directions of X, scaled so max |coordinate| = scale_to."""
    Xc = X - X.mean(0, keepdim=True)
    cov = (Xc.T.double() @ Xc.double()) / X.shape[0]
    evals, evecs = torch.linalg.eigh(cov)
    Y = (Xc.double() @ evecs[:, -dims:].flip(1))
    Y = Y * (scale_to / Y.abs().max())
    return Y


def random_knn_graph(n, k, seed, device="cpu"):
    """C4's P: k partners per row, union-symmetrised, Exp(1) weights summing to 1/2."""
    g = torch.Generator(device="cpu").manual_seed(int(seed))
    i = torch.arange(n).repeat_interleave(k)
    j = torch.randint(0, n - 1, (n * k,), generator=g)
    j = j + (j >= i).long()
    i, j = i.to(device), j.to(device)
    key = torch.unique(torch.minimum(i, j) * n + torch.maximum(i, j))
    rows, cols = key // n, key % n
    vals = torch.empty(rows.numel(), dtype=torch.float64).exponential_(1.0, generator=g).to(device)
    vals /= 2.0 * vals.sum()
    return rows, cols, vals


def blobs2d(n, k, span, std, seed, dirichlet=True):
    rng = np.random.default_rng(seed)
    c = rng.uniform(-span, span, (k, 2))
    sizes = rng.multinomial(n, rng.dirichlet(np.ones(k))) if dirichlet else np.full(k, n // k)
    if not dirichlet:
        sizes[: n - sizes.sum()] += 1
    return np.concatenate([c[i] + std * rng.standard_normal((s, 2)) for i, s in enumerate(sizes)])


class Upper:
    """Minimal SparseAffinities-compatible holder (upper COO, numpy)."""

    def __init__(self, n, rows, cols, values):
        self.n = int(n)
        self.rows = np.asarray(rows, dtype=np.int64)
        self.cols = np.asarray(cols, dtype=np.int64)
        self.values = np.asarray(values, dtype=np.float64)

    @property
    def ordered_total(self):
        return 2.0 * float(self.values.sum())


class DeviceUpper:
    """Upper-COO P held on the device as torch tensors (C4's 450M pairs need
    no host round trip; the drop-in API accepts tensors for rows/cols/values)."""

    def __init__(self, n, rows, cols, values):
        self.n, self.rows, self.cols, self.values = int(n), rows, cols, values

    @property
    def ordered_total(self):
        return 2.0 * float(self.values.sum().item())


def c4(device="cuda", n=10_000_000, seed=4):
    """Config 4: random kNN graph P (device tensors) + 100-blob 2-D Y."""
    r, c, v = random_knn_graph(n, 45, seed=seed, device=device)
    Y = blobs2d(n, 100, 100.0, 2.0, seed=seed)
    return DeviceUpper(n, r, c, v), Y


def c5(device="cuda", n=1_000_000, seed=5):
    """Config 5 inputs: 30-cluster mixture, kNN P, 1-D Y (top PCA direction)."""
    X, _ = mixture(n, 50, 30, seed, device=device)
    rows, cols, vals = affinities(X, 90, 30.0)
    Y = pca2(X, 150.0, dims=1)
    P = Upper(n, rows.cpu().numpy(), cols.cpu().numpy(), vals.cpu().numpy())
    return P, Y.cpu().numpy()


def shuffle(P, Y, seed=0):
    """The same (P, Y) with the points in a random order (upper COO kept
    rows < cols): real data arrive in no cluster order."""
    n = int(P.n)
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n)            # new i <- old perm[i]
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n)
    r, c = inv[P.rows], inv[P.cols]
    lo, hi = np.minimum(r, c), np.maximum(r, c)
    return Upper(n, lo, hi, P.values), np.ascontiguousarray(Y[perm])


def c3(device="cuda", n=1_300_000, seed=3):
    """Config 3 inputs: (P upper COO numpy holder, Y (n, 2) float64 numpy)."""
    X, _ = mixture(n, 50, 40, seed, anisotropic=True, power=1.5, device=device)
    rows, cols, vals = affinities(X, 90, 30.0)
    Y = pca2(X, 100.0)
    P = Upper(n, rows.cpu().numpy(), cols.cpu().numpy(), vals.cpu().numpy())
    return P, Y.cpu().numpy()
