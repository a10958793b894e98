"""Data -> affinities on the GPU (the step before the gradient path).

Counterpart of the reference's affinities.affinities_from_data
(affinities.py:332-358) used by ``run_tsne(data=...)``:

  kNN           exact squared-Euclidean k nearest neighbours (affinities.py:117-135),
                blocked |x|^2 + |y|^2 - 2 x.y with a library GEMM + top-k on the
                device; or the reference's random-projection forest
                (knn_approx, affinities.py:138-206; method="approx", and "auto"
                above exact_max_n points as in affinities.py:344-345): the trees
                are grown on the host with the reference's random stream (so the
                forest, hence the candidate sets, are the reference's), the
                candidates are re-ranked by true distance on the device.
  bandwidths    per-row bisection of sigma to the target perplexity with the
                reference's bracket and tolerance (affinities.py:228-285)
  symmetrize    p_ij = (p_j|i + p_i|j) / 2N over the union of directed edges
                (affinities.py:294-316) -> SparseAffinities (upper COO)

PCA front end (run_tsne, optimizer.py:355-363): randomized PCA with centred
columns and 2 power iterations, like oocpca.randomized_pca_dense.

These are one-off preprocessing steps built from library GEMM / top-k / sort
primitives; the per-iteration gradient path is the hand-written CUDA library.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .affinities import SparseAffinities

__all__ = ["AffinityConfig", "knn_exact", "knn_approx", "calibrate_bandwidths", "symmetrize",
           "affinities_from_data", "pca_reduce"]

PERPLEXITY_TOL = 1e-4        # affinities.py:28
MAX_BISECTION_ITERS = 200    # affinities.py:29
_SIGMA_LO, _SIGMA_HI = 1e-20, 1e20


@dataclass
class AffinityConfig:
    """Same knobs as the reference (affinities.py:319-329)."""

    perplexity: float = 30.0
    n_neighbors: int | None = None
    method: str = "auto"          # auto | exact | approx
    n_trees: int = 50
    subsample: int | None = None
    seed: int = 0
    exact_max_n: int = 20_000


@dataclass
class BandwidthResult:
    sigma: np.ndarray
    achieved_perplexity: np.ndarray
    conditional: np.ndarray
    converged: np.ndarray


@torch.no_grad()
def knn_exact(X: torch.Tensor, k: int, block: int = 4096):
    """(indices (N, k) int64, squared distances (N, k)) ascending, self excluded."""
    n = X.shape[0]
    if not 0 < k < n:
        raise ValueError("k must satisfy 0 < k < N")
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        sq = (X * X).sum(1)
        idx = torch.empty((n, k), dtype=torch.int64, device=X.device)
        dist = torch.empty((n, k), dtype=X.dtype, device=X.device)
        for a in range(0, n, block):
            b = min(a + block, n)
            d2 = sq[a:b, None] + sq[None, :] - 2.0 * (X[a:b] @ X.T)
            d2.clamp_(min=0.0)
            r = torch.arange(a, b, device=X.device)
            d2[r - a, r] = float("inf")
            v, j = torch.topk(d2, k, dim=1, largest=False, sorted=True)
            idx[a:b] = j
            dist[a:b] = v
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old
    return idx, dist


def _forest_leaves(x: np.ndarray, rng: np.random.Generator, leaf_cap: int) -> list[np.ndarray]:
    """Leaves of one randomized-projection tree (affinities.py:138-164).

    A node larger than leaf_cap is cut by the hyperplane through the midpoint
    of two of its points drawn with rng.choice (a random normal if they
    coincide; a random halving if one side comes out empty).  The random calls
    are made in the reference's order, depth first with the right child first,
    so a given seed grows the reference's forest.
    """
    work = [np.arange(x.shape[0], dtype=np.int64)]
    out: list[np.ndarray] = []
    while work:
        node = work.pop()
        m = node.size
        if m <= leaf_cap:
            out.append(node)
            continue
        pick = rng.choice(m, size=2, replace=False)
        u, v = x[node[pick[0]]], x[node[pick[1]]]
        w = u - v
        if not w.any():
            w = rng.standard_normal(x.shape[1])
        centre = 0.5 * (u + v)
        s = x[node] @ w - centre @ w
        lo, hi = node[s <= 0.0], node[s > 0.0]
        if lo.size == 0 or hi.size == 0:
            shuffle = rng.permutation(m)
            lo, hi = node[shuffle[: m // 2]], node[shuffle[m // 2:]]
        work.append(lo)
        work.append(hi)
    return out


@torch.no_grad()
def knn_approx(X: torch.Tensor, k: int, n_trees: int = 50, seed: int = 0, block: int = 65536):
    """Approximate kNN from a randomized-projection forest (affinities.py:167-206).

    Candidates of a point = its leaf mates over n_trees trees (leaves of at
    most max(k, 32) points); they are re-ranked by true squared distance,
    ties towards the smaller index.  The forest is grown on the host in
    float64 with the reference's seeds; the re-ranking runs on X's device, one
    tree at a time, keeping each point's k best so far.  Returns (indices
    (N, k) int64, squared distances (N, k)) like knn_exact.
    """
    n, d = X.shape
    if not 0 < k < n:
        raise ValueError("k must satisfy 0 < k < N")
    if n_trees < 1:
        raise ValueError("n_trees must be >= 1")
    cap = max(k, 32)
    xh = X.detach().to("cpu", torch.float64).numpy()
    Xd = X.to(torch.float64)
    dev = X.device
    inf = float("inf")
    best_i = torch.full((n, k), -1, dtype=torch.int64, device=dev)
    best_d = torch.full((n, k), inf, dtype=torch.float64, device=dev)
    for ss in np.random.SeedSequence(seed).spawn(n_trees):
        leaves = _forest_leaves(xh, np.random.default_rng(ss), cap)
        width = max(leaf.size for leaf in leaves)
        members = np.full((len(leaves), width), -1, dtype=np.int64)
        leaf_of = np.empty(n, dtype=np.int64)
        for j, leaf in enumerate(leaves):
            members[j, : leaf.size] = leaf
            leaf_of[leaf] = j
        members_d = torch.from_numpy(members).to(dev)
        leaf_of_d = torch.from_numpy(leaf_of).to(dev)
        for a in range(0, n, block):
            b = min(a + block, n)
            rows = torch.arange(a, b, device=dev)
            cand = members_d[leaf_of_d[a:b]]                        # (m, width)
            ok = (cand >= 0) & (cand != rows[:, None])
            diff = Xd[cand.clamp(min=0)] - Xd[a:b, None, :]
            dist = (diff * diff).sum(2)
            dist = torch.where(ok, dist, torch.full_like(dist, inf))
            ci = torch.cat([best_i[a:b], torch.where(ok, cand, torch.full_like(cand, -1))], 1)
            cd = torch.cat([best_d[a:b], dist], 1)
            # drop repeats (a point met in several trees), then the k smallest
            # distances with ties towards the smaller index: two stable sorts
            o = torch.argsort(ci, dim=1, stable=True)
            ci, cd = torch.gather(ci, 1, o), torch.gather(cd, 1, o)
            rep = torch.zeros_like(ci, dtype=torch.bool)
            rep[:, 1:] = (ci[:, 1:] == ci[:, :-1]) & (ci[:, 1:] >= 0)
            cd = torch.where(rep, torch.full_like(cd, inf), cd)
            o = torch.argsort(cd, dim=1, stable=True)[:, :k]
            best_i[a:b] = torch.gather(ci, 1, o)
            best_d[a:b] = torch.gather(cd, 1, o)
    short = torch.nonzero(torch.isinf(best_d).any(1)).flatten().cpu().numpy()
    if short.size:
        # fewer than k leaf mates in the whole forest: fill with the smallest
        # unused indices (affinities.py:193-196)
        bi, bd = best_i.cpu().numpy(), best_d.cpu().numpy()
        for i in short:
            have = np.sort(bi[i][np.isfinite(bd[i])])
            spare = np.setdiff1d(np.arange(n, dtype=np.int64), np.append(have, i), assume_unique=True)
            cands = np.sort(np.concatenate([have, spare[: k - have.size]]))
            df = xh[cands] - xh[i]
            d2 = (df * df).sum(axis=1)
            sel = np.argsort(d2, kind="stable")[:k]
            bi[i], bd[i] = cands[sel], d2[sel]
        best_i, best_d = torch.from_numpy(bi).to(dev), torch.from_numpy(bd).to(dev)
    return best_i, best_d.to(X.dtype)


@torch.no_grad()
def _perplexities(d2, sigma):
    t = d2 / (2.0 * sigma[:, None] ** 2)
    t = t - t.min(dim=1, keepdim=True).values
    e = torch.exp(-t)
    s = e.sum(1)
    cond = e / s[:, None]
    ent = torch.log(s) + (t * e).sum(1) / s
    return torch.exp(ent), cond


@torch.no_grad()
def calibrate_bandwidths(d2: torch.Tensor, perplexity: float, tol: float = PERPLEXITY_TOL,
                         max_iters: int = MAX_BISECTION_ITERS) -> BandwidthResult:
    """Bisection on sigma per row to the target perplexity (affinities.py:239-285)."""
    d2 = d2.to(torch.float64)
    n, k = d2.shape
    if not 0 < perplexity < k:
        raise ValueError("target perplexity must lie in (0, k)")
    if bool((d2.max(dim=1).values == 0).any()):
        raise ValueError("each row needs at least one positive distance")
    lo = torch.full((n,), _SIGMA_LO, dtype=torch.float64, device=d2.device)
    hi = torch.full((n,), _SIGMA_HI, dtype=torch.float64, device=d2.device)
    for _ in range(60):  # bracket expansion
        p_hi, _ = _perplexities(d2, hi)
        p_lo, _ = _perplexities(d2, lo)
        grow = p_hi < perplexity
        shrink = p_lo > perplexity
        if not bool(grow.any() or shrink.any()):
            break
        hi = torch.where(grow, hi * 10.0, hi)
        lo = torch.where(shrink, lo * 0.1, lo)
    sigma = torch.sqrt(lo * hi)
    for _ in range(max_iters):
        perp, cond = _perplexities(d2, sigma)
        err = perp - perplexity
        if bool((err.abs() <= tol).all()):
            break
        hi = torch.where(err > 0, sigma, hi)
        lo = torch.where(err < 0, sigma, lo)
        sigma = torch.sqrt(lo * hi)
    perp, cond = _perplexities(d2, sigma)
    return BandwidthResult(sigma=sigma.cpu().numpy(), achieved_perplexity=perp.cpu().numpy(),
                           conditional=cond, converged=((perp - perplexity).abs() <= tol).cpu().numpy())


@torch.no_grad()
def symmetrize(cond: torch.Tensor, idx: torch.Tensor, n: int) -> SparseAffinities:
    """p_ij = (p_j|i + p_i|j) / 2N on the union of directed edges (affinities.py:294-316)."""
    k = idx.shape[1]
    i = torch.arange(n, device=idx.device).repeat_interleave(k)
    j = idx.reshape(-1)
    v = cond.reshape(-1).to(torch.float64)
    lo = torch.minimum(i, j)
    hi = torch.maximum(i, j)
    uk, inv = torch.unique(lo * n + hi, return_inverse=True)
    vals = torch.zeros(uk.numel(), dtype=torch.float64, device=idx.device)
    vals.index_add_(0, inv, v)
    vals /= 2.0 * n
    return SparseAffinities(n=n, rows=(uk // n).cpu().numpy(), cols=(uk % n).cpu().numpy(),
                            values=vals.cpu().numpy())


@torch.no_grad()
def _subsample(idx, d2, m, seed):
    if m == idx.shape[1]:
        return idx, d2
    # the reference's random keys (affinities.py:215-216), so the kept neighbours are its own
    keys = torch.from_numpy(np.random.default_rng(seed).random(tuple(idx.shape))).to(idx.device)
    pick = torch.argsort(keys, dim=1)[:, :m]
    idx = torch.gather(idx, 1, pick)
    d2 = torch.gather(d2, 1, pick)
    # sort by distance with index tiebreak (affinities.py:221-227: two stable passes)
    by_id = torch.argsort(idx, dim=1, stable=True)
    idx, d2 = torch.gather(idx, 1, by_id), torch.gather(d2, 1, by_id)
    by_d = torch.argsort(d2, dim=1, stable=True)
    return torch.gather(idx, 1, by_d), torch.gather(d2, 1, by_d)


def affinities_from_data(data, config: AffinityConfig | None = None, device: int | None = None):
    """(SparseAffinities, BandwidthResult) from raw data (affinities.py:332-358)."""
    cfg = config or AffinityConfig()
    dev = torch.cuda.current_device() if device is None else device
    X = torch.as_tensor(np.asarray(data, dtype=np.float64)).to(device=dev)
    if X.dim() != 2:
        raise ValueError("data must be (N, d)")
    n = X.shape[0]
    k = cfg.n_neighbors or int(round(3 * cfg.perplexity))
    k = min(k, n - 1)
    if cfg.perplexity >= k:
        raise ValueError(f"perplexity {cfg.perplexity} needs more neighbors than k={k}")
    if cfg.method not in ("auto", "exact", "approx"):
        raise ValueError(f"unknown neighbor method: {cfg.method!r}")
    method = cfg.method
    if method == "auto":
        method = "exact" if n <= cfg.exact_max_n else "approx"
    if method == "exact":
        idx, d2 = knn_exact(X, k)
    else:
        idx, d2 = knn_approx(X, k, n_trees=cfg.n_trees, seed=cfg.seed)
    target = cfg.perplexity
    if cfg.subsample is not None:
        if not 1 <= cfg.subsample <= k:
            raise ValueError("m must satisfy 1 <= m <= k")
        idx, d2 = _subsample(idx, d2, cfg.subsample, cfg.seed)
        target = min(cfg.perplexity, cfg.subsample - PERPLEXITY_TOL)
    bw = calibrate_bandwidths(d2, target)
    P = symmetrize(bw.conditional, idx, n)
    bw.conditional = bw.conditional.cpu().numpy()
    return P, bw


@torch.no_grad()
def pca_reduce(x, k: int, seed: int = 0, device: int | None = None) -> np.ndarray:
    """U S of a rank-k randomized PCA of x with centred columns (2 power iterations)."""
    dev = torch.cuda.current_device() if device is None else device
    X = torch.as_tensor(np.asarray(x, dtype=np.float64)).to(device=dev)
    torch.manual_seed(int(seed))
    U, S, _ = torch.pca_lowrank(X, q=min(k + 2, min(X.shape)), center=True, niter=2)
    return (U[:, :k] * S[:k]).cpu().numpy()
