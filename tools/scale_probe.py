"""C4-like (N=10M, 2-D, random kNN P, 100 blobs in [-100,100]^2) and C5-like
(N=1M, 1-D) single-GPU gradient timings (parity at scale via properties)."""
import argparse, ctypes as C, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from tools import synth
from paper_1712_09005_b200 import _lib
from paper_1712_09005_b200.affinities import csr_from_full, DeviceCSR

ap = argparse.ArgumentParser()
ap.add_argument("--case", default="c4")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--tiled", type=int, default=1, help="FITSNE_OPT_TILED_SPMV (0 CSR, 1 auto, 2 force)")
a = ap.parse_args()
dev = 0
if a.case == "c4":
    n = a.n or 10_000_000
    y = synth.blobs2d(n, 100, 100.0, 2.0, seed=4, dirichlet=False)
    s = 2
    k = 45
else:
    n = a.n or 1_000_000
    rng = np.random.default_rng(5)
    c = rng.uniform(-200, 200, 30)
    y = (c[rng.integers(0, 30, n)] + 3.0 * rng.standard_normal(n))[:, None]
    s = 1
    k = 45
t0 = time.time()
r, cc, v = synth.random_knn_graph(n, k, seed=7, device="cuda")
rr = torch.cat([r, cc]); c2 = torch.cat([cc, r]); vv = torch.cat([v, v])
csr = csr_from_full(n, rr, c2, vv, torch.float32)
del r, cc, v, rr, c2, vv
torch.cuda.synchronize()
print(f"{a.case}: N={n} nnz={csr.col.numel()} setup {time.time()-t0:.1f}s")
yt = torch.from_numpy(y).to(device=dev, dtype=torch.float32)
ctx = _lib.Context(dev, s, torch.float32, 3, 50)
_lib.check(ctx.lib.fitsne_set_option(ctx.h, 5, a.tiled))
ctx.set_affinities(csr)
g = torch.empty_like(yt)
def step():
    _lib.check(ctx.lib.fitsne_gradient(ctx.h, _lib.ptr(yt), 1.0, _lib.ptr(g), None, ctx.stream))
for _ in range(3): step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); [step() for _ in range(a.reps)]; e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1) / a.reps
gr = _lib.Grid()
_lib.check(ctx.lib.fitsne_make_grid(ctx.h, _lib.ptr(yt), n, C.byref(gr), ctx.stream))
print(f"{a.case}: {ms:.3f} ms/grad = {1e3/ms:.1f} grad evals/s  (n_int={gr.n_intervals}, L={gr.fft_len}); "
      f"|g| finite: {bool(torch.isfinite(g).all())}")
