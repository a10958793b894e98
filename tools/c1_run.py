"""C1 full run (fp64 + fp32) vs the reference's KL trajectory; prints timings."""
import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from tools import synth
from paper_1712_09005_b200 import optimizer as opt
from paper_1712_09005_b200.affinities import SparseAffinities
X, _ = synth.mixture(10_000, 50, 10, seed=1, centre_std=5.0)
r, c, v = synth.affinities(X.double().cuda(), 90, 30.0)
P = SparseAffinities(n=10_000, rows=r.cpu().numpy(), cols=c.cpu().numpy(), values=v.cpu().numpy())
ref = np.load("/root/repo/tests/golden/c1_reference.npz")
for dt in ("float64", "float32"):
    cfg = opt.TsneConfig(dims=2, n_iter=1000, learning_rate=200.0, min_intervals=50, points_per_interval=3,
                         exaggeration=opt.ExaggerationSchedule(12.0, 250), seed=0, pca_dims=None,
                         repulsion_method="fft", dtype=dt)
    opt.run_tsne(affinities=P, config=cfg)  # warm
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = opt.run_tsne(affinities=P, config=cfg)
    torch.cuda.synchronize(); t = time.perf_counter() - t0
    kl = res.kl_log
    print(f"{dt}: {t:.3f} s ({1000/t:.0f} it/s); KL[0]={kl[0]:.6f} ref {ref['kl_log'][0]:.6f}; "
          f"final {kl[-1]:.6f} ref {ref['kl_log'][-1]:.6f} ({(kl[-1]/ref['kl_log'][-1]-1)*100:+.3f}%); "
          f"ref run {float(ref['run_s'][0]):.1f} s")
