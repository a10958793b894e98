import sys, numpy as np, torch
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from tools import synth
from paper_1712_09005_b200.affinities import SparseAffinities
from paper_1712_09005_b200 import optimizer as opt
X, _ = synth.mixture(10_000, 50, 10, seed=1, centre_std=5.0)
r, c, v = synth.affinities(X.double().cuda(), 90, 30.0)
P = SparseAffinities(n=10_000, rows=r.cpu().numpy(), cols=c.cpu().numpy(), values=v.cpu().numpy())
ref = dict(np.load("/root/repo/tests/golden/c1_reference.npz"))
for dt in ("float32",)*8 + ("float64",)*2:
    cfg = opt.TsneConfig(dims=2, n_iter=1000, learning_rate=200.0, min_intervals=50, points_per_interval=3,
                         exaggeration=opt.ExaggerationSchedule(12.0, 250), seed=0, pca_dims=None,
                         repulsion_method="fft", dtype=dt)
    res = opt.run_tsne(affinities=P, config=cfg)
    kl, kref = res.kl_log, ref["kl_log"]
    early = np.max(np.abs(kl[:10] - kref[:10]) / kref[:10])
    span = np.ptp(res.embedding, axis=0)
    print(dt, f"early {early:.2e} final {kl[-1]:.5f} ref {kref[-1]:.5f} rel {(kl[-1]-kref[-1])/kref[-1]:+.4f} span {span} ref {ref['emb_span']}", flush=True)
