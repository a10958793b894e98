"""C3 full run (short) for launch-list profiling: python tools/fullrun_probe.py [n_iter]"""
import sys, time
sys.path.insert(0, "/root/repo")
import torch
from tools import synth
from paper_1712_09005_b200 import optimizer
n_iter = int(sys.argv[1]) if len(sys.argv) > 1 else 300
P, Y = synth.c3(device="cuda", n=1_300_000, seed=3)
cfg = optimizer.TsneConfig(dims=2, n_iter=n_iter, learning_rate=200.0, min_intervals=50,
                           exaggeration=optimizer.ExaggerationSchedule(12.0, 250), seed=0,
                           pca_dims=None, repulsion_method="fft", dtype="float32")
torch.cuda.synchronize(); t0 = time.perf_counter()
res = optimizer.run_tsne(affinities=P, config=cfg)
torch.cuda.synchronize()
print(f"{n_iter} iterations: {time.perf_counter() - t0:.3f} s; KL {res.kl_log[-1]:.4f}")
