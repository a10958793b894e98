"""Time the repulsion stages on a C3-sized synthetic embedding (no P needed).
Usage: python tools/stage_probe.py [--n N] [--sorted 0|1] [--reps R]"""
import argparse, ctypes as C, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_1712_09005_b200 import _lib

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_300_000)
ap.add_argument("--sorted", type=int, default=1)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--case", default="blobs")
a = ap.parse_args()
rng = np.random.default_rng(0)
if a.case == "c3like":
    # 40 power-law-sized anisotropic blobs, span ~200 (n_int ~ 200 < 219: counting-sort path)
    w = np.arange(1, 41, dtype=float) ** -1.5; w /= w.sum()
    lab = rng.choice(40, a.n, p=w)
    c = rng.uniform(-70, 70, (40, 2)); s = rng.uniform(3, 15, (40, 2))
    y = c[lab] + s[lab] * rng.standard_normal((a.n, 2))
elif a.case == "blobs":
    c = rng.uniform(-80, 80, (40, 2)); s = rng.uniform(2, 12, 40)
    lab = rng.integers(0, 40, a.n)
    y = c[lab] + s[lab, None] * rng.standard_normal((a.n, 2))
else:
    y = rng.normal(0, 1e-4, (a.n, 2))
yt = torch.from_numpy(y).to(device=0, dtype=torch.float32)
ctx = _lib.Context(0, 2, torch.float32, 3, 50)
_lib.check(ctx.lib.fitsne_set_option(ctx.h, 1, a.sorted))
g = _lib.Grid()
_lib.check(ctx.lib.fitsne_make_grid(ctx.h, _lib.ptr(yt), a.n, C.byref(g), ctx.stream))
acc = torch.zeros(int(ctx.lib.fitsne_grid_accum_len(ctx.h)), dtype=torch.float32, device=0)
st = torch.cuda.current_stream()
def spread():
    _lib.check(ctx.lib.fitsne_spread_tsne(ctx.h, _lib.ptr(yt), a.n, _lib.ptr(acc), ctx.stream))
def fft():
    _lib.check(ctx.lib.fitsne_fft_tsne(ctx.h, _lib.ptr(acc), a.n, 0, None, ctx.stream))
for name, fn in (("spread", spread), ("fft", fft)):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(a.reps): fn()
    e1.record(st); e1.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) / a.reps * 1e3:.1f} us  (n_int={g.n_intervals}, L={g.fft_len})")
