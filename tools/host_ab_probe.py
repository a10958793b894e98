import sys, time
sys.path.insert(0, ".")
import torch
from tools import synth
from paper_1712_09005_b200 import _lib, optimizer
P, Y = synth.c3(device="cuda")
yh = torch.from_numpy(Y).float().pin_memory(); gh = torch.empty_like(yh).pin_memory()
api = lambda: optimizer.gradient(P, yh, 1.0, 50, 3, "fft", out=gh)
api()
ctx = _lib.context(0, 2, torch.float32, 3, 50, 1.0)
res = {0: [], 2: []}
for rep in range(6):
    for h in (0, 2):
        _lib.check(ctx.lib.fitsne_set_option(ctx.h, 10, h), "o")
        for _ in range(3): api()
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(20): api()
        torch.cuda.synchronize(); res[h].append((time.perf_counter() - t) / 20 * 1e3)
for h in res: print(h, ["%.3f" % x for x in res[h]], "median %.3f" % sorted(res[h])[3])
