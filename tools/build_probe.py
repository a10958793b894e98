"""One-time costs of a new P at C3: device CSR from the upper COO, the tiled
layout build (with / without the relabelling decision).  GPU probe."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from tools import synth  # noqa: E402
from paper_1712_09005_b200 import _lib  # noqa: E402
from paper_1712_09005_b200.affinities import device_csr  # noqa: E402

cache = sys.argv[sys.argv.index("--inputs-cache") + 1] if "--inputs-cache" in sys.argv else ""
if cache and Path(cache).exists():
    with np.load(cache) as z:
        P = synth.Upper(int(z["n"]), z["rows"], z["cols"], z["values"])
        Y = z["Y"]
else:
    P, Y = synth.c3(device="cuda")
y = torch.from_numpy(np.asarray(Y, dtype=np.float32)).cuda()
g = torch.empty_like(y)
torch.cuda.synchronize()
t0 = time.perf_counter()
csr = device_csr(P, torch.float32, 0)
torch.cuda.synchronize()
print(f"device_csr (upper COO on the host -> full CSR on the device): {time.perf_counter() - t0:.3f} s", flush=True)
for relabel in (0, -1):
    ctx = _lib.Context(0, 2, torch.float32, 3, 50, 1.0)
    if relabel >= 0:
        _lib.check(ctx.lib.fitsne_set_option(ctx.h, _lib.OPT_RELABEL, relabel), "relabel")
    ctx.set_affinities(csr)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _lib.check(ctx.lib.fitsne_gradient(ctx.h, _lib.ptr(y), 1.0, _lib.ptr(g), None, ctx.stream), "g")
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    _lib.check(ctx.lib.fitsne_gradient(ctx.h, _lib.ptr(y), 1.0, _lib.ptr(g), None, ctx.stream), "g")
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"relabel option {'default' if relabel < 0 else relabel}: first gradient (layout build) {t1 - t0:.3f} s, "
          f"second {1e3 * (t2 - t1):.2f} ms", flush=True)
