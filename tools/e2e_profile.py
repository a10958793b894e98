"""cProfile of the host-buffer gradient call (the bench's e2e step) at C3:
Python / ctypes overhead per call beside the library's own time.  GPU probe."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from tools import synth  # noqa: E402
from paper_1712_09005_b200 import optimizer  # noqa: E402

cache = sys.argv[sys.argv.index("--inputs-cache") + 1] if "--inputs-cache" in sys.argv else ""
if cache and Path(cache).exists():
    with np.load(cache) as z:
        P = synth.Upper(int(z["n"]), z["rows"], z["cols"], z["values"])
        Y = z["Y"]
else:
    P, Y = synth.c3(device="cuda")
y_host = torch.from_numpy(np.asarray(Y, dtype=np.float32)).pin_memory()
g_host = torch.empty_like(y_host).pin_memory()
api = lambda: optimizer.gradient(P, y_host, 1.0, 50, 3, "fft", out=g_host)  # noqa: E731
for _ in range(50):
    api()
ts = []
for _ in range(200):
    t0 = time.perf_counter()
    api()
    ts.append(time.perf_counter() - t0)
ts = np.array(ts) * 1e6
print(f"per call (us): min {ts.min():.0f} p10 {np.percentile(ts, 10):.0f} median {np.median(ts):.0f} "
      f"p90 {np.percentile(ts, 90):.0f} max {ts.max():.0f}")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    api()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
