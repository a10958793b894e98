"""CUPTI timeline of consecutive fused iterations (fitsne_iterate) of a C3 run:
kernel start / end relative to the first kernel of an iteration, for the
iterations around --at (default 60), launched back to back as run_tsne does.
GPU probe; not part of the product.

    python tools/timeline_iterate.py [--inputs-cache /tmp/c3_inputs.npz] [--at 60] [--tiled-ctas N]
"""
from __future__ import annotations

import ctypes as C
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from tools import synth  # noqa: E402
from paper_1712_09005_b200 import _lib  # noqa: E402
from paper_1712_09005_b200.affinities import device_csr  # noqa: E402


def arg(name, default):
    return type(default)(sys.argv[sys.argv.index(name) + 1]) if name in sys.argv else default


def main():
    cache = arg("--inputs-cache", "")
    if cache and Path(cache).exists():
        with np.load(cache) as z:
            P = synth.Upper(int(z["n"]), z["rows"], z["cols"], z["values"])
            Yb = z["Y"]
    else:
        P, Yb = synth.c3(device="cuda")
    n = P.n
    rng = np.random.default_rng(0)
    ya = torch.from_numpy((1e-4 * rng.standard_normal((n, 2))).astype(np.float32)).cuda()
    if "--bench-y" in sys.argv:   # the bench's embedding (span 200) instead of a run's collapsed start
        ya = torch.from_numpy(np.asarray(Yb, dtype=np.float32)).cuda()
    yb = torch.empty_like(ya)
    vel, gains = torch.zeros_like(ya), torch.ones_like(ya)
    at, nprof = arg("--at", 60), 4
    kl = torch.zeros(at + nprof + 200, dtype=torch.float64, device="cuda")
    status = torch.zeros(at + nprof + 200, dtype=torch.int32, device="cuda")
    csr = device_csr(P, torch.float32, 0)
    ctx = _lib.Context(0, 2, torch.float32, 3, 50, 1.0)
    if "--tiled-ctas" in sys.argv:
        _lib.check(ctx.lib.fitsne_set_option(ctx.h, _lib.OPT_TILED_CTAS, arg("--tiled-ctas", 0)), "ctas")
    if "--overlap" in sys.argv:
        _lib.check(ctx.lib.fitsne_set_option(ctx.h, _lib.OPT_OVERLAP, arg("--overlap", 1)), "overlap")
    lr = arg("--lr", 200.0)
    ctx.set_affinities(csr)
    it = 0

    def step():
        nonlocal ya, yb, it
        alpha, mom = 12.0, 0.5
        if "--schedule" in sys.argv:   # the bench's full run: 12 until 250, 1 until 750, then 4; momentum 0.8 from 250
            alpha = 12.0 if it < 250 else (4.0 if it >= 750 else 1.0)
            mom = 0.5 if it < 250 else 0.8
        rc = ctx.lib.fitsne_iterate(ctx.h, _lib.ptr(ya), _lib.ptr(yb), _lib.ptr(vel), _lib.ptr(gains), alpha, mom,
                                    lr, C.c_void_p(kl.data_ptr() + 8 * it), C.c_void_p(status.data_ptr() + 4 * it),
                                    ctx.stream)
        _lib.check(rc, "iterate")
        ya, yb = yb, ya
        it += 1

    for _ in range(at):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(100):
        step()
    torch.cuda.synchronize()
    per_it = (time.perf_counter() - t0) / 100
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(nprof):
            step()
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    starts = [i for i, e in enumerate(evs) if "k_bbox" in e.name]
    # the last two whole iterations
    a = starts[-2] if len(starts) >= 2 else 0
    sel = evs[a:starts[-1]] if len(starts) >= 2 else evs
    t_ref = sel[0].time_range.start
    rows = [{"kernel": e.name.split("(")[0][:70], "start_us": round(e.time_range.start - t_ref, 1),
             "end_us": round(e.time_range.end - t_ref, 1), "dur_us": round(e.time_range.end - e.time_range.start, 1)}
            for e in sel]
    span = float((ya.max(0).values - ya.min(0).values).max().item())
    print(json.dumps({"wall_us_per_iteration": round(per_it * 1e6, 1), "span": span, "iteration": it,
                      "kernels": rows}, indent=0))


main()
