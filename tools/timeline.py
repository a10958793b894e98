"""CUPTI timeline of one C3 gradient evaluation (fitsne_gradient): per-kernel
start / end relative to the first kernel of the step, and which stream
(SpMV or repulsion chain) ends last.  GPU probe; not part of the product.

    python tools/timeline.py [--inputs-cache /tmp/c3_inputs.npz] > gpurun_out/timeline.json
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from tools import synth  # noqa: E402
from paper_1712_09005_b200 import _lib  # noqa: E402
from paper_1712_09005_b200.affinities import device_csr  # noqa: E402


def main():
    cache = sys.argv[sys.argv.index("--inputs-cache") + 1] if "--inputs-cache" in sys.argv else None
    if cache and Path(cache).exists():
        with np.load(cache) as z:
            P = synth.Upper(int(z["n"]), z["rows"], z["cols"], z["values"])
            Y = z["Y"]
    else:
        P, Y = synth.c3(device="cuda")
    y = torch.from_numpy(Y).float().cuda()
    g = torch.empty_like(y)
    csr = device_csr(P, torch.float32, 0)
    ctx = _lib.Context(0, 2, torch.float32, 3, 50, 1.0)
    for name, opt in (("--overlap", _lib.OPT_OVERLAP), ("--tiled-ctas", _lib.OPT_TILED_CTAS)):
        if name in sys.argv:
            _lib.check(ctx.lib.fitsne_set_option(ctx.h, opt, int(sys.argv[sys.argv.index(name) + 1])), name)
    ctx.set_affinities(csr)

    def step():
        _lib.check(ctx.lib.fitsne_gradient(ctx.h, _lib.ptr(y), 1.0, _lib.ptr(g), None, ctx.stream), "g")

    for _ in range(10):
        step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(3):
            step()
            torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    # split into the three steps at the bbox kernel (first kernel of a step)
    starts = [i for i, e in enumerate(evs) if "k_bbox" in e.name]
    last = evs[starts[-1]:] if starts else evs
    t0 = last[0].time_range.start
    rows = [{"kernel": e.name.split("(")[0][:80], "start_us": round(e.time_range.start - t0, 1),
             "end_us": round(e.time_range.end - t0, 1), "dur_us": round(e.time_range.end - e.time_range.start, 1)}
            for e in last]
    spmv = [r for r in rows if "attract" in r["kernel"]]
    chain = [r for r in rows if "attract" not in r["kernel"] and "combine" not in r["kernel"]]
    out = {"step_kernels": rows,
           "spmv_end_us": max(r["end_us"] for r in spmv) if spmv else None,
           "chain_end_us": max(r["end_us"] for r in chain) if chain else None,
           "step_end_us": max(r["end_us"] for r in rows)}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
