"""Where does the end-to-end (host buffers) gradient time go?  (GPU probe.)"""
import sys
import time

import torch

sys.path.insert(0, ".")
from tools import synth  # noqa: E402
from paper_1712_09005_b200 import _lib  # noqa: E402
from paper_1712_09005_b200.affinities import csr_from_full  # noqa: E402


def wall(fn, steps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(steps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / steps * 1e3


def main():
    n = 1_300_000
    P, Y = synth.c3(device="cuda", n=n)
    r = torch.from_numpy(P.rows).cuda()
    c = torch.from_numpy(P.cols).cuda()
    v = torch.from_numpy(P.values).cuda()
    csr = csr_from_full(n, torch.cat([r, c]), torch.cat([c, r]), torch.cat([v, v]), torch.float32, 0, n)
    del r, c, v
    y = torch.from_numpy(Y).float().cuda()
    yh = y.cpu().pin_memory()
    gh = torch.empty_like(yh).pin_memory()
    g = torch.empty_like(y)
    ctx = _lib.Context(0, 2, torch.float32, 3, 50, 1.0)
    ctx.set_affinities(csr)

    def dev():
        _lib.check(ctx.lib.fitsne_gradient(ctx.h, _lib.ptr(y), 1.0, _lib.ptr(g), None, ctx.stream), "g")

    def h2d():
        y.copy_(yh, non_blocking=True)

    def d2h():
        gh.copy_(g, non_blocking=True)

    def seq():
        h2d()
        dev()
        d2h()
        torch.cuda.current_stream().synchronize()

    def host():
        _lib.check(ctx.lib.fitsne_gradient_host(ctx.h, _lib.ptr(yh), 1.0, _lib.ptr(gh), ctx.stream), "h")

    from torch.profiler import ProfilerActivity, profile
    modes = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:] if "," in a] or [(1, 1)]
    runs = []
    for md in modes:
        sm, om = md[0], md[1]
        reps = md[2] if len(md) > 2 else 4
        cols = md[3] if len(md) > 3 else 2

        def setm(sm=sm, om=om, reps=reps, cols=cols):
            _lib.check(ctx.lib.fitsne_set_option(ctx.h, 1, sm), "opt")
            _lib.check(ctx.lib.fitsne_set_option(ctx.h, 2, om), "opt")
            _lib.check(ctx.lib.fitsne_set_option(ctx.h, 4, reps), "opt")
            _lib.check(ctx.lib.fitsne_set_option(ctx.h, 11, cols), "opt")
        runs.append((f"dev spread{sm} overlap{om} reps{reps} cols{cols}", setm, dev))
    if "--host" in sys.argv:
        runs.append(("host", lambda: (_lib.check(ctx.lib.fitsne_set_option(ctx.h, 1, 1), "o"),
                                      _lib.check(ctx.lib.fitsne_set_option(ctx.h, 2, 1), "o")), host))
    for name, setm, fn in runs:
        setm()
        print(f"{name}: {wall(fn):.3f} ms")
        fn()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            fn()
            torch.cuda.synchronize()
        evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
        t0 = min(e.time_range.start for e in evs)
        print(f"--- timeline {name}")
        for e in sorted(evs, key=lambda e: e.time_range.start):
            print(f"  {e.time_range.start - t0:8.1f} {e.time_range.end - t0:8.1f}  {e.name[:60]}")
    from paper_1712_09005_b200 import optimizer
    api = lambda: optimizer.gradient(P, yh, 1.0, 50, 3, "fft", out=gh)  # noqa: E731

    def pieces(v):
        return lambda: _lib.check(ctx.lib.fitsne_set_option(ctx.h, 10, v), "o")
    if "--host" not in sys.argv:
        return
    for name, fn in (("device", dev), ("h2d", h2d), ("d2h", d2h), ("seq", seq), ("host", host),
                     ("api", api), ("pieces1", pieces(1)), ("host", host), ("pieces0", pieces(0)),
                     ("host", host), ("device", dev), ("api", api)):
        print(f"{name:8s} {wall(fn):8.3f} ms", flush=True)


if __name__ == "__main__":
    main()
