"""Tiled SpMV sweep on the C3 inputs (GPU probe, not a test).

python tools/tiled_probe.py [R,C,CTAS ...]   e.g. 4096,8192,0 2048,8192,0
Times fitsne_gradient_rows (SpMV + finish) and fitsne_gradient for the CSR
kernel and each tile shape.  With --ncu only the first shape is run once
(for an ncu capture of k_attract_tiled).
"""
import sys
import time

import torch

sys.path.insert(0, ".")
from tools import synth  # noqa: E402
from paper_1712_09005_b200 import _lib  # noqa: E402
from paper_1712_09005_b200.affinities import csr_from_full  # noqa: E402


def timed(fn, steps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / steps


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    ncu = "--ncu" in sys.argv
    shapes = [tuple(int(x) for x in a.split(",")) for a in args] or [(2048, 10240, 0)]
    shapes = [sh if len(sh) == 4 else (*sh, 1) for sh in shapes]  # R, C, ctas, bank order
    n = 1_300_000
    t0 = time.time()
    P, Y = synth.c3(device="cuda", n=n)
    r = torch.from_numpy(P.rows).cuda()
    c = torch.from_numpy(P.cols).cuda()
    v = torch.from_numpy(P.values).cuda()
    csr = csr_from_full(n, torch.cat([r, c]), torch.cat([c, r]), torch.cat([v, v]), torch.float32, 0, n)
    del r, c, v
    y = torch.from_numpy(Y).float().cuda()
    print(f"inputs {time.time() - t0:.1f}s", flush=True)
    f = torch.zeros_like(y)
    g = torch.empty_like(y)
    configs = ([] if ncu else [(0, 0, 0, 0, 0)]) + [(2, *s) for s in shapes]
    for mode, R, C, ctas, bank in configs:
        ctx = _lib.Context(0, 2, torch.float32, 3, 50, 1.0)
        _lib.check(ctx.lib.fitsne_set_option(ctx.h, 5, mode), "opt")
        if mode:
            _lib.check(ctx.lib.fitsne_set_option(ctx.h, 7, 2), "opt")  # shrink first
            _lib.check(ctx.lib.fitsne_set_option(ctx.h, 6, R), "opt")
            _lib.check(ctx.lib.fitsne_set_option(ctx.h, 7, C), "opt")
            _lib.check(ctx.lib.fitsne_set_option(ctx.h, 8, ctas), "opt")
            _lib.check(ctx.lib.fitsne_set_option(ctx.h, 9, bank), "opt")
        ctx.set_affinities(csr)

        def rows():
            _lib.check(ctx.lib.fitsne_gradient_rows(ctx.h, _lib.ptr(y), _lib.ptr(f), 1.0, _lib.ptr(g),
                                                    ctx.stream), "rows")

        def grad():
            _lib.check(ctx.lib.fitsne_gradient(ctx.h, _lib.ptr(y), 1.0, _lib.ptr(g), None, ctx.stream),
                       "grad")
        tb = time.time()
        rows()
        torch.cuda.synchronize()
        build = time.time() - tb
        if mode:
            import ctypes
            st = (ctypes.c_int64 * 8)()
            _lib.check(ctx.lib.fitsne_tiled_stats(ctx.h, _lib.ptr(y), st, ctx.stream), "stats")
            print(f"  tiles {st[1]} slabs {st[2]} groups {st[3]} segments {st[4]} nnz {st[5]}: "
                  f"entries/segment {st[5] / max(st[4], 1):.2f} groups/slab {st[3] / max(st[2], 1):.2f} "
                  f"slot fill {st[5] / max(32 * st[3], 1):.3f}", flush=True)
        if ncu:
            rows()
            torch.cuda.synchronize()
            break
        zc = __import__("ctypes").c_double()

        def kl():
            _lib.check(ctx.lib.fitsne_kl(ctx.h, _lib.ptr(y), 1.0, __import__("ctypes").byref(zc),
                                         ctx.stream), "kl")
        vel = torch.zeros_like(y)
        gains = torch.ones_like(y)
        y2 = y.clone()
        kd = torch.zeros(1, dtype=torch.float64, device=y.device)
        stt = torch.zeros(1, dtype=torch.int32, device=y.device)

        def iterate():
            _lib.check(ctx.lib.fitsne_iterate(ctx.h, _lib.ptr(y), _lib.ptr(y2), _lib.ptr(vel),
                                              _lib.ptr(gains), 1.0, 0.5, 200.0, _lib.ptr(kd),
                                              _lib.ptr(stt), ctx.stream), "iterate")
        t_rows = timed(rows)
        t_grad = timed(grad)
        t_kl = timed(kl)
        t_it = timed(iterate)
        print(f"mode {mode} R {R:5d} C {C:5d} ctas {ctas:4d} bank {bank}: first call {build * 1e3:8.1f} ms  "
              f"spmv {t_rows * 1e3:7.1f} us  gradient {t_grad * 1e3:7.1f} us  kl {t_kl * 1e3:7.1f} us  "
              f"iterate {t_it * 1e3:7.1f} us", flush=True)
        del ctx


if __name__ == "__main__":
    main()
