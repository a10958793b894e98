"""Row-block x column-chunk tile statistics of the C3 P (GPU probe).

For a 2-D tiled SpMV (rows in blocks of R, Y staged in shared memory in
chunks of C points) report: non-empty tiles, entries per tile, padding to
groups of G entries, and the chunk bytes loaded per evaluation.
"""
import sys
import time

import torch

sys.path.insert(0, ".")
from tools import synth  # noqa: E402
from paper_1712_09005_b200.affinities import csr_from_full  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_300_000
    t0 = time.time()
    X, _ = synth.mixture(n, 50, 40, 3, anisotropic=True, power=1.5, device="cuda")
    rows, cols, vals = synth.affinities(X, 90, 30.0)
    r = torch.cat([rows, cols])
    c = torch.cat([cols, rows])
    v = torch.cat([vals, vals])
    csr = csr_from_full(n, r, c, v, torch.float32, 0, n)
    del r, c, v, X
    nnz = csr.col.numel()
    deg = csr.rowptr[1:] - csr.rowptr[:-1]
    row_of = torch.repeat_interleave(torch.arange(n, device="cuda"), deg, output_size=nnz)
    col = csr.col.long()
    print(f"inputs {time.time() - t0:.1f}s nnz {nnz}", flush=True)
    for R in (2048, 4096, 8192):
        for C in (4096, 8192, 16384):
            key = (row_of // R) * ((n + C - 1) // C) + col // C
            _, cnt = torch.unique(key, return_counts=True)
            for G in (256, 512):
                pad = int(((cnt + G - 1) // G * G - cnt).sum())
                nt = cnt.numel()
                print(f"R {R:5d} C {C:5d} G {G}: tiles {nt:6d} entries/tile mean {nnz / nt:8.0f} "
                      f"median {int(cnt.median()):6d} p10 {int(cnt.float().quantile(0.1)):6d} "
                      f"pad {pad / nnz * 100:5.2f}% chunk MB {nt * C * 8 / 1e6:8.0f}", flush=True)


if __name__ == "__main__":
    main()
