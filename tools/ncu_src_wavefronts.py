"""Per-instruction shared-memory wavefronts and stall samples of one kernel
from an `ncu --set full --import-source on` report (source page, SASS view).

usage: python tools/ncu_src_wavefronts.py report.ncu-rep [kernel-regex] [top]"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    rx = sys.argv[2] if len(sys.argv) > 2 else "k_attract_tiled"
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--kernel-name", f"regex:{rx}"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    r = max(rows[2:], key=lambda q: float(q[hdr.index("gpu__time_duration.sum")]))
    kid = r[hdr.index("ID")]
    keys = ["gpu__time_duration.sum", "launch__grid_size", "sm__cycles_elapsed.max", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__throughput.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__cycles_active.avg", "sm__warps_active.avg.pct_of_peak_sustained_active"]
    for k in keys:
        if k in hdr:
            print(f"{k:75s} {r[hdr.index(k)]} {rows[1][hdr.index(k)]}")
    for k, v in zip(hdr, r):
        if "issue_stalled" in k and "per_issue_active" in k and "not_issued" not in k:
            print(f"  {k.split('issue_stalled_')[1].split('_per_issue')[0]:28s} {float(v):.2f}")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{rx}", "--launch-skip", "0", "--launch-count", "1"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hdr = rows[1]
    iS, iW, iI, iE, iN = (hdr.index(x) for x in ("Source", "L1 Wavefronts Shared", "L1 Wavefronts Shared Ideal",
                                                   "Instructions Executed", "# Samples"))
    out, tot, samples = [], 0.0, 0.0
    per = []
    for q in rows[2:]:
        if len(q) < len(hdr):
            if q and q[0] == "Kernel Name":
                break  # next launch of the report
            continue
        if q[iW] == "L1 Wavefronts Shared":
            continue
        w = float(q[iW] or 0)
        n = float(q[iN] or 0)
        samples += n
        per.append((n, float(q[iE] or 0), q[iS][:70]))
        if w > 0:
            out.append((w, float(q[iI] or 0), float(q[iE] or 0), q[iS][:60]))
            tot += w
    print(f"shared wavefronts total {tot / 1e6:.2f}M, stall samples {samples:.0f}")
    for w, i, e, s in sorted(out, reverse=True)[:top]:
        print(f"{w / 1e6:8.2f}M ideal {i / 1e6:7.2f}M exec {e / 1e6:7.3f}M wf/inst {w / max(e, 1):5.2f}  {s}")
    print("top stall-sample instructions")
    for n, e, s in sorted(per, reverse=True)[:25]:
        print(f"{n / samples * 100:6.2f}%  exec {e / 1e6:7.3f}M  {s}")


main()
