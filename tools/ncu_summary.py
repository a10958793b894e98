"""Summarise ncu outputs: launch list CSV (per-kernel mean time + share) and a
--set full report (key throughput metrics per kernel)."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def launches(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    agg = defaultdict(list)
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0]
        unit = d["Metric Unit"]
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0,
                 "msecond": 1e3, "ms": 1e3}
        v = v * scale[unit]
        agg[name].append(v)
    tot = sum(sum(v) for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append({"kernel": k, "launches": len(v), "mean_us": sum(v) / len(v),
                    "share": sum(v) / tot})
    return out


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__throughput.avg.pct_of_peak_sustained_active",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           "smsp__average_warp_latency_issue_stalled_barrier"]


def full(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for m in METRICS:
            if m in hdr:
                d[f"{m} [{units[hdr.index(m)]}]"] = r[hdr.index(m)]
        out.append(d)
    return out


def stalls(rep):
    """Per kernel: warp stall reasons (cycles per issued instruction) and the
    headline throughputs, largest first."""
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    pre, suf = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        st = {k[len(pre):-len(suf)]: float(v) for k, v in d.items()
              if k.startswith(pre) and k.endswith(suf) and v not in ("", "n/a")}
        st = dict(sorted(st.items(), key=lambda x: -x[1])[:8])
        keep = {m: d.get(m) for m in METRICS if m in d}
        out.append({"kernel": d["Kernel Name"].split("(")[0], "stalls": st, **keep})
    return out


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    res = {"launches": launches, "full": full, "stalls": stalls}[kind](path)
    print(json.dumps(res, indent=1))
