"""Summaries of ncu outputs (run here, no GPU): launch-list shares and key raw metrics."""
import csv
import subprocess
import sys
from collections import defaultdict


def launches(path, top=15):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if mi is not None and r[mi] != "gpu__time_duration.sum":
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except (ValueError, IndexError):
            continue
        agg[r[ki].split("(")[0][-60:]][0] += 1
        agg[r[ki].split("(")[0][-60:]][1] += v
    tot = sum(v[1] for v in agg.values())
    out = []
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{v[1] / 1e3:11.1f} us {v[0]:4d} launches {v[1] / 1e3 / v[0]:9.1f} us/launch {100 * v[1] / tot:5.1f}%  {k}")
    return "\n".join(out)


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "sm__cycles_elapsed.avg",
        "launch__shared_mem_per_block_dynamic", "l1tex__t_bytes.sum", "sm__cycles_elapsed.avg.per_second",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", "dram__bytes_read.sum.per_second",
        "dram__bytes_write.sum.per_second"]


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        out.append("---- " + r[h.index("Kernel Name")][:90])
        for w in WANT:
            if w in h:
                i = h.index(w)
                out.append(f"  {w:70s} {r[i]:>16s} {units[i]}")
        stalls = sorted(((k, r[j]) for j, k in enumerate(h) if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                         and not k.endswith("_not_issued") and r[j] not in ("", "0")),
                        key=lambda x: -float(x[1].replace(",", "")))[:8]
        out.append("  top stall reasons (pc samples): " + ", ".join(f"{k[33:]}={v}" for k, v in stalls))
    return "\n".join(out)


if __name__ == "__main__":
    for a in sys.argv[1:]:
        print(f"== {a}")
        print(launches(a) if a.endswith(".csv") else raw(a))
