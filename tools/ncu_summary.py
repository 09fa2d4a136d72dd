"""Summarise ncu evidence into small text files for profiles/.

  python tools/ncu_summary.py rep  <file.ncu-rep> <out.txt>   # --set full capture
  python tools/ncu_summary.py list <launches.csv> <out.txt>   # gpu__time_duration launch list
"""
import collections
import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def rep(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary of {path}"]
    for r in rows[2:]:
        lines.append(f"\n## {r[h.index('Kernel Name')][:120]}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                lines.append(f"{k:70s} {r[i]:>18s} {units[i]}")
        stalls = [(h[i], r[i]) for i in range(len(h)) if "warp_issue_stalled" in h[i] and "pct" in h[i]]
        top = sorted(((float(v.replace(',', '') or 0), n) for n, v in stalls), reverse=True)[:6]
        for v, n in top:
            lines.append(f"{n:70s} {v:18.2f} %")
    open(out, "w").write("\n".join(lines) + "\n")


def launches(path, out):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    h = rows[0]
    iK, iV = h.index("Kernel Name"), h.index("Metric Value")
    iM = h.index("Metric Name") if "Metric Name" in h else None
    iG = h.index("Grid Size") if "Grid Size" in h else None
    iID = h.index("ID") if "ID" in h else None
    per = collections.defaultdict(dict)  # launch id -> {metric: value}
    key_of = {}
    for r in rows[1:]:
        try:
            v = float(r[iV].replace(",", ""))
        except ValueError:
            continue
        lid = r[iID] if iID is not None else len(per)
        name = r[iK].split("(")[0].replace("void ", "").replace("sd::", "").replace("<unnamed>::", "")
        key_of[lid] = (name, r[iG] if iG is not None else "")
        per[lid][r[iM] if iM is not None else "gpu__time_duration.sum"] = v
    t = collections.defaultdict(list)
    for lid, m in per.items():
        if "gpu__time_duration.sum" in m:
            t[key_of[lid]].append(m)
    tot = sum(m["gpu__time_duration.sum"] for v in t.values() for m in v)
    has_dram = any("dram__bytes_read.sum" in m for v in t.values() for m in v)
    lines = [f"# ncu launch list ({path}): gpu__time_duration.sum per launch, cold-cache & serialised",
             f"# {sum(len(v) for v in t.values())} launches, {tot/1e6:.3f} ms total",
             f"{'kernel':48s} {'grid':14s} {'n':>5s} {'avg_us':>10s} {'share':>7s}"
             + (f" {'dram_rd_MB':>11s} {'dram_wr_MB':>11s}" if has_dram else "")]
    for k, v in sorted(t.items(), key=lambda kv: -sum(m["gpu__time_duration.sum"] for m in kv[1])):
        d = [m["gpu__time_duration.sum"] for m in v]
        line = f"{k[0][:48]:48s} {k[1]:14s} {len(v):5d} {sum(d)/len(d)/1e3:10.2f} {sum(d)/tot*100:6.1f}%"
        if has_dram:
            rd = sum(m.get("dram__bytes_read.sum", 0) for m in v) / len(v)
            wr = sum(m.get("dram__bytes_write.sum", 0) for m in v) / len(v)
            line += f" {rd/1e6:11.1f} {wr/1e6:11.1f}"
        lines.append(line)
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    {"rep": rep, "list": launches}[sys.argv[1]](sys.argv[2], sys.argv[3])
