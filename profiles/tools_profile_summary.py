"""Summarise ncu captures into markdown for profiles/ (run in the build container)."""
import csv, collections, subprocess, sys

def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {k: hdr.index(k) for k in ["ID", "Kernel Name", "Metric Name", "Metric Value"]}
    per = collections.OrderedDict()
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        per.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]]})[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    agg = collections.OrderedDict()
    for v in per.values():
        nm = v["name"].split("(")[0].replace("mfreg_b200::<unnamed>::", "").replace("void ", "")
        a = agg.setdefault(nm, [0, 0.0, 0.0, 0.0])
        a[0] += 1; a[1] += v.get("gpu__time_duration.sum", 0); a[2] += v.get("dram__bytes_read.sum", 0); a[3] += v.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    out = ["| kernel | launches | us/launch | share | DRAM MB read/launch | DRAM MB write/launch | DRAM GB/s |", "|---|---|---|---|---|---|---|"]
    for nm, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        us = a[1] / a[0] / 1e3
        out.append(f"| {nm} | {a[0]} | {us:.2f} | {a[1]/tot:.1%} | {a[2]/a[0]/1e6:.2f} | {a[3]/a[0]/1e6:.2f} | {(a[2]+a[3])/a[0]/(us*1e-6)/1e9:.0f} |")
    return "\n".join(out)

def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr = rows[0]
    keys = [("gpu__time_duration.sum", "duration us", 1e0), ("dram__bytes_read.sum", "DRAM read MB", 1), ("dram__bytes_write.sum", "DRAM write MB", 1),
            ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak", 1), ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak", 1),
            ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %", 1), ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %", 1),
            ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %", 1), ("launch__registers_per_thread", "regs/thread", 1),
            ("launch__grid_size", "grid", 1), ("launch__block_size", "block", 1), ("smsp__inst_executed.sum", "warp instructions", 1)]
    out = ["| kernel | " + " | ".join(k[1] for k in keys) + " | top stalls (per issue) |", "|" + "---|" * (len(keys) + 2)]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")].split("(")[0].replace("mfreg_b200::<unnamed>::", "").replace("void ", "")
        cells = []
        for k, _, _ in keys:
            v = vals[hdr.index(k)] if k in hdr else ""
            cells.append(v)
        st = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
                try: st.append((float(vals[i]), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
                except ValueError: pass
        top = ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True)[:4])
        out.append(f"| {name} | " + " | ".join(cells) + f" | {top} |")
    return "\n".join(out)

if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(launches(path) if kind == "launches" else full(path))
