"""Per-source-line instruction / stall summary of one kernel from an ncu report
(`ncu -i rep --page source --print-source cuda,sass`). Usage: ncu_lines.py rep kernel_regex [top]"""
import csv, collections, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}", "--launch-count", "1",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
agg = collections.defaultdict(lambda: [0, 0, 0, ""])  # inst, samples, n sass
tot_i = tot_s = 0
fname = ""
hdr = None
cur = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    # rows: line-level rows carry Line No + Source; sass rows carry Address
    ln, src = r[0], r[1]
    if ln:
        cur = (fname, int(ln), src.strip()[:90])
    if r[2]:
        try:
            ins = int(r[hdr.index("Instructions Executed", 3)])
            smp = int(r[hdr.index("Warp Stall Sampling (All Samples)", 3)])
        except (ValueError, IndexError):
            continue
        a = agg[cur]
        a[0] += ins
        a[1] += smp
        a[2] += 1
        tot_i += ins
        tot_s += smp
print(f"total warp inst {tot_i:.3e}, samples {tot_s}")
for k, (i, s, n, _) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{i / tot_i:6.1%} inst {s / max(tot_s,1):6.1%} stall  n={n:4d}  {k[0]}:{k[1]}  {k[2]}")
