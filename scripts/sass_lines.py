"""Per-source-line dynamic instruction counts of one kernel: joins an ncu SASS source page
(--page source --print-source sass --csv) with the line table of the kernel's cubin
(nvdisasm -g, build with -lineinfo).

    python scripts/sass_lines.py k.csv paper_1804_10541_b200/build/hv3.o k_hv3IdE [units]
"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import Counter, defaultdict


def line_table(obj, fn_pat):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
    out, cur, infn = {}, None, False
    for ln in txt.splitlines():
        if ln.startswith("//---") and ".text." in ln:
            infn = fn_pat in ln
            continue
        if not infn:
            continue
        m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', ln)
        if m:
            cur = f"{m.group(1)}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            out[int(m.group(1), 16)] = (cur, m.group(2).strip())
    return out


def main(csvp, obj, fn_pat, units=None):
    rows = list(csv.reader(open(csvp)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    i0 = rows.index(hdr)
    ca, ci, cs = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    data = [(int(r[ca], 16), float(r[ci] or 0), float(r[cs] or 0)) for r in rows[i0 + 1:] if len(r) > ci and r[ca].startswith("0x")]
    base = data[0][0]
    lt = line_table(obj, fn_pat)
    per, stl, ops = Counter(), Counter(), defaultdict(Counter)
    for a, n, st in data:
        line, ins = lt.get(a - base, ("?", "?"))
        per[line] += n
        stl[line] += st
        ops[line][ins.split()[0] if ins else "?"] += n
    tot = sum(per.values())
    f = (32.0 / units) if units else 1.0
    for line, n in per.most_common(45):
        top = ", ".join(f"{o} {f * c:.1f}" for o, c in ops[line].most_common(4))
        print(f"{line:18s} {f * n:8.1f} {100 * n / tot:5.1f}%  stall {100 * stl[line] / max(1, sum(stl.values())):5.1f}%  {top}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4]) if len(sys.argv) > 4 else None)
