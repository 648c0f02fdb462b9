"""Dynamic SASS instruction mix of one kernel from an ncu report (source page, SASS view).

    ncu -i rep.ncu-rep --page source --csv --kernel-name regex:k_hv2 --launch-count 1 \
        --print-source sass > k.csv
    python scripts/sass_mix.py k.csv [units]     # units: voxels per launch -> instr per voxel
"""
import csv
import sys
from collections import Counter


def main(path, units=None):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == "Address")
    i0 = rows.index(hdr)
    ci, cs, cst = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    mix, stall = Counter(), Counter()
    tot = 0
    for r in rows[i0 + 1:]:
        if len(r) <= ci:
            continue
        try:
            n = float(r[ci].replace(",", ""))
        except ValueError:
            continue
        src = r[cs].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        op = op.split(".")[0]
        mix[op] += n
        stall[op] += float(r[cst] or 0)
        tot += n
    print(f"total warp instructions {tot:.4g}" + (f"  thread-instr/unit {32 * tot / units:.1f}" if units else ""))
    st = sum(stall.values()) or 1
    for op, n in mix.most_common(40):
        extra = f"  per-unit {32 * n / units:6.1f}" if units else ""
        print(f"{op:10s} {n:14.4g} {100 * n / tot:5.1f}%{extra}  stall-samples {100 * stall[op] / st:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None)
