"""Summarise an ncu --csv launch list (profiles helper): per-kernel count, mean time, DRAM bytes."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ix = {k: hdr.index(k) for k in ["ID", "Kernel Name", "Metric Name", "Metric Value"]}
per = collections.OrderedDict()
for r in rows[start + 1:]:
    if len(r) < len(hdr):
        continue
    per.setdefault(r[ix["ID"]], {"name": r[ix["Kernel Name"]]})[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
agg = collections.OrderedDict()
for k, v in per.items():
    nm = v["name"].split("(")[0].replace("mfreg_b200::<unnamed>::", "")
    a = agg.setdefault(nm, [0, 0.0, 0.0, 0.0])
    a[0] += 1
    a[1] += v.get("gpu__time_duration.sum", 0)
    a[2] += v.get("dram__bytes_read.sum", 0)
    a[3] += v.get("dram__bytes_write.sum", 0)
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':40s} {'n':>4s} {'us/launch':>10s} {'share':>6s} {'MB rd':>8s} {'MB wr':>8s}")
for nm, a in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{nm[:40]:40s} {a[0]:4d} {a[1]/a[0]/1e3:10.2f} {a[1]/tot:6.1%} {a[2]/a[0]/1e6:8.2f} {a[3]/a[0]/1e6:8.2f}")
