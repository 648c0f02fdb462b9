"""Print an ncu --csv launch list (gpu__time_duration + dram bytes) as a per-launch table."""
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
k, order = {}, []
for r in csv.DictReader(lines[start:]):
    i = r["ID"]
    if i not in k:
        k[i] = {"name": r["Kernel Name"].split("(")[0].replace("mfreg_b200::<unnamed>::", "")[:40], "grid": r["Grid Size"],
                "stream": r["Stream"]}
        order.append(i)
    k[i][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
tot = 0.0
for i in order:
    d = k[i]
    t = d["gpu__time_duration.sum"]
    tot += t
    print(f"{i:>3} s{d['stream']:>3} {d['name']:40s} {d['grid']:>16s} {t/1e3:8.1f} us  "
          f"R {d['dram__bytes_read.sum']/1e6:8.1f} MB W {d['dram__bytes_write.sum']/1e6:8.1f} MB")
print(f"total {tot/1e3:.1f} us")
