"""Summarise an ncu source page (SASS) for one kernel: opcode mix and hottest instructions."""
import csv, sys, collections
path, which = sys.argv[1], sys.argv[2]
ntop = int(sys.argv[3]) if len(sys.argv) > 3 else 40
rows = list(csv.reader(open(path)))
blocks = []; cur = None
for r in rows:
    if r and r[0] == "Kernel Name": cur = [r[1], None, []]; blocks.append(cur); continue
    if r and r[0] == "Address": cur[1] = r; continue
    if cur and cur[1] and r: cur[2].append(r)
name, hdr, body = [b for b in blocks if which in b[0]][0]
i_s = hdr.index("Warp Stall Sampling (All Samples)"); i_e = hdr.index("Instructions Executed")
stall_cols = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
f = lambda x: float(x or 0)
ts = sum(f(r[i_s]) for r in body); te = sum(f(r[i_e]) for r in body)
print(name[:80], "samples", ts, "warp inst", te)
op = collections.Counter(); ops = collections.Counter()
for r in body:
    o = r[1].split()[0] if not r[1].strip().startswith("@") else r[1].split()[1]
    o = o.split(".")[0]
    op[o] += f(r[i_e]); ops[o] += f(r[i_s])
print("opcode mix (inst %, samples %):")
for o, v in op.most_common(25): print(f"  {o:10s} {v/te*100:5.1f}%  {ops[o]/ts*100:5.1f}%")
print("hot instructions:")
for k, r in sorted(enumerate(body), key=lambda kr: -f(kr[1][i_s]))[:ntop]:
    st = sorted(((f(r[i]), h[6:]) for i, h in stall_cols), reverse=True)[:2]
    print(f"  #{k:5d} {f(r[i_s])/ts*100:5.2f}% x{f(r[i_e]):9.0f} {r[1].strip()[:70]:70s} {st}")
