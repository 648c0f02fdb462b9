import sys, json
for line in sys.stdin:
    line=line.strip()
    if not line.startswith("{"): continue
    l=json.loads(line)
    gn=l.get("gn_registration") or {}
    if gn: print("  gn:", {k: gn[k] for k in ("wall_s", "outer_iters", "cg_iters", "final_J")})
    print("value %.3f eval %.1f us hv %.1f us e2e %.3f gn %s launches %s frac %.3f" % (l["value"], l["ms_grad_eval"]*1e3, l["ms_gn_hv"]*1e3, l["e2e"]["value"], gn.get("wall_s"), l["gpu_launches"], l["roofline"]["frac"]))
