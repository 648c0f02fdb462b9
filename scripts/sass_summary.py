"""Static SASS summary of the hot kernels of the built library: registers,
shared memory and the instruction classes that prove the execution scheme — TMA tensor loads
(UTMALDG), mbarrier waits (SYNCS), fp64 arithmetic, shared loads, shuffles, barriers.

    python scripts/sass_summary.py > profiles/r2_sass_summary.md
"""
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_1804_10541_b200", "build")
KERNELS = ["k_hv2", "k_ev2", "k_warp_z", "k_warp_fast", "k_nodal_finalize", "k_lap3", "k_bilap", "k_hv_closed_canon",
           "k_transfer_T", "k_chunks_warp"]
CLASSES = [("UTMALDG", r"UTMALDG"), ("SYNCS (mbarrier)", r"SYNCS"), ("DFMA", r"\bDFMA"), ("DADD", r"\bDADD"),
           ("DMUL", r"\bDMUL"), ("LDS", r"\bLDS"), ("STS", r"\bSTS"), ("LDG", r"\bLDG"), ("STG", r"\bSTG"),
           ("SHFL", r"\bSHFL"), ("BAR", r"\bBAR\b"), ("total", r".")]


def demangle_short(name):
    for k in KERNELS:
        if k in name:
            t = "<float>" if "IfE" in name else ("<double>" if "IdE" in name else "")
            return k + t
    return None


def main():
    rows = []
    for f in sorted(os.listdir(OBJ)):
        if not f.endswith(".o"):
            continue
        path = os.path.join(OBJ, f)
        sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
        res = subprocess.run(["cuobjdump", "-res-usage", path], capture_output=True, text=True).stdout
        usage = {}
        cur = None
        for line in res.splitlines():
            m = re.search(r"Function (\S+):", line)
            if m:
                cur = m.group(1)
            m = re.search(r"REG:(\d+).*SHARED:(\d+)", line)
            if m and cur:
                usage[cur] = (int(m.group(1)), int(m.group(2)))
        for block in sass.split("Function : ")[1:]:
            name = block.split("\n", 1)[0].strip()
            short = demangle_short(name)
            if not short:
                continue
            ins = [l for l in block.splitlines() if re.match(r"\s+/\*[0-9a-f]{4}\*/", l)]
            cnt = collections.OrderedDict((c, sum(1 for l in ins if re.search(rx, l))) for c, rx in CLASSES)
            reg, smem = usage.get(name, (0, 0))
            rows.append((short, f, reg, smem, cnt))
    print("| kernel | object | regs | static smem B | " + " | ".join(c for c, _ in CLASSES) + " |")
    print("|" + "---|" * (4 + len(CLASSES)))
    for short, f, reg, smem, cnt in rows:
        print(f"| {short} | {f} | {reg} | {smem} | " + " | ".join(str(v) for v in cnt.values()) + " |")


if __name__ == "__main__":
    main()
