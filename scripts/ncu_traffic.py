"""Turn an `ncu --set full` capture of the bench workload into profiles/traffic.json.

bench.py quotes `roofline.traffic` (dram__bytes_read.sum + dram__bytes_write.sum per launch)
only from this file, and only while the CUDA sources hash to the value recorded here.

    ncu --set full --import-source on --clock-control none -k regex:"k_hv2|k_ev2|k_warp_fast" \
        -s 3 -c 6 -o gpurun_out/full_c4 -f python bench.py --workload c4 --steps 1 --warmup 1 \
        --no-gn --no-cpu --no-fast32
    python scripts/ncu_traffic.py c4 gpurun_out/full_c4.ncu-rep
"""
import csv
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import TRAFFIC_FILE, csrc_sha  # noqa: E402

KERNELS = {"k_hv2": "hv_pass", "k_ev2": "eval_pass", "k_warp_z": "warp", "k_warp_fast": "warp"}
EXTRA = {"fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
         "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
         "dram_pct_of_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
         "warp_inst": "smsp__inst_executed.sum"}


def main(workload: str, rep: str) -> None:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    # the raw page scales each metric to a display unit (row 2): convert to bytes / ns
    scale_of = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                "nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9,
                "ns": 1.0, "us": 1e3, "ms": 1e6, "s": 1e9}
    col = {k: hdr.index(k) for k in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum")}
    col.update({k: hdr.index(v) for k, v in EXTRA.items() if v in hdr})
    per = {}
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        key = next((v for k, v in KERNELS.items() if k in name and "<float>" not in name), None)
        if key is None:
            continue
        f = lambda c: float(r[col[c]].replace(",", "")) * scale_of.get(units[col[c]], 1.0)  # noqa: E731
        per.setdefault(key, []).append((f("dram__bytes_read.sum") + f("dram__bytes_write.sum"), f("gpu__time_duration.sum"),
                                        {k: f(k) for k in EXTRA if k in col}))
    try:
        with open(TRAFFIC_FILE) as fh:
            out = json.load(fh)
    except FileNotFoundError:
        out = {}
    sha = csrc_sha()
    for k, v in per.items():
        e = {"bytes": statistics.median(b for b, _, _ in v), "launches": len(v),
             "duration_us_ncu": statistics.median(t for _, t, _ in v) / 1e3, "csrc_sha": sha,
             "source": os.path.relpath(rep, ROOT)}
        for x in EXTRA:
            if x in v[0][2]:
                e[x] = statistics.median(m[x] for _, _, m in v)
        out.setdefault(workload, {})[k] = e
    with open(TRAFFIC_FILE, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out[workload], indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
