"""Summarise one kernel launch of an ncu --set full report and record it
for bench.py (profiles/ncu_traffic.json, stamped with the kernel sources'
digest so a stale capture is never reported).

    python tools/ncu_summary.py REPORT.ncu-rep KEY [KERNEL_SUBSTR] [--md OUT.md]

KEY is the bench workload ("terrain1m") or "rows_torus500k".
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "smsp__inst_executed.sum": "warp_instructions",
}
SCALE = {"duration": {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3},
         "bytes": {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}}


def read_raw(rep, kernel):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        rec = dict(zip(hdr, r))
        if kernel in rec.get("Kernel Name", ""):
            res = {"kernel_name": rec["Kernel Name"]}
            for m, k in METRICS.items():
                if m not in rec:
                    continue
                u = units[hdr.index(m)]
                v = float(rec[m].replace(",", ""))
                if k == "duration":
                    v *= SCALE["duration"].get(u, 1.0)
                elif k in ("dram_read", "dram_write"):
                    v *= SCALE["bytes"].get(u, 1.0)
                res[k] = v
            return res
    raise SystemExit(f"no launch of {kernel!r} in {rep}")


def main():
    args = sys.argv[1:]
    md = None
    if "--md" in args:
        i = args.index("--md")
        md = args[i + 1]
        del args[i:i + 2]
    rep, key = args[0], args[1]
    kernel = args[2] if len(args) > 2 else "pch_live"
    from bench import kernel_sha
    r = read_raw(rep, kernel)
    entry = {"kernel_sha": kernel_sha(), "report": os.path.basename(rep),
             "kernel_ms": r["duration"], "dram_bytes": int(r.get("dram_read", 0) + r.get("dram_write", 0)),
             "dram_read_bytes": int(r.get("dram_read", 0)), "dram_write_bytes": int(r.get("dram_write", 0)),
             "fp64_pipe_frac": round(r.get("fp64_pipe_pct", 0.0) / 100, 4),
             "issue_active_frac": round(r.get("issue_active_pct", 0.0) / 100, 4),
             "warps_active_frac": round(r.get("warps_active_pct", 0.0) / 100, 4),
             "l2_hit_frac": round(r.get("l2_hit_pct", 0.0) / 100, 4),
             "registers": int(r.get("registers", 0)),
             "warp_instructions": int(r.get("warp_instructions", 0))}
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            allt = json.load(f)
    except Exception:
        allt = {}
    allt = {k: v for k, v in allt.items() if isinstance(v, dict)}  # drop round-1 flat entries
    allt[key] = entry
    with open(path, "w") as f:
        json.dump(allt, f, indent=1)
    print(json.dumps(entry, indent=1))
    if md:
        with open(md, "w") as f:
            f.write(f"# ncu --set full: `{r['kernel_name']}` ({key})\n\n")
            f.write(f"kernel sources digest `{entry['kernel_sha']}`, report `{entry['report']}`\n\n")
            f.write("| metric | value |\n|---|---|\n")
            for m, k in METRICS.items():
                if k in r:
                    f.write(f"| {m} | {r[k]:.4g} |\n")


if __name__ == "__main__":
    main()
