"""Summarise ncu reports into profiles/: per-kernel key counters (JSON) and
the per-launch duration list.  Runs here (no GPU): ncu -i <report>.

    python tools/ncu_summary.py gpurun_out/prof_heat3d.ncu-rep heat3d r01
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "ms": 1e3, "usecond": 1,
         "msecond": 1e3, "nsecond": 1e-3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep, name, rnd = Path(sys.argv[1]), sys.argv[2], sys.argv[3]
    h, u, rows = raw(rep)
    v = rows[0]
    d = {"kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else "?", "report": rep.name}
    stall = {}
    for i, k in enumerate(h):
        if k in KEYS:
            try:
                x = float(v[i].replace(",", ""))
            except ValueError:
                continue
            unit = u[i]
            if unit in SCALE and ("bytes" in k or "duration" in k):
                x *= SCALE[unit]
                unit = "byte" if "bytes" in k else "us"
            d[k] = x
            d[k + ".unit"] = unit
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                f = float(v[i])
            except ValueError:
                continue
            if f > 0.05:
                stall[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = f
    d["stalls_per_issue"] = dict(sorted(stall.items(), key=lambda kv: -kv[1]))
    out = ROOT / "profiles" / f"{rnd}_{name}_ncu.json"
    out.write_text(json.dumps(d, indent=1))
    tj = ROOT / "profiles" / "traffic.json"
    t = json.loads(tj.read_text()) if tj.exists() else {}
    t[name] = {"kernel": d["kernel"][:80],
               "dram_bytes_per_launch": d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0),
               "dram_read": d.get("dram__bytes_read.sum"), "dram_write": d.get("dram__bytes_write.sum"),
               "ncu_duration_us": d.get("gpu__time_duration.sum"),
               "source": f"profiles/{out.name} (ncu --set full --clock-control none, cold cache)"}
    tj.write_text(json.dumps(t, indent=1))
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()
