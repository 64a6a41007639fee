"""Summarise an ncu --set full report: time, DRAM traffic, pipe use, stalls, FP64 op counts."""
import csv
import subprocess
import sys

rep = sys.argv[1]
cells = float(sys.argv[2]) if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
get = {h: (vals[i], units[i]) for i, h in enumerate(hdr)}


def f(name):
    v = get.get(name, ("nan", ""))[0].replace(",", "")
    try:
        return float(v)
    except ValueError:
        return float("nan")


out = {
    "kernel": get.get("Kernel Name", ("?",))[0],
    "duration_ms": f("gpu__time_duration.sum") * (1e-6 if get.get("gpu__time_duration.sum", ("", ""))[1] == "ns" else
                                                   (1e-3 if get.get("gpu__time_duration.sum", ("", ""))[1] == "us" else 1)),
    "dram_read_MB": f("dram__bytes_read.sum"), "dram_write_MB": f("dram__bytes_write.sum"),
    "registers": f("launch__registers_per_thread"), "grid": f("launch__grid_size"),
    "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "fp64_pipe_pct": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "alu_pct": f("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
    "lsu_pct": f("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
    "xu_pct": f("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
    "sm_cycles": f("sm__cycles_elapsed.avg"),
}
fp64_rate = sum(f(f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed") for op in ("dfma", "dmul", "dadd"))
out["fp64_thread_ops_per_cycle"] = fp64_rate
if cells:
    out["fp64_ops_per_node"] = fp64_rate * out["sm_cycles"] / cells
st = [(h.split("stalled_")[1], float(vals[i])) for i, h in enumerate(hdr)
      if "smsp__pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued") and vals[i] not in ("", "n/a")]
tot = sum(v for _, v in st) or 1
out["stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st, key=lambda x: -x[1])[:8]}
import json
print(json.dumps(out, indent=1))
