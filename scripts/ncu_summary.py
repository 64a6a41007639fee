"""Summarise an ncu --set full report: time, DRAM traffic, pipe use, stalls, FP64 op counts.

    python scripts/ncu_summary.py REPORT.ncu-rep [NODES] [--stamp KEY] [--traffic KEY]

Every quantity is converted to base units from the unit row ncu prints
(bytes, ms), so a report in GB or MB reads the same.  NODES = node-stages one
launch updates (for the per-node FP64 count).  --stamp KEY records the FP64
ops per node in profiles/fp64_ops.json together with the sha256 of the
kernel's SASS in the built library (bench.py trusts the count only while the
hash matches); --traffic KEY records the launch's DRAM bytes in
profiles/traffic.json.
"""
import csv
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "B": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0}


def load(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    return [{h: (r[i], units[i]) for i, h in enumerate(hdr)} for r in rows[2:]]


def value(get, name, base=False):
    v, unit = get.get(name, ("nan", ""))
    try:
        x = float(v.replace(",", ""))
    except ValueError:
        return float("nan")
    return x * SCALE.get(unit, 1.0) if base else x


def mangled_fragment(kernel: str) -> str:
    """'void k_stage_brick<3, 3, 2, 0, 2>(StageArgs, int)' -> 'k_stage_brickILi3ELi3ELi2ELi0ELi2EE'
    (int template arguments), the substring of the mangled symbol cuobjdump prints."""
    m = re.search(r"(\w+)<([^>]*)>", kernel)
    if not m:
        return re.search(r"(\w+)\(", kernel).group(1)
    args = [a.strip() for a in m.group(2).split(",")]
    return m.group(1) + "I" + "".join(f"Li{a}E" for a in args) + "E"


def summary(get, cells=None):
    out = {
        "kernel": get.get("Kernel Name", ("?",))[0],
        "duration_ms": value(get, "gpu__time_duration.sum", base=True),
        "dram_read_bytes": value(get, "dram__bytes_read.sum", base=True),
        "dram_write_bytes": value(get, "dram__bytes_write.sum", base=True),
        "registers": value(get, "launch__registers_per_thread"), "grid": value(get, "launch__grid_size"),
        "warps_active_pct": value(get, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "fp64_pipe_pct": value(get, "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": value(get, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "alu_pct": value(get, "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
        "lsu_pct": value(get, "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
        "xu_pct": value(get, "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
        "sm_cycles": value(get, "sm__cycles_elapsed.avg"),
        "inst_executed": value(get, "smsp__inst_executed.sum"),
    }
    fp64_rate = sum(value(get, f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed")
                    for op in ("dfma", "dmul", "dadd"))
    out["fp64_thread_ops_per_cycle"] = fp64_rate
    fp64_warp = sum(value(get, f"smsp__sass_inst_executed_op_{op}.sum") for op in ("dfma", "dmul", "dadd"))
    if fp64_warp == fp64_warp and out["inst_executed"] == out["inst_executed"] and out["inst_executed"] > 0:
        out["fp64_share_of_warp_instructions"] = fp64_warp / out["inst_executed"]
    if cells:
        out["nodes"] = cells
        out["fp64_ops_per_node"] = fp64_rate * out["sm_cycles"] / cells
        out["dram_bytes_per_node"] = (out["dram_read_bytes"] + out["dram_write_bytes"]) / cells
    hdr = list(get.keys())
    st = []
    for h in hdr:
        if "smsp__pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued"):
            try:
                st.append((h.split("stalled_")[1], float(get[h][0].replace(",", ""))))
            except ValueError:
                pass
    tot = sum(v for _, v in st) or 1
    out["stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(st, key=lambda x: -x[1])[:8]}
    return out


def main():
    args = [a for a in sys.argv[1:]]
    stamp = traffic = None
    if "--stamp" in args:
        i = args.index("--stamp")
        stamp = args[i + 1]
        del args[i:i + 2]
    if "--traffic" in args:
        i = args.index("--traffic")
        traffic = args[i + 1]
        del args[i:i + 2]
    rep = args[0]
    cells = float(args[1]) if len(args) > 1 else None
    rows = load(rep)
    outs = [summary(r, cells) for r in rows]
    print(json.dumps(outs if len(outs) > 1 else outs[0], indent=1))
    # a report of several launches is one stage's kernel sequence (the per-axis
    # walk pipeline): the stamp and the traffic are the sums over them
    if stamp and cells:
        import bench   # sass_hash of the built library

        path = os.path.join(ROOT, "profiles", "fp64_ops.json")
        d = json.load(open(path)) if os.path.exists(path) else {}
        ks = []
        for o in outs:
            sym = bench.kernel_symbol(o["kernel"])
            ks.append({"kernel": o["kernel"], "symbol": sym, "sass_sha256": bench.sass_hash(sym),
                       "ops_per_node": o["fp64_ops_per_node"]})
        names = " + ".join(o["kernel"] for o in outs)
        ent = {"ops_per_node": sum(k["ops_per_node"] for k in ks),
               "kernel": names,
               "source": f"ncu --set full {os.path.basename(rep)}: DFMA+DMUL+DADD thread instructions / "
                         f"{int(cells)} nodes of one stage ({names})"}
        if len(ks) == 1:
            ent.update(symbol=ks[0]["symbol"], sass_sha256=ks[0]["sass_sha256"])
        else:
            ent["kernels"] = ks
        d[stamp] = ent
        json.dump(d, open(path, "w"), indent=1)
    if traffic:
        path = os.path.join(ROOT, "profiles", "traffic.json")
        d = json.load(open(path)) if os.path.exists(path) else {}
        d[traffic] = sum(o["dram_read_bytes"] + o["dram_write_bytes"] for o in outs)
        json.dump(d, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
