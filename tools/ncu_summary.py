"""Summarise ncu captures into profiles/ (tracked): launch-list shares and the
full-set metrics of the profiled kernels.

    python tools/ncu_summary.py --round r1 --launches gpurun_out/launches_r1.csv \
        --rep walk=gpurun_out/prof_walk2_r1.ncu-rep --rep sort=gpurun_out/prof_sort_r1.ncu-rep \
        --workload cfg4

Writes profiles/<round>_launches.csv (copy), profiles/<round>_summary.md and
profiles/ncu_summary.json (read by bench.py for the roofline `traffic`).
"""
import argparse
import csv
import io
import json
import os
import shutil
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

DETAILS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate",
           "L2 Hit Rate", "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput",
           "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Theoretical Occupancy",
           "Achieved Occupancy", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
           "No Eligible", "Executed Instructions", "Dynamic Shared Memory Per Block", "Block Size", "Grid Size"]
UNIT_NS = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    tot, cnt = defaultdict(float), defaultdict(int)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"].split("(")[0].replace("void ", "").strip()
        tot[name] += float(d["Metric Value"].replace(",", "")) * UNIT_NS.get(d["Metric Unit"], 1e-6)
        cnt[name] += 1
    return tot, cnt


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def details(rep):
    res = {}
    rows = ncu_csv(rep, "details")
    if rows:
        h = rows[0]
        iN, iU, iV = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
        for r in rows[1:]:
            if len(r) > iV and r[iN] in DETAILS and r[iN] not in res:
                res[r[iN]] = f"{r[iV]} {r[iU]}".strip()
            if len(r) > 4 and "kernel" not in res:
                res["kernel"] = r[4]
    raw = ncu_csv(rep, "raw")
    if len(raw) >= 3:
        h, u, v = raw[0], raw[1], raw[2]
        m = dict(zip(h, zip(u, v)))
        b = 0.0
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if k in m:
                unit, val = m[k]
                res[k] = f"{val} {unit}"
                b += float(val.replace(",", "")) * SCALE.get(unit, 1)
        res["dram_bytes_per_launch"] = b
        stalls = {}
        for k, (unit, val) in m.items():
            if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio"):
                try:
                    x = float(val)
                except ValueError:
                    continue
                if x > 0.05:
                    stalls[k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")] = x
        res["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda t: -t[1]))
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r1")
    ap.add_argument("--launches")
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--workload", default="cfg4")
    ap.add_argument("--command", default="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline")
    ap.add_argument("--exclude", default="k_walk<*, 1>;k_vel4to3;k_relabel;k_pack;k_iota",
                    help="semicolon-separated kernels launched outside the timed steps (shares also shown without them)")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    md = [f"# ncu summary, round {a.round}", "", f"Workload: BASELINE {a.workload}; command `{a.command}` on one B200 "
          "(gpurun), `--clock-control none`.", ""]
    js = {"round": a.round, "workload": a.workload, "command": a.command, "kernels": {}}
    if a.launches:
        shutil.copy(a.launches, os.path.join(PROF, f"{a.round}_launches.csv"))
        tot, cnt = launches(a.launches)
        T = sum(tot.values())
        md += ["## Launch list (`--metrics gpu__time_duration.sum`, cold-cache and serialised: compare shares)", "",
               "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        import fnmatch

        pats = [x.strip() for x in a.exclude.split(";") if x.strip()]
        # (the stats walk: the k_walk instance whose last template argument, STATS, is 1)
        excl = sorted({k for k in tot for pt in pats if fnmatch.fnmatchcase(k, pt)})
        Ts = sum(v for k, v in tot.items() if k not in excl)
        md[-2] = md[-2].replace("| share |", "| share | share of the step kernels |")
        md[-1] = "|---|---|---|---|---|"
        for k, v in sorted(tot.items(), key=lambda t: -t[1]):
            step = "untimed helper" if k in excl else f"{100 * v / Ts:.2f}%"
            md.append(f"| `{k}` | {cnt[k]} | {v:.3f} | {100 * v / T:.2f}% | {step} |")
        md.append("")
        md.append(f"Excluded from the step shares: {', '.join(excl) or 'nothing'} (launched outside bh_step: the untimed stats walk bench.py runs once for the flop model, "
                  "bh_create's relabelling, the ownership-balance read-out).")
        md.append("")
        js["launch_share"] = {k: v / T for k, v in tot.items()}
        js["launch_share_step"] = {k: v / Ts for k, v in tot.items() if k not in excl}
    for spec in a.rep:
        key, rep = spec.split("=", 1)
        d = details(rep)
        js["kernels"][key] = d
        md += [f"## `{key}` (`ncu --set full`, {os.path.basename(rep)})", "", "| metric | value |", "|---|---|"]
        for k in ["kernel"] + DETAILS + ["dram__bytes_read.sum", "dram__bytes_write.sum", "dram_bytes_per_launch"]:
            if k in d:
                md.append(f"| {k} | {d[k]} |")
        if d.get("stalls_per_issue"):
            md.append("| stall reasons (cycles per issued instruction) | " +
                      ", ".join(f"{k} {v:.2f}" for k, v in d["stalls_per_issue"].items()) + " |")
        md.append("")
    with open(os.path.join(PROF, f"{a.round}_summary.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    with open(os.path.join(PROF, "ncu_summary.json"), "w") as f:
        json.dump(js, f, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
