"""Summarise an ncu capture of the rollout kernel plus a launch list into
profiles/rollout_kernel_ncu.json (the file bench.py reads ``traffic`` from).

usage: python tools/ncu_summary.py REP.ncu-rep LAUNCHES.csv CAPTURE_CMD LAUNCH_CMD [OUT.json]

REP is one ``ncu --set full --import-source on -k regex:rollout_kernel -c 1``
report; LAUNCHES is the ``--metrics gpu__time_duration.sum --csv`` launch list of
the bench command (cold caches, serialised: only the shares are comparable with
bench.py's live timings).
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import OrderedDict

KEYS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum", "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second",
]
UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def as_bytes(val, unit):
    return float(val.replace(",", "")) * UNIT.get(unit.strip(), 1.0)


def launch_list(path):
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    agg = OrderedDict()
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        ns = float(r["Metric Value"].replace(",", "")) * {"ns": 1, "us": 1e3, "usecond": 1e3,
                                                             "ms": 1e6, "msecond": 1e6}.get(r["Metric Unit"], 1)
        name = r["Kernel Name"].split("(")[0][:60]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += ns
    total = sum(v[1] for v in agg.values()) or 1.0
    return {k: {"launches": n, "mean_us": round(t / n / 1e3, 1), "share": round(t / total, 4)}
            for k, (n, t) in agg.items()}


def main():
    rep, launches, cap_cmd, launch_cmd = sys.argv[1:5]
    out = sys.argv[5] if len(sys.argv) > 5 else os.path.join(os.path.dirname(__file__), "..", "profiles",
                                                              "rollout_kernel_ncu.json")
    head, units, rows = raw_rows(rep)
    r = rows[0]
    col = {k: i for i, k in enumerate(head)}
    metrics = {k: f"{r[col[k]]} {units[col[k]]}".strip() for k in KEYS if k in col}
    dram = sum(as_bytes(r[col[k]], units[col[k]]) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(r[col[k]].replace(",", "") or 0)
              for k in head if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")}
    tot = sum(stalls.values()) or 1.0
    top = dict(sorted(((k, round(v / tot, 3)) for k, v in stalls.items()), key=lambda kv: -kv[1])[:8])
    doc = OrderedDict()
    doc["capture"] = cap_cmd
    doc["kernel"] = f"{r[col['Kernel Name']]} grid {r[col['launch__grid_size']]} x {r[col['launch__block_size']]}"
    doc["metrics"] = metrics
    doc["dram_bytes_per_launch"] = dram
    doc["stall_samples_top"] = top
    doc[f"launch_list ({launch_cmd})"] = launch_list(launches)
    with open(out, "w") as fh:
        json.dump(doc, fh, indent=1)
    print(json.dumps({"dram_bytes_per_launch": dram, "stalls": top}))


if __name__ == "__main__":
    main()
