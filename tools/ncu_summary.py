"""Summarise ncu captures into profiles/ncu_<tag>.json (run here, no GPU needed).

  python tools/ncu_summary.py <tag>    # reads gpurun_out/prof_<kernel>_<tag>.ncu-rep
                                       #   and gpurun_out/launches_<tag>.csv
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_requests_srcunit_tex_op_red.sum",
    "lts__t_sectors_srcunit_tex_op_red.sum", "lts__t_sectors_srcunit_tex_op_atom.sum",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor.avg.pct_of_peak_sustained_active",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
]


def raw(rep):
    if rep.endswith(".csv"):   # exported on the GPU box (large reports are not copied back)
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            res[m] = {"value": vals[i], "unit": units[i]}
    return res


def launches(path):
    per = defaultdict(list)
    with open(path) as f:
        lines = [ln for ln in f if not ln.startswith("==")]
        for r in csv.DictReader(lines):
            if r.get("Metric Name") == "gpu__time_duration.sum":
                name = r["Kernel Name"].split("(")[0].replace("void ", "")
                name = name.replace("nfg::", "").replace("<unnamed>::", "")
                per[name].append(float(r["Metric Value"]) / 1000.0)
    return {k: {"launches": len(v), "mean_us": sum(v) / len(v)} for k, v in per.items()}


def main():
    tag = sys.argv[1]
    out = {"round": 2 if tag.startswith("r2") else 1, "tag": tag,
           "source": "ncu --set full --clock-control none --import-source on (one launch each, bench.py config-2 "
                     "workload); launch list: ncu --metrics gpu__time_duration.sum --clock-control none",
           "kernels": {}}
    for k in ("k_train", "k_adam", "k_infer"):
        rep = os.path.join(ROOT, "gpurun_out", f"prof_{k}_{tag}.ncu-rep")
        csv_ = os.path.join(ROOT, "gpurun_out", f"prof_{k}_{tag}_raw.csv")
        if os.path.exists(rep):
            out["kernels"][k] = raw(rep)
        elif os.path.exists(csv_):
            out["kernels"][k] = raw(csv_)
    lp = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
    if os.path.exists(lp):
        out["launch_list_us"] = launches(lp)
    np_ = os.path.join(ROOT, "gpurun_out", f"nerf_launches_{tag}.csv")
    if os.path.exists(np_):
        out["nerf_launch_list_us"] = launches(np_)
    dst = os.path.join(ROOT, "profiles", f"ncu_{tag}.json")
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: {m: v["value"] for m, v in d.items()} for k, d in out["kernels"].items()}, indent=1))
    print(json.dumps(out.get("launch_list_us"), indent=1))


if __name__ == "__main__":
    main()
