"""Summarise ncu outputs into profiles/: the launch list (per-kernel device time per
training step, serialised / cold-cache, so compare SHARES) and key counters of the
--set full captures (duration, DRAM bytes, tensor-pipe / SM throughput, occupancy).

usage: python scripts/ncu_summarize.py <launches.csv|-> <steps_in_run> <out_prefix> [--config C3] [rep.ncu-rep ...]

--config tags the summary with the workload it was captured on: bench.py takes roofline.traffic only
from a summary of its own config (profiles/r*_ncu_*.json with "config" == its config).
"""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name.replace("void ", "").replace("blstm::", "")
    return name


def launch_list(path, steps, ours_only=True):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.DictReader(io.StringIO("".join(lines))))
    agg = defaultdict(lambda: [0.0, 0])
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        agg[k][0] += float(r["Metric Value"]) / 1e3  # us
        agg[k][1] += 1
    return agg


REP_METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__cluster_dim_x": "cluster_x",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
}


def rep_summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": short(r[hdr.index("Kernel Name")])}
        for m, key in REP_METRICS.items():
            if m in hdr:
                v = r[hdr.index(m)].replace(",", "")
                try:
                    d[key] = float(v)
                except ValueError:
                    d[key] = v
                d[key + "_unit"] = units[hdr.index(m)]
        res.append(d)
    return res


def main():
    argv = sys.argv[1:]
    config = None
    if "--config" in argv:
        i = argv.index("--config")
        config = argv[i + 1]
        del argv[i:i + 2]
    launches, steps, prefix = argv[0], int(argv[1]), argv[2]
    agg = launch_list(launches, steps) if launches != "-" else {}
    total = sum(v[0] for v in agg.values()) or 1.0
    ours = {k: v for k, v in agg.items() if not k.startswith("at::") and "at::" not in k}
    summary = {"source": launches, "note": "ncu --metrics gpu__time_duration.sum --clock-control none; serialised, "
                                          "cold-cache per-launch times: compare shares, not absolutes",
               "kernels": {k: {"us_total": v[0], "launches": v[1], "share_of_listed": v[0] / total}
                           for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])},
               "ours_us_total": sum(v[0] for v in ours.values()), "all_us_total": total}
    summary["config"] = config
    reps = {}
    for rp in argv[3:]:
        reps[rp] = rep_summary(rp)
    summary["full_captures"] = reps
    json.dump(summary, open(prefix + ".json", "w"), indent=1)
    with open(prefix + ".md", "w") as f:
        f.write(f"# ncu launch list ({launches})\n\nSerialised, cold-cache per-launch device times "
                f"(`gpu__time_duration.sum`); compare shares.\n\n| kernel | launches | total us | share |\n|---|---|---|---|\n")
        for k, v in summary["kernels"].items():
            f.write(f"| {k} | {v['launches']} | {v['us_total']:.1f} | {100 * v['share_of_listed']:.1f}% |\n")
        for rp, lst in reps.items():
            f.write(f"\n## full capture {rp}\n\n")
            for d in lst:
                f.write("- " + ", ".join(f"{k}={v}" for k, v in d.items() if not k.endswith("_unit")) + "\n")
    print(open(prefix + ".md").read())


if __name__ == "__main__":
    main()
