#!/usr/bin/env python3
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) and a
--set full capture of the apply kernel into profiles/<tag>_*.{md,json}.

usage: tools/summarize_profiles.py <tag> <launches.csv> <fold.ncu-rep> [<bench.json>]
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launch_list(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    per = collections.OrderedDict()
    count = collections.Counter()
    seq = []
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0]
        ns = float(r[ix["Metric Value"]]) * (1e3 if r[ix["Metric Unit"]] == "usecond" else
                                             1e6 if r[ix["Metric Unit"]] == "msecond" else 1.0)
        per[name] = per.get(name, 0.0) + ns
        count[name] += 1
        seq.append((name, ns))
    return per, count, seq


def raw_metrics(rep, kernel_regex="k_fold_runs"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "sm__cycles_active.avg", "gpc__cycles_elapsed.max"]
    res = {}
    for r in rows[2:]:
        d = dict(zip(h, r))
        if kernel_regex not in d.get("Kernel Name", ""):
            continue
        for k in want:
            if k in d:
                res[k] = d[k]
        res["units"] = {k: rows[1][h.index(k)] for k in want if k in h}
        break
    return res


def main():
    tag, launches, rep = sys.argv[1:4]
    bench = json.load(open(sys.argv[4])) if len(sys.argv) > 4 else None
    per, count, seq = launch_list(launches)
    total = sum(per.values())
    lines = [f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)", "",
             "Cold-cache, serialised per-launch times of `python bench.py --steps 1 --warmup 3` (all steps:"
             " 3 warm-up + 1 timed device-resident + 3 e2e). Compare SHARES, not absolutes.", "",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(per.items(), key=lambda x: -x[1]):
        lines.append(f"| `{k}` | {count[k]} | {v / 1e6:.3f} | {100 * v / total:.1f}% |")
    lines.append(f"| **total** | {sum(count.values())} | {total / 1e6:.3f} | 100% |")
    m = raw_metrics(rep)
    fold = {}
    if m:
        dur_ns = float(m["gpu__time_duration.sum"]) * (1e6 if m["units"].get("gpu__time_duration.sum") == "ms" else
                                                        1e3 if m["units"].get("gpu__time_duration.sum") == "us" else 1)
        def to_bytes(k):
            u = m["units"].get(k, "byte")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            return float(m[k]) * scale
        traffic = to_bytes("dram__bytes_read.sum") + to_bytes("dram__bytes_write.sum")
        fold = {"kernel": "k_fold_runs", "duration_ms": dur_ns / 1e6, "dram_bytes_read": to_bytes("dram__bytes_read.sum"),
                "dram_bytes_write": to_bytes("dram__bytes_write.sum"), "dram_traffic_bytes": traffic,
                "l2_hit_rate_pct": m.get("lts__t_sector_hit_rate.pct"),
                "registers": m.get("launch__registers_per_thread"),
                "sm_throughput_pct": m.get("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                "warps_active_pct": m.get("sm__warps_active.avg.pct_of_peak_sustained_active"),
                "sm_cycles_active_avg": m.get("sm__cycles_active.avg"),
                "cycles_elapsed_max": m.get("gpc__cycles_elapsed.max")}
        lines += ["", f"## `k_fold_runs` (apply), ncu --set full", "", "```", json.dumps(fold, indent=1), "```"]
        if bench:
            alg = bench["roofline"]["algorithmic_bytes"]
            lines.append(f"Algorithmic bytes per launch (16 B/update + 24 B/voxel): {alg:.3e}; DRAM traffic "
                         f"{traffic:.3e} ({traffic / alg:.2f}x).")
    if bench:
        lines += ["", "## bench line (same build)", "", "```", json.dumps(bench, indent=1)[:4000], "```"]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"{tag}_summary.md"), "w").write("\n".join(lines) + "\n")
    json.dump({"launch_ms": {k: v / 1e6 for k, v in per.items()}, "launch_count": count, "fold_full": fold},
              open(os.path.join(ROOT, "profiles", f"{tag}_summary.json"), "w"), indent=1)
    if fold:
        json.dump({"apply_dram_bytes_per_launch": fold["dram_traffic_bytes"], "source": f"profiles/{tag}_summary.json"},
                  open(os.path.join(ROOT, "profiles", "roofline_inputs.json"), "w"), indent=1)
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    main()
