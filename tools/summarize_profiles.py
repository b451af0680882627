#!/usr/bin/env python3
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) and a
--set full capture of the hot kernels of one step into profiles/<tag>_*.{md,json},
and refresh profiles/roofline_inputs.json (DRAM bytes per step of the
record_sort and apply stages, read by bench.py).

usage: tools/summarize_profiles.py <tag> <launches.csv> <full.ncu-rep> <sort_passes> [<bench.json>]
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0}
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]


def launch_list(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    per = collections.OrderedDict()
    count = collections.Counter()
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0]
        ms = float(r[ix["Metric Value"]]) * SCALE.get(r[ix["Metric Unit"]], 1e-6)
        per[name] = per.get(name, 0.0) + ms
        count[name] += 1
    return per, count


def full_capture(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        m = {"kernel": d.get("Kernel Name", "").split("(")[0]}
        for k in WANT:
            if k in d:
                u = units[h.index(k)]
                try:
                    v = float(d[k].replace(",", ""))
                except ValueError:
                    continue
                if k.startswith("dram__bytes"):
                    v *= SCALE.get(u, 1)
                elif k == "gpu__time_duration.sum":
                    v *= SCALE.get(u, 1e-6)  # -> ms
                m[k] = v
        res.append(m)
    return res


RECORD_SORT = "<7,"


def main():
    tag, launches, rep, passes = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
    bench = json.load(open(sys.argv[5])) if len(sys.argv) > 5 else None
    per, count = launch_list(launches)
    total = sum(per.values())
    lines = [f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)", "",
             "Cold-cache, serialised per-launch times of `python tools/bench_once.py 100 2` (two cfg1 steps of "
             "100 frames; the fold is one grid, k_fold_all, long and short runs together). "
             "Compare SHARES, not absolutes.", "",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(per.items(), key=lambda x: -x[1]):
        lines.append(f"| `{k}` | {count[k]} | {v:.3f} | {100 * v / total:.1f}% |")
    lines.append(f"| **total** | {sum(count.values())} | {total:.3f} | 100% |")
    caps = full_capture(rep)
    lines += ["", "## ncu --set full (one launch each, second step)", "",
              "| kernel | ms | DRAM read | DRAM write | L2 hit % | DRAM % peak | SM % | issue % | regs |",
              "|---|---|---|---|---|---|---|---|---|"]
    for m in caps:
        lines.append(f"| `{m['kernel']}` | {m.get('gpu__time_duration.sum', 0):.3f} | "
                     f"{m.get('dram__bytes_read.sum', 0) / 1e9:.3f} GB | {m.get('dram__bytes_write.sum', 0) / 1e9:.3f} GB | "
                     f"{m.get('lts__t_sector_hit_rate.pct', 0):.1f} | {m.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                     f"{m.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} | "
                     f"{m.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                     f"{m.get('launch__registers_per_thread', 0):.0f} |")

    def dram(names):
        return sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0) for m in caps
                   if any(n in m["kernel"] for n in names))

    # one launch of each sort kernel was captured per pass position; scale one pass by the pass count
    # (the record sort is the 7-bit-digit instantiation; <8, ...> is the bundling key sort)
    sort_caps = [m for m in caps if "k_sort_" in m["kernel"] and RECORD_SORT in m["kernel"]]
    n_sort_launches = max(1, len([m for m in sort_caps if "downsweep" in m["kernel"]]))
    sort_step = sum(m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
                    for m in sort_caps) * passes / n_sort_launches
    apply_step = dram(["k_fold_all", "k_fold_runs", "k_fold_short"])
    inputs = {"record_sort_dram_bytes_per_step": sort_step, "apply_dram_bytes_per_step": apply_step,
              "source": f"profiles/{tag}_summary.json", "sort_passes": passes}
    lines += ["", f"DRAM bytes per step: record_sort {sort_step:.3e} ({passes} passes), apply {apply_step:.3e}."]
    if bench:
        for st, r in bench.get("roofline_stages", {}).items():
            t = inputs.get(f"{st}_dram_bytes_per_step")
            lines.append(f"* {st}: algorithmic {r['algorithmic_bytes']:.3e} B, achieved {r['achieved']:.0f} GB/s "
                         f"({100 * r['frac']:.1f}% of {r['peak']:.0f}), DRAM traffic {t:.3e} B "
                         f"({t / r['algorithmic_bytes']:.2f}x algorithmic)" if t else f"* {st}: no capture")
        lines += ["", "## bench line (same build)", "", "```", json.dumps(bench, indent=1)[:6000], "```"]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    open(os.path.join(ROOT, "profiles", f"{tag}_summary.md"), "w").write("\n".join(lines) + "\n")
    json.dump({"launch_ms": per, "launch_count": count, "full": caps, "roofline_inputs": inputs},
              open(os.path.join(ROOT, "profiles", f"{tag}_summary.json"), "w"), indent=1)
    ri_path = os.path.join(ROOT, "profiles", "roofline_inputs.json")
    try:
        ri = json.load(open(ri_path))
    except Exception:
        ri = {}
    ri[(bench or {}).get("config", {}).get("workload", "cfg1_rgbd_merged_640x480_x100")] = inputs
    json.dump(ri, open(ri_path, "w"), indent=1)
    print("\n".join(lines[:60]))


if __name__ == "__main__":
    main()
