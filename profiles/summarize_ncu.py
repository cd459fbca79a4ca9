"""Summarise ncu captures into profiles/: per-kernel launch shares from a
`--metrics gpu__time_duration.sum` CSV and the key `--set full` metrics
(DRAM bytes per launch -> the roofline `traffic` field bench.py reports).

  python profiles/summarize_ncu.py <launches.csv> <prof.ncu-rep> <tag> [config]
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

HERE = os.path.dirname(os.path.abspath(__file__))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
SHORT = {"score_fast_kernel": "decode_score", "sketch_score_kernel": "sketch_score",
         "sketch_select_kernel": "select", "select_kernel": "decode_select",
         "attn_stream_kernel": "attn", "stream_merge_kernel": "attn_merge",
         "attn_mma_kernel": "attn_split", "advance_kernel": "advance",
         "prefill_attn_kernel": "prefill_attn", "prefill_plan_kernel": "prefill_plan",
         "prefill_scores_kernel": "prefill_scores", "split_select_kernel": "split_select",
         "merge_records_kernel": "split_merge"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def short(name):
    for k, v in SHORT.items():
        if k in name:
            return v
    return None


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[h + 1:]:
        agg[r[ki].split("(")[0].replace("void ", "")].append(float(r[vi].replace(",", "")))
    return agg


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = defaultdict(list)
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        rec = {}
        for k in KEYS:
            if k in hdr:
                v = r[hdr.index(k)].replace(",", "")
                try:
                    rec[k] = (float(v), units[hdr.index(k)])
                except ValueError:
                    pass
        res[name.split("(")[0].replace("void ", "")].append(rec)
    return res


def main():
    lpath, rpath, tag = sys.argv[1:4]
    config = sys.argv[4] if len(sys.argv) > 4 else "C3"
    L = launches(lpath)
    F = full(rpath)
    lines = [f"# ncu summary {tag} ({config})", "",
             f"Launch list `{os.path.basename(lpath)}` (gpu__time_duration.sum; cold-cache and "
             "serialised, so compare shares, not absolutes):", "",
             "| kernel | launches | mean us | share of hot-path time |", "|---|---|---|---|"]
    once = ("centroids", "sketch_build", "sketch_absmax")  # prefill-time, not per step
    hot = {k: v for k, v in L.items() if "dhsa::" in k and not any(o in k for o in once)}
    tot = sum(sum(v) / len(v) for v in hot.values())
    for k, v in sorted(hot.items(), key=lambda kv: -sum(kv[1]) / len(kv[1])):
        m = sum(v) / len(v)
        lines.append(f"| `{k}` | {len(v)} | {m / 1e3:.1f} | {100 * m / tot:.1f}% |")
    lines += ["", f"Full capture `{os.path.basename(rpath)}` (--set full, one row per launch):", ""]
    traffic = {}
    for k, recs in F.items():
        lines.append(f"## `{k}`")
        for rec in recs:
            lines.append("- " + "; ".join(f"{key}={val:g} {unit}" for key, (val, unit) in rec.items()))
        s = short(k)
        t = [r["dram__bytes_read.sum"][0] * SCALE.get(r["dram__bytes_read.sum"][1], 1) +
             r["dram__bytes_write.sum"][0] * SCALE.get(r["dram__bytes_write.sum"][1], 1)
             for r in recs if "dram__bytes_read.sum" in r and "dram__bytes_write.sum" in r]
        if s and t:
            traffic[s] = sum(t) / len(t)
        lines.append("")
    with open(os.path.join(HERE, f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines) + "\n")
    tp = os.path.join(HERE, "ncu_traffic.json")
    allt = json.load(open(tp)) if os.path.exists(tp) else {}
    traffic["source"] = f"{tag} ncu --set full (dram__bytes_read.sum + dram__bytes_write.sum per launch)"
    allt[config] = traffic
    json.dump(allt, open(tp, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
