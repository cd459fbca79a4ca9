"""Summarise `ncu --page raw --csv` exports (one row per captured launch)
into a markdown table: duration, DRAM bytes, achieved DRAM GB/s (bytes /
duration) and its fraction of the measured copy bandwidth, DRAM / SM /
tensor-pipe utilisation, registers, grid.

  python profiles/summarize_raw.py <prof.raw.csv> [title] [peak_gbs]
"""
import csv
import sys

KEYS = {
    "dur": "gpu__time_duration.sum",
    "rd": "dram__bytes_read.sum",
    "wr": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "warps": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "tensor": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "issue": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "fp64": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
}
TIME = {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3,
        "second": 1.0, "s": 1.0}
BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "B": 1, "KB": 1e3,
         "MB": 1e6, "GB": 1e9}


def load(path):
    with open(path) as f:
        rows = list(csv.reader(f))
    head, units, data = rows[0], rows[1], rows[2:]
    col = {n: i for i, n in enumerate(head)}
    out = []
    for r in data:
        if len(r) != len(head):
            continue
        e = {"name": r[col["Kernel Name"]].split("(")[0].split("<")[0].replace("void ", ""),
             "full": r[col["Kernel Name"]][:90]}
        for k, m in KEYS.items():
            if m not in col:
                continue
            raw = r[col[m]].replace(",", "")
            try:
                v = float(raw)
            except ValueError:
                continue
            u = units[col[m]]
            if k == "dur":
                v *= TIME.get(u, 1e-9)
            elif k in ("rd", "wr"):
                v *= BYTES.get(u, 1)
            e[k] = v
        out.append(e)
    return out


def main():
    path = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else path
    peak = float(sys.argv[3]) if len(sys.argv) > 3 else 6536.4
    rows = load(path)
    print(f"### {title}\n")
    print(f"Source: `{path}` (ncu --set full --clock-control none, cold-cache serialised "
          f"replays).  GB/s = (DRAM read + write) / duration; frac of {peak:.0f} GB/s "
          f"(MEASURED_PEAKS.json hbm_gbs).\n")
    print("| kernel | grid x block | regs | us | DRAM MB | GB/s | frac | DRAM % | SM % | "
          "warps % | issue % | tensor % | fp64 % |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for e in rows:
        mb = (e.get("rd", 0) + e.get("wr", 0)) / 1e6
        us = e.get("dur", 0) * 1e6
        gbs = mb * 1e6 / (e["dur"]) / 1e9 if e.get("dur") else 0
        print(f"| `{e['name']}` | {int(e.get('grid', 0))} x {int(e.get('block', 0))} | "
              f"{int(e.get('regs', 0))} | {us:.1f} | {mb:.1f} | {gbs:.0f} | {gbs / peak:.2f} | "
              f"{e.get('dram_pct', 0):.0f} | {e.get('sm_pct', 0):.0f} | {e.get('warps', 0):.0f} | "
              f"{e.get('issue', 0):.0f} | {e.get('tensor', 0):.0f} | {e.get('fp64', 0):.0f} |")
    print()


if __name__ == "__main__":
    main()
