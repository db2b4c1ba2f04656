"""Summarise ncu outputs into markdown for profiles/ (development tool).

usage: ncu_summary.py launches <launches.csv> <title>
       ncu_summary.py launches_dram <launches.csv> <title>   (time + dram__bytes_read/write per kernel)
       ncu_summary.py full <report.ncu-rep> <title>
"""
import collections
import csv
import io
import math
import subprocess
import sys


def launches(path, title):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    i_name, i_val = hdr.index("Kernel Name"), hdr.index("Metric Value")
    i_met, i_unit = hdr.index("Metric Name"), hdr.index("Metric Unit")
    scale = {"ns": 1.0, "nsecond": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[i_met] != "gpu__time_duration.sum":
            continue
        try:
            v = float(r[i_val].replace(",", "")) * scale.get(r[i_unit], 1.0)
        except ValueError:
            continue
        if not math.isfinite(v):
            continue
        nm = r[i_name].split("(")[0].split("::")[-1]
        agg[nm][0] += 1
        agg[nm][1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"# {title}", "", "ncu `--metrics gpu__time_duration.sum --clock-control none` launch list "
           "(cold-cache, serialised replay: compare shares, not absolutes).", "",
           "| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {v[0]} | {v[1] / 1e6:.3f} | {100 * v[1] / tot:.1f}% |")
    out.append(f"| total | {sum(v[0] for v in agg.values())} | {tot / 1e6:.3f} | 100% |")
    return "\n".join(out)


def launches_dram(path, title):
    lines = open(path).read().splitlines()
    start = [i for i, l in enumerate(lines) if l.startswith('"ID"')][0]
    rows = list(csv.reader(lines[start:]))
    hdr = rows[0]
    i_name, i_val = hdr.index("Kernel Name"), hdr.index("Metric Value")
    i_met, i_unit = hdr.index("Metric Name"), hdr.index("Metric Unit")
    tsc = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    bsc = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for r in rows[1:]:
        nm = r[i_name].split("(")[0].split("::")[-1]
        try:
            v = float(r[i_val].replace(",", ""))
        except ValueError:
            continue
        if r[i_met] == "gpu__time_duration.sum":
            agg[nm][0] += 1
            agg[nm][1] += v * tsc.get(r[i_unit], 1.0)
        elif r[i_met] == "dram__bytes_read.sum":
            agg[nm][2] += v * bsc.get(r[i_unit], 1e-9)
        elif r[i_met] == "dram__bytes_write.sum":
            agg[nm][3] += v * bsc.get(r[i_unit], 1e-9)
    tot = sum(v[1] for v in agg.values())
    out = [f"# {title}", "", "| kernel | launches | total ms | share | DRAM read GB | DRAM write GB | DRAM GB/s |",
           "|---|---:|---:|---:|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {v[0]} | {v[1]:.3f} | {100 * v[1] / tot:.1f}% | {v[2]:.2f} | {v[3]:.2f} | "
                   f"{(v[2] + v[3]) / v[1] * 1e3:.0f} |")
    out.append(f"| total | {sum(v[0] for v in agg.values())} | {tot:.3f} | 100% | | | |")
    return "\n".join(out)


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__average_warp_latency_issue_stalled_barrier",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "sm__cycles_elapsed.max"]


def full(path, title):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = [f"# {title}", "", f"`ncu --set full --clock-control none` capture `{path.split('/')[-1]}`.", ""]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        out += [f"## `{name.split('(')[0]}`", "", "| metric | value | unit |", "|---|---:|---|"]
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                out.append(f"| {w} | {r[i]} | {units[i]} |")
        out.append("")
    return "\n".join(out)


if __name__ == "__main__":
    mode, path, title = sys.argv[1], sys.argv[2], sys.argv[3]
    print({"launches": launches, "launches_dram": launches_dram}.get(mode, full)(path, title))
