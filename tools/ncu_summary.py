"""Markdown summary of an .ncu-rep (key metrics per kernel) and of an ncu
launch-list CSV (per-kernel share of device time).
usage: python tools/ncu_summary.py rep REP  |  python tools/ncu_summary.py launches CSV"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "DRAM rd"), ("dram__bytes_write.sum", "DRAM wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
        ("lts__t_sector_hit_rate.pct", "L2 hit %"), ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 thr %"),
        ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
        ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads/inst"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid")]


def rep(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ki = hdr.index("Kernel Name")
    cols = [(hdr.index(k), lab, units[hdr.index(k)]) for k, lab in KEYS if k in hdr]
    print("| kernel | " + " | ".join(f"{lab} ({u})" if u else lab for _, lab, u in cols) + " | sectors/req |")
    print("|---" * (len(cols) + 2) + "|")
    s_i = hdr.index("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum") if "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum" in hdr else None
    r_i = hdr.index("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum") if "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum" in hdr else None
    for d in data:
        name = d[ki].split("(")[0].replace("void ", "")[:60]
        spr = ""
        try:
            spr = f"{float(d[s_i]) / float(d[r_i]):.1f}"
        except Exception:
            pass
        print(f"| {name} | " + " | ".join(d[i] for i, _, _ in cols) + f" | {spr} |")


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[h + 1:]:
        if len(r) > vi:
            agg.setdefault(r[ki].split("(")[0].replace("void ", "")[:70], []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print("| kernel | launches | total ms | avg us | share |")
    print("|---|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| {k} | {len(v)} | {sum(v) / 1e6:.3f} | {sum(v) / len(v) / 1e3:.1f} | {sum(v) / tot * 100:.1f}% |")


if __name__ == "__main__":
    {"rep": rep, "launches": launches}[sys.argv[1]](sys.argv[2])
