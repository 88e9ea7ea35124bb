"""profiles/ncu_traffic.json from an `ncu --set full` capture of one bench
step (tools/ncu_step.py): per kernel of the query — horizons, window
descriptors, mining — its duration, DRAM bytes and executed warp
instructions.  bench.py reads it for roofline.traffic, the issue roofline and
hbm_pct_of_peak (ncu DRAM bytes over the query's kernels).
usage: python tools/ncu_query_json.py REP.ncu-rep [out.json] [note]"""
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2310_02800_b200 import motifs as M  # noqa: E402

METRICS = {"gpu__time_duration.sum": "time_ms", "dram__bytes_read.sum": "dram_read",
           "dram__bytes_write.sum": "dram_write", "smsp__inst_executed.sum": "warp_inst",
           "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
           "lts__t_sector_hit_rate.pct": "l2_hit_pct", "sm__warps_active.avg.pct_of_peak_sustained_active":
           "occupancy_pct", "smsp__thread_inst_executed_per_inst_executed.ratio": "threads_per_inst",
           "launch__registers_per_thread": "regs"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1,
         "ns": 1e-6, "us": 1e-3, "ms": 1, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "inst": 1, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9}


def code(mot):   # tmg::motif_code: L | u_i << (3 + 6i) | v_i << (6 + 6i), vertices by first appearance
    lab, u, v = {}, [], []
    for a, b in mot:
        for x in (a, b):
            lab.setdefault(x, len(lab))
        u.append(lab[a]); v.append(lab[b])
    c = len(mot)
    for i in range(len(mot)):
        c |= u[i] << (3 + 6 * i) | v[i] << (6 + 6 * i)
    return c


CODES = {code(m): n for n, m in M.NAMED.items()}
MODES = {0: "kCount", 1: "kEnum", 4: "kCountPfx", 5: "kResume", 6: "kCountSib"}


def main(rep, out=os.path.join(ROOT, "profiles", "ncu_traffic.json"), note=""):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ki = hdr.index("Kernel Name")
    kernels = []
    for d in data:
        name = d[ki]
        k = {"name": name.split("(")[0].replace("void ", "")}
        for met, key in METRICS.items():
            if met in hdr:
                i = hdr.index(met)
                try:
                    k[key] = float(d[i].replace(",", "")) * SCALE.get(units[i], 1)
                except ValueError:
                    pass
        k["dram_bytes"] = k.pop("dram_read", 0) + k.pop("dram_write", 0)
        mm = re.search(r"PlanC<(\d+)(?:ul?)?, (?:false|0)>, (\d+)>", name.replace("(unsigned long)", ""))
        if mm:
            k["motif"] = CODES.get(int(mm.group(1)), mm.group(1))
            k["mode"] = MODES.get(int(mm.group(2)), mm.group(2))
        kernels.append(k)
    doc = {"config": "C4", "round": 2, "kernels": kernels,
           "query_dram_bytes": sum(k["dram_bytes"] for k in kernels),
           "query_time_ms_serialised": sum(k.get("time_ms", 0) for k in kernels),
           "source": note or ("ncu --set full --clock-control none --import-source on -k regex:'mine_kernel|k_horizon|k_hrank' "
                                "python tools/ncu_step.py (one bench query on C4)")}
    json.dump(doc, open(out, "w"), indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
