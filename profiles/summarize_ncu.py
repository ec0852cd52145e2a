"""Summarise ncu captures into the JSON files kept under profiles/.

    python profiles/summarize_ncu.py full  <out.json> <a.ncu-rep> [...]
    python profiles/summarize_ncu.py launches <out.json> <launch-list.csv>

`full` keeps the headline metrics of each captured launch (time, DRAM bytes,
throughputs, occupancy, registers).  `launches` aggregates a
`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`
launch list per kernel (count, total/avg time, share, DRAM bytes per launch)
and writes the per-tag traffic file bench.py reads for `roofline.traffic`.
"""
from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys

KEEP = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "smsp__inst_executed.sum"]

# bench.py kernel tags of the launch-list kernel names
TAGS = {"k_mgs_tma": "mgs", "k_dia": "spmv:DIA/LibA", "k_rows_pipe": "spmv:CSR/LibA/32"}


def full(out, reps):
    res = {}
    for rep in reps:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        hdr, units = rows[0], rows[1]
        res[rep.rsplit("/", 1)[-1]] = [
            {k: (f"{v} {u}".strip()) for k, u, v in zip(hdr, units, r) if k in KEEP} for r in rows[2:]]
    json.dump(res, open(out, "w"), indent=1)


def launches(out, path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.OrderedDict()
    for r in rows[1:]:
        per.setdefault(int(r[ii]), {"name": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in per.values():
        name = d["name"].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
        a = agg[name]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    kernels = {n: {"launches": a[0], "us_total": a[1] / 1e3, "us_avg": a[1] / a[0] / 1e3,
                   "share": a[1] / tot, "dram_bytes_per_launch": a[2] / a[0]}
               for n, a in sorted(agg.items(), key=lambda x: -x[1][1])}
    traffic = {TAGS[n]: k["dram_bytes_per_launch"] for n, k in kernels.items() if n in TAGS}
    json.dump({"source": path, "launches": len(per), "kernels": kernels, "traffic_by_tag": traffic},
              open(out, "w"), indent=1)


if __name__ == "__main__":
    mode, out, *rest = sys.argv[1:]
    (full if mode == "full" else launches)(out, rest if mode == "full" else rest[0])
