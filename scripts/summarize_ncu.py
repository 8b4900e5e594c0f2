"""Summarise ncu outputs into profiles/ JSON.

  launches <csv> <out.json> <command>   : ncu --metrics gpu__time_duration.sum --csv launch list
                                          -> per-kernel launches, total us, share
  full <rep> <out.json> <command>       : ncu --set full report -> key metrics per launch
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "lts__t_sector_hit_rate.pct",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"]


def launches(path, out, command):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "")
        us = v / 1e3 if unit in ("ns", "nsecond") else v * 1e3 if unit in ("ms", "msecond") else v
        k = d["Kernel Name"]
        agg[k][0] += 1
        agg[k][1] += us
    tot = sum(v[1] for v in agg.values()) or 1.0
    ks = sorted(agg.items(), key=lambda kv: -kv[1][1])
    json.dump({"command": command,
               "note": "cold-cache, serialised launches under ncu: compare shares, not absolutes",
               "kernels": [{"kernel": k, "launches": n, "total_us": round(us, 1),
                            "share": round(us / tot, 4)} for k, (n, us) in ks]},
              open(out, "w"), indent=1)


def full(rep, out, command):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = (r[i] + " " + units[i]).strip()
        res.append(d)
    json.dump({"command": command, "launches": res}, open(out, "w"), indent=1)


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](*sys.argv[2:5])
