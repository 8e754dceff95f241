#!/usr/bin/env python
"""Summarises ncu output into profiles/ (tracked):

    python tools/ncu_summary.py --tag r01 --launches gpurun_out/launches_s2.csv \
        --rep gpurun_out/prof_price_s2.ncu-rep --rep gpurun_out/prof_update_s2.ncu-rep

* the launch list (``ncu --metrics gpu__time_duration.sum``, cold-cache and
  serialised) -> per-kernel launch count, total and mean duration, share;
* each ``--set full`` capture -> duration, DRAM bytes read/written (the bench's
  ``roofline.traffic``), DRAM throughput, occupancy, top warp stalls.

Writes profiles/<tag>_ncu_summary.json. bench.py reads ``traffic`` from it.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def kname(full: str) -> str:
    return full.split("::")[-1].split("(")[0]


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[i]
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[i + 1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3}.get(d["Metric Unit"], 1e-3)
        a = agg[kname(d["Kernel Name"])]
        a[0] += 1
        a[1] += float(d["Metric Value"].replace(",", "")) * scale
    tot = sum(v[1] for v in agg.values()) or 1.0
    return {k: {"launches": v[0], "us_total": round(v[1], 1), "us_mean": round(v[1] / v[0], 2),
                "share": round(v[1] / tot, 4)} for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])}


KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__bytes.sum.per_second": "dram_bw",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__warps_active.avg.per_cycle_active": "warps_per_sm",
    "sm__cycles_active.avg": "sm_cycles_active",
    "gpc__cycles_elapsed.max": "cycles_elapsed",
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3,
        "byte/s": 1, "Kbyte/s": 1e3, "Mbyte/s": 1e6, "Gbyte/s": 1e9, "Tbyte/s": 1e12}


def capture(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        e = {"kernel": kname(d["Kernel Name"])}
        for k, short in KEYS.items():
            if k in d and d[k] != "":
                v = float(d[k].replace(",", ""))
                e[short] = v * UNIT.get(units[hdr.index(k)], 1)
        stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace(
            "_per_issue_active.ratio", ""): float(v.replace(",", "") or 0)
            for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_")
            and k.endswith("_per_issue_active.ratio")}
        e["top_stalls_cycles_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:5])
        samp = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", "") or 0)
                for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                and not k.endswith("_not_issued")}
        tot = sum(samp.values()) or 1.0
        e["top_stalls_pc_samples_share"] = {k: round(v / tot, 3) for k, v in
                                            sorted(samp.items(), key=lambda kv: -kv[1])[:8]}
        if "dram_read" in e and "dram_write" in e:
            e["traffic_bytes"] = e["dram_read"] + e["dram_write"]
        if "duration" in e and "traffic_bytes" in e:
            e["traffic_gbs"] = round(e["traffic_bytes"] / e["duration"] / 1e9, 1)
        e["source"] = os.path.basename(path)
        res.append(e)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    out = {"tag": a.tag, "note": a.note}
    if a.launches:
        out["launch_list"] = launches(a.launches)
        out["launch_list_source"] = os.path.basename(a.launches)
    caps = []
    for r in a.rep:
        caps += capture(r)
    names = [c["kernel"] for c in caps]
    out["captures"] = {(c["kernel"] if names.count(c["kernel"]) == 1 else f'{c["kernel"]}@{c["source"]}'): c
                       for c in caps}
    path = os.path.join(ROOT, "profiles", f"{a.tag}_ncu_summary.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(path)
    print(json.dumps(out, indent=1)[:3000])


if __name__ == "__main__":
    main()
