#!/usr/bin/env python
"""Summarise the text exports of ncu runs (scripts/gpu_ncu_r2.sh) into profiles/.

    python scripts/ncu_summary_r2.py full DIR profiles/r02_ncu_full.json
    python scripts/ncu_summary_r2.py launches CSV profiles/r02_launches_X.md
"""
import csv
import glob
import io
import json
import os
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_bytes.sum",
           "sm__cycles_active.avg", "gpc__cycles_elapsed.max",
           "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
           "launch__shared_mem_per_block_dynamic"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
         "msecond": 1e6, "ns": 1, "us": 1e3, "ms": 1e6}


def num(v, unit):
    return float(str(v).replace(",", "")) * SCALE.get(unit, 1)


def full(src_dir, dst):
    res = {}
    for path in sorted(glob.glob(os.path.join(src_dir, "r02_*.raw.csv"))):
        rows = list(csv.reader(open(path)))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]
        tag = os.path.basename(path)[:-len(".raw.csv")]
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            u = dict(zip(hdr, units))
            e = {"kernel": d.get("Kernel Name", "")[:200]}
            for m in METRICS:
                if d.get(m, "") != "":
                    e[m] = f"{d[m]} {u.get(m, '')}".strip()
            try:
                e["dram_bytes_total"] = int(num(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"]) +
                                            num(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"]))
                e["duration_ns"] = num(d["gpu__time_duration.sum"], u["gpu__time_duration.sum"])
                e["dram_gbs"] = round(e["dram_bytes_total"] / e["duration_ns"], 1)
            except (KeyError, ValueError):
                pass
            res[tag] = e
    json.dump(res, open(dst, "w"), indent=1)
    print(f"wrote {dst}: {list(res)}")


def launches(src, dst):
    text = open(src).read()
    rows = list(csv.DictReader(io.StringIO(text[text.index('"ID"'):])))
    per = {}
    for r in rows:
        k = r["ID"]
        e = per.setdefault(k, {"name": r["Kernel Name"].split("(")[0].replace("void ", ""),
                               "grid": r["Grid Size"], "block": r["Block Size"]})
        e[r["Metric Name"]] = num(r["Metric Value"], r["Metric Unit"])
    ks = [per[k] for k in sorted(per, key=int)]
    total = sum(e.get("gpu__time_duration.sum", 0) for e in ks)
    out = ["| # | kernel | grid | block | time (us) | DRAM read+write (MB) | DRAM GB/s | share |",
           "|---|---|---|---|---|---|---|---|"]
    for i, e in enumerate(ks):
        t = e.get("gpu__time_duration.sum", 0)
        b = e.get("dram__bytes_read.sum", 0) + e.get("dram__bytes_write.sum", 0)
        out.append(f"| {i} | `{e['name'][:90]}` | {e['grid']} | {e['block']} | {t / 1e3:.2f} | "
                   f"{b / 1e6:.1f} | {b / t if t else 0:.0f} | {100 * t / total:.1f}% |")
    hdr = (f"# ncu launch list: `{os.path.basename(src)}`\n\n`ncu --nvtx --nvtx-include timed/ "
           f"--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
           f"--clock-control none` (bench.py's timed region only; cold-cache, serialised: compare "
           f"shares, not absolutes).  {len(ks)} launches, {total / 1e3:.1f} us total.\n\n")
    open(dst, "w").write(hdr + "\n".join(out) + "\n")
    print(f"wrote {dst}: {len(ks)} launches")


if __name__ == "__main__":
    {"full": full, "launches": launches}[sys.argv[1]](*sys.argv[2:])
