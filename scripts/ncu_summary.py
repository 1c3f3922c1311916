#!/usr/bin/env python
"""Summarise ncu outputs brought back from gpurun into profiles/.

    python scripts/ncu_summary.py launches gpurun_out/launches_vgg.csv profiles/r01_launches_vgg.md
    python scripts/ncu_summary.py full profiles/r01_ncu_full.json gpurun_out/prof_*.ncu-rep
    python scripts/ncu_summary.py traffic profiles/r01_ncu_full.json profiles/ncu_traffic.json \
        vgg_pools=prof_pool_vgg1 pl5=prof_pool_pl5 ...
"""
import csv
import io
import json
import os
import subprocess
import sys

OURS = ("pool_", "transpose2d", "permute4d", "softmax_", "row_max", "row_sum", "sub_rowvec",
        "exp_kernel", "scale_rowvec", "conv", "gemm", "lcnn")
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "launch__occupancy_limit_registers", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
           "lts__t_bytes.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio",
           "launch__shared_mem_per_block_dynamic", "launch__shared_mem_per_block_static"]


def ours(name):
    return any(k in name for k in OURS) and "at::" not in name


def launches(src, dst):
    text = open(src).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    mine = [r for r in rows if ours(r["Kernel Name"]) and
            r.get("Metric Name", "gpu__time_duration.sum") == "gpu__time_duration.sum"]
    scale = {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6}
    for r in mine:  # normalise to ns
        r["Metric Value"] = str(float(r["Metric Value"].replace(",", "")) *
                                scale.get(r.get("Metric Unit", "nsecond"), 1.0))
    total = sum(float(r["Metric Value"]) for r in mine)
    out = ["| # | kernel | grid | block | time (us) | share of our launches |", "|---|---|---|---|---|---|"]
    for i, r in enumerate(mine):
        t = float(r["Metric Value"]) / 1e3
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        out.append(f"| {i} | `{name}` | {r['Grid Size']} | {r['Block Size']} | {t:.2f} | "
                   f"{100 * t * 1e3 / total:.1f}% |")
    hdr = (f"# ncu launch list: `{os.path.basename(src)}`\n\n`ncu --metrics gpu__time_duration.sum "
           f"--clock-control none` (cold-cache, serialised: compare shares, not absolutes).  "
           f"{len(mine)} of our launches, {total / 1e3:.1f} us total; torch RNG/fill kernels "
           f"of the setup are excluded.\n\n")
    with open(dst, "w") as f:
        f.write(hdr + "\n".join(out) + "\n")
    print(f"wrote {dst}: {len(mine)} launches")


def full(dst, reps):
    res = {}
    for rep in reps:
        csvtext = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                 text=True).stdout
        rows = list(csv.reader(io.StringIO(csvtext)))
        if len(rows) < 3:
            continue
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            entry = {"kernel": d.get("Kernel Name", "")[:160]}
            for m in METRICS:
                if m in d and d[m] != "":
                    entry[m] = f"{d[m]} {units[hdr.index(m)]}".strip()
            try:
                rd = _bytes(d["dram__bytes_read.sum"], units[hdr.index("dram__bytes_read.sum")])
                wr = _bytes(d["dram__bytes_write.sum"], units[hdr.index("dram__bytes_write.sum")])
                entry["dram_bytes_total"] = int(rd + wr)
            except (KeyError, ValueError):
                pass
            res[os.path.basename(rep).replace(".ncu-rep", "")] = entry
    with open(dst, "w") as f:
        json.dump(res, f, indent=1)
    print(f"wrote {dst}: {len(res)} kernels")


def _bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}[unit]
    return float(v.replace(",", "")) * scale


def traffic(full_json, dst, pairs):
    data = json.load(open(full_json))
    out = json.load(open(dst)) if os.path.exists(dst) else {}
    for p in pairs:
        wl, rep = p.split("=")
        if rep in data and "dram_bytes_total" in data[rep]:
            out[wl] = data[rep]["dram_bytes_total"]
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    print(f"wrote {dst}: {out}")


def sections(dst_prefix, details):
    """`ncu --page details --csv` files -> {section: {metric: "value unit"}} JSON."""
    keep = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Compute Workload Analysis",
            "Launch Statistics", "Occupancy", "Warp State Statistics")
    for path in details:
        rows = list(csv.reader(open(path)))
        if not rows:
            continue
        hdr = rows[0]
        ix = {h: i for i, h in enumerate(hdr)}
        out = {}
        for r in rows[1:]:
            sec = r[ix["Section Name"]]
            if sec in keep:
                out.setdefault(sec, {})[r[ix["Metric Name"]]] = \
                    f"{r[ix['Metric Value']]} {r[ix['Metric Unit']]}".strip()
        name = os.path.basename(path).replace("_details.csv", "")
        dst = f"{dst_prefix}{name}_sections.json"
        with open(dst, "w") as f:
            json.dump(out, f, indent=1)
        print(f"wrote {dst}")


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "launches":
        launches(sys.argv[2], sys.argv[3])
    elif cmd == "full":
        full(sys.argv[2], sys.argv[3:])
    elif cmd == "sections":
        sections(sys.argv[2], sys.argv[3:])
    elif cmd == "traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4:])
