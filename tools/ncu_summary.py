#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) and an
ncu --set full report into profiles/<tag>_*.{md,json}.

  python tools/ncu_summary.py --tag r01 --launches gpurun_out/launches.csv \
      --report gpurun_out/prof.ncu-rep --packets 100000000
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__t_sectors_srcunit_tex_op_red.sum", "lts__t_sectors_srcunit_tex_op_red_lookup_hit.sum",
    "lts__t_sectors_srcunit_ltcfabric.sum", "lts__d_atomic_input_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "l1tex__t_requests_pipe_lsu_mem_global_op_red.sum",
    "sm__inst_issued.avg.pct_of_peak_sustained_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed_op_shared_atom.sum",
    "lts__t_sectors_op_read.sum", "lts__t_sectors_op_write.sum", "lts__t_sectors_op_red.sum",
]


def to_ns(v, unit):
    v = float(v.replace(",", ""))
    return v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(unit, 1)


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in data:
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += to_ns(r[vi], r[ui])
    return agg


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for m in METRICS:
            if m in h:
                i = h.index(m)
                d[m] = r[i] + (" " + units[i] if units[i] else "")
        res.append(d)
    return res


def num(s):
    return float(s.split()[0].replace(",", ""))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--report")
    ap.add_argument("--packets", type=int, default=100_000_000)
    ap.add_argument("--out", default="profiles")
    a = ap.parse_args()
    os.makedirs(a.out, exist_ok=True)
    md = ["# ncu summary %s\n" % a.tag]
    js = {}
    if a.launches:
        agg = launches(a.launches)
        tot = sum(v for _, v in agg.values())
        md.append("## Launch list (`--metrics gpu__time_duration.sum --clock-control none`; cold, serialised: compare shares)\n")
        md.append("| kernel | launches | total us | avg us | share |\n|---|---|---|---|---|")
        js["launches"] = {}
        for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
            md.append("| %s | %d | %.1f | %.1f | %.1f%% |" % (k, n, v / 1e3, v / 1e3 / n, 100 * v / tot))
            js["launches"][k] = dict(n=n, total_us=v / 1e3)
        md.append("")
    if a.report:
        res = full(a.report)
        js["full"] = res
        md.append("## `ncu --set full` (one launch per kernel)\n")
        for d in res:
            md.append("### %s\n" % d["kernel"])
            for m in METRICS:
                if m in d:
                    md.append("- `%s` = %s" % (m, d[m]))
            md.append("")
        scans = [d for d in res if "k_scan" in d["kernel"]]
        if scans:
            d = scans[0]
            scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
            def mbytes(v):
                x, u = v.split()[0], v.split()[1]
                return float(x.replace(",", "")) * scale[u]
            mb, wb = mbytes(d["dram__bytes_read.sum"]), mbytes(d["dram__bytes_write.sum"])
            per = (mb + wb) * 1e6 / a.packets
            kname = d["kernel"].split("::")[-1].split("<")[0]
            with open(os.path.join(a.out, "scan_traffic.json"), "w") as f:
                json.dump({"source": "%s %s ncu --set full" % (a.tag, d["kernel"]), "kernel": kname,
                           "packets_per_launch": a.packets, "dram_bytes_per_launch": (mb + wb) * 1e6,
                           "dram_bytes_per_packet": per}, f, indent=1)
    if a.report:
        # per-kernel counters bench.py reports next to its live timings (roofline.traffic,
        # the scan's random-access evidence, k_fold's DRAM bytes)
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        kt = {"source": "%s ncu --set full --clock-control none (one launch per kernel)" % a.tag,
              "packets_per_scan_launch": a.packets, "kernels": {}}
        for d in res:
            short = d["kernel"].split("::")[-1].split("<")[0].split("(")[0].strip()
            if short in kt["kernels"]:
                continue
            e = {"instantiation": d["kernel"]}
            for key, m in (("dram_read_bytes", "dram__bytes_read.sum"), ("dram_write_bytes", "dram__bytes_write.sum")):
                if m in d:
                    v, u = d[m].split()[0], d[m].split()[1]
                    e[key] = float(v.replace(",", "")) * scale[u]
            for key, m in (("l2_hit_rate_pct", "lts__t_sector_hit_rate.pct"),
                           ("lts_throughput_pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
                           ("dram_throughput_pct", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                           ("l1_shared_pipe_pct", "l1tex__throughput.avg.pct_of_peak_sustained_active"),
                           ("issue_pct", "sm__inst_issued.avg.pct_of_peak_sustained_active"),
                           ("shared_wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
                           ("shared_atom_wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum"),
                           ("shared_bank_conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
                           ("lts_sectors_read", "lts__t_sectors_op_read.sum"),
                           ("lts_sectors_write", "lts__t_sectors_op_write.sum"),
                           ("lts_sectors_red", "lts__t_sectors_op_red.sum"),
                           ("inst_executed", "smsp__inst_executed.sum"),
                           ("duration_us", "gpu__time_duration.sum")):
                if m in d:
                    e[key] = num(d[m])
            if "dram_read_bytes" in e and "dram_write_bytes" in e:
                e["dram_bytes"] = e["dram_read_bytes"] + e["dram_write_bytes"]
            kt["kernels"][short] = e
        with open(os.path.join(a.out, "kernel_traffic.json"), "w") as f:
            json.dump(kt, f, indent=1)
    with open(os.path.join(a.out, "%s_ncu_summary.md" % a.tag), "w") as f:
        f.write("\n".join(md) + "\n")
    with open(os.path.join(a.out, "%s_ncu_summary.json" % a.tag), "w") as f:
        json.dump(js, f, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
