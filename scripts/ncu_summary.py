"""Summarise ncu captures into profiles/ (run here, on the CPU box, after gpurun brings the files back).

    python scripts/ncu_summary.py full  gpurun_out/x.ncu-rep  profiles/r01_fused_cfg3.md  [--entries N] [--workload name]
    python scripts/ncu_summary.py launches gpurun_out/launches.csv profiles/r01_launches_cfg3.md
"""
import collections
import csv
import json
import os
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % (achieved occupancy)"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem/CTA"),
    ("launch__occupancy_limit_shared_mem", "occupancy limit (smem) CTAs/SM"),
    ("launch__occupancy_limit_registers", "occupancy limit (regs) CTAs/SM"),
    ("launch__grid_size", "grid"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
]

TO_BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9}
TO_MS = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}


def full(rep, out, entries=None, workload=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary: `{os.path.basename(rep)}`", ""]
    js = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        lines += [f"## {name}", "", "| metric | value | unit |", "|---|---|---|"]
        rec = {"kernel": name}
        for key, label in METRICS:
            if key in h:
                i = h.index(key)
                lines.append(f"| {label} (`{key}`) | {r[i]} | {units[i]} |")
                rec[key] = (r[i], units[i])
        rd = float(r[h.index("dram__bytes_read.sum")].replace(",", "")) * TO_BYTES[units[h.index("dram__bytes_read.sum")]]
        wr = float(r[h.index("dram__bytes_write.sum")].replace(",", "")) * TO_BYTES[units[h.index("dram__bytes_write.sum")]]
        dur = float(r[h.index("gpu__time_duration.sum")].replace(",", "")) * TO_MS[units[h.index("gpu__time_duration.sum")]]
        rec["dram_bytes"] = rd + wr
        rec["duration_ms"] = dur
        lines.append(f"| DRAM bytes per launch (read+write) | {rd + wr:.4g} | byte |")
        lines.append(f"| DRAM GB/s (cold, serialised) | {(rd + wr) / dur / 1e6:.1f} | GB/s |")
        if entries:
            lines.append(f"| DRAM bytes per plan entry | {(rd + wr) / entries:.2f} | B |")
            inst = float(r[h.index("smsp__inst_executed.sum")].replace(",", ""))
            lines.append(f"| warp instructions per plan entry | {inst / entries:.3f} | |")
        lines.append("")
        js.append(rec)
    open(out, "w").write("\n".join(lines) + "\n")
    if workload:
        # one record per (workload, kernel mode) in profiles/ncu_traffic.json: the MODE template
        # argument of k_badmm_tma<T, MP, NCH, MODE, DP> names it (1 FUSED, 7 GMID, ...)
        tr = os.path.join(os.path.dirname(out), "ncu_traffic.json")
        names = {"1": "fused", "5": "fusedx", "6": "gin", "7": "gmid", "8": "gxout", "3": "p1init"}
        try:
            recs = json.load(open(tr))
            recs = recs if isinstance(recs, list) else [recs]
        except (OSError, ValueError):
            recs = []
        for x in js:
            parts = x["kernel"].split("k_badmm_tma<")[-1].split(">")[0].split(",")
            variant = names.get(parts[3].strip(), "other") if len(parts) >= 5 else "other"
            recs = [r for r in recs if not (r.get("workload") == workload and r.get("kernel_variant") == variant)]
            recs.append({"workload": workload, "kernel_variant": variant, "kernel": x["kernel"],
                         "dram_bytes_per_launch": x["dram_bytes"], "duration_ms_cold": x["duration_ms"],
                         "source": os.path.basename(out)})
        json.dump(recs, open(tr, "w"), indent=1)
    print(open(out).read())


def launches(csvf, out):
    rows = list(csv.reader(open(csvf)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        ms = float(r[vi].replace(",", "")) * TO_MS.get(r[ui], 1e-6)
        key = r[ki].split("(")[0]
        tot[key] += ms
        cnt[key] += 1
    T = sum(tot.values())
    lines = [f"# ncu launch list: `{os.path.basename(csvf)}` (gpu__time_duration.sum, cold & serialised — compare shares)",
             "", "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"| `{k}` | {cnt[k]} | {v:.3f} | {100 * v / T:.1f}% |")
    lines.append(f"| total | {sum(cnt.values())} | {T:.3f} | |")
    open(out, "w").write("\n".join(lines) + "\n")
    print(open(out).read())


if __name__ == "__main__":
    mode, src, dst = sys.argv[1:4]
    kw = {}
    if "--entries" in sys.argv:
        kw["entries"] = float(sys.argv[sys.argv.index("--entries") + 1])
    if "--workload" in sys.argv:
        kw["workload"] = sys.argv[sys.argv.index("--workload") + 1]
    full(src, dst, **kw) if mode == "full" else launches(src, dst)
