"""Summarise an ncu capture (.ncu-rep, `--set full`) and an ncu launch list (csv) into a text file for profiles/.

    python tools/ncu_summary.py gpurun_out/prof_chain.ncu-rep gpurun_out/launches.csv > profiles/r01_chain.txt

Reads the report with `ncu -i … --page raw/source --csv` (no GPU needed).
"""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
    "launch__block_size", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "lts__t_sector_hit_rate.pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg",
]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def raw(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, data = rows[0], rows[1], rows[2:]
    for r in data:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"== kernel {name}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:62s} {r[i]:>18s} {units[i]}")
        if "dram__bytes_read.sum" in hdr:
            def val(k):
                v = float(r[hdr.index(k)].replace(",", ""))
                u = units[hdr.index(k)]
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            print(f"  traffic (dram read+write) per launch: {val('dram__bytes_read.sum') + val('dram__bytes_write.sum'):.4g} B")


def source(rep):
    """Per kernel in the report: warp-stall samples and the SASS opcode mix (the source page repeats its header
    for every kernel)."""
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass"))))
    sections, hdr = [], None
    for r in rows:
        if r and r[0] == "Address":
            hdr = r
            sections.append((hdr, []))
        elif hdr is not None and len(r) >= len(hdr):
            sections[-1][1].append(r)
    for n, (hdr, data) in enumerate(sections):
        ix = {k: i for i, k in enumerate(hdr)}
        stalls = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
        tot, ops = Counter(), Counter()
        for r in data:
            for k in stalls:
                try:
                    tot[k] += float(r[ix[k]] or 0)
                except ValueError:
                    pass
            parts = r[1].split()
            if not parts:
                continue
            op = (parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]).split(".")[0]
            try:
                ops[op] += float(r[ix["Instructions Executed"]] or 0)
            except ValueError:
                pass
        S = sum(tot.values()) or 1
        print(f"== source section {n}: warp stall samples (share of all samples)")
        for k, v in tot.most_common(10):
            print(f"  {k:28s} {100 * v / S:5.1f}%")
        T = sum(ops.values()) or 1
        print(f"== source section {n}: SASS opcode mix (warp instructions executed, total {T:.4g})")
        for k, v in ops.most_common(20):
            print(f"  {k:10s} {v:12.4g} {100 * v / T:5.1f}%")


def launches(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    d = defaultdict(list)
    for r in rows[h + 1:]:
        if len(r) > mi:
            d[r[ki].split("(")[0]].append(float(r[mi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    print("== launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"  {len(v):4d} launches  mean {sum(v) / len(v) / 1e3:10.1f} us  share {100 * sum(v) / tot:5.1f}%  {k}")


if __name__ == "__main__":
    for a in sys.argv[1:]:
        if a.endswith(".ncu-rep"):
            raw(a)
            source(a)
        elif a.endswith(".csv"):
            launches(a)
