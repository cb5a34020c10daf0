"""Summarise ncu captures (gpurun_out/*.ncu-rep, launch-list CSVs) into profiles/.

    python profiles/summarize.py <tag> <rep> [<rep> ...] [--launches <csv>]

Writes profiles/<tag>_ncu.json (key metrics per captured kernel) and, with
--launches, profiles/<tag>_launches.csv (our kernels only + a per-kernel
aggregate).  Reads the reports with `ncu -i ... --page raw --csv`.
"""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

HERE = os.path.dirname(os.path.abspath(__file__))
METRICS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "nvlrx__bytes.sum", "nvltx__bytes.sum", "sm__cycles_elapsed.avg.per_second",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True, capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = {"value": vals[i], "unit": units[i]}
        res.append(d)
    return res


OUR_KERNELS = ("kvm::", "migrate_bulk_kernel", "migrate_ldg_kernel", "reprefill_pair_kernel", "reprefill_kernel",
               "decode_gqa_kernel", "decode_combine_kernel", "wait_flag_kernel", "rope_table_kernel")


def _ours(name):
    return any(k in name for k in OUR_KERNELS)


def launches(path, tag):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[h]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    ours = [r for r in rows[h + 1:] if _ours(r[ki])]
    agg = defaultdict(list)
    for r in rows[h + 1:]:
        agg[r[ki]].append(float(r[vi].replace(",", "")))
    with open(os.path.join(HERE, f"{tag}_launches.csv"), "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["kernel", "launches", "mean_ns", "total_ns", "ours"])
        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
            w.writerow([k, len(v), round(sum(v) / len(v), 1), round(sum(v)), _ours(k)])
        w.writerow([])
        w.writerow(["# per-launch list (ours)"])
        for r in ours:
            w.writerow([r[ki], 1, r[vi], r[vi], True])


def main():
    tag, args = sys.argv[1], sys.argv[2:]
    reps, lcsv = [], None
    while args:
        a = args.pop(0)
        if a == "--launches":
            lcsv = args.pop(0)
        else:
            reps.append(a)
    summary = {}
    for rep in reps:
        summary[os.path.basename(rep)] = raw(rep)
    with open(os.path.join(HERE, f"{tag}_ncu.json"), "w") as fh:
        json.dump(summary, fh, indent=1)
    if lcsv:
        launches(lcsv, tag)


if __name__ == "__main__":
    main()
