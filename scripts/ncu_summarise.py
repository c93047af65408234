"""Summarise `ncu --set full` reports into the JSON shape of profiles/r01_full_capture_metrics.json.

usage: python scripts/ncu_summarise.py OUT.json name=path.ncu-rep[:note] ...
Reads each report with `ncu -i REP --page raw --csv` and keeps the metrics the profiles cite.
"""
import csv
import io
import json
import subprocess
import sys

KEEP = [
    "Kernel Name", "launch__grid_size", "launch__block_size", "gpu__time_duration.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "smsp__inst_executed.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, first = rows[0], rows[1], rows[2]
    return {k: [first[hdr.index(k)], units[hdr.index(k)]] for k in KEEP if k in hdr}


def main():
    dst = sys.argv[1]
    res = {}
    for arg in sys.argv[2:]:
        name, rest = arg.split("=", 1)
        rep, _, note = rest.partition(":")
        try:
            res[name] = summarise(rep)
        except Exception as e:  # a missing capture is reported, not fatal
            res[name] = {"error": str(e)[:200]}
        if note:
            res[name]["note"] = [note, ""]
    with open(dst, "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
