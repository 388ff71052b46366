"""Summarise an .ncu-rep (raw page) into the few numbers the roofline needs.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--grep REGEX]
"""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "lts__t_bytes.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warp_latency_issue_stalled", "launch__shared_mem_per_block_dynamic",
]


def main():
    rep = sys.argv[1]
    extra = None
    if "--grep" in sys.argv:
        extra = re.compile(sys.argv[sys.argv.index("--grep") + 1])
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        print("----")
        for h, u, v in zip(hdr, units, r):
            if h in KEYS or (extra and extra.search(h)):
                print(f"{h} = {v} {u}")


if __name__ == "__main__":
    main()
