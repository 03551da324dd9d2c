"""Summarise an `ncu --set full` report into the profiles/*.json format:
one entry per captured launch with the metrics the round's tables quote.
python tools/ncu_summary.py REPORT.ncu-rep "how it was captured" > profiles/X.json"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "lts__t_sector_hit_rate.pct", "launch__grid_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def main():
    rep, how = sys.argv[1], sys.argv[2]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head = rows[0]
    kernels = []
    for r in rows[2:]:
        if len(r) != len(head):
            continue
        e = {"kernel": r[head.index("Kernel Name")].split("(")[0]}
        for m in METRICS:
            if m in head:
                e[m] = r[head.index(m)]
        t = float(e["gpu__time_duration.sum"]) * 1e-6  # us -> s
        rd, wr = float(e["dram__bytes_read.sum"]), float(e["dram__bytes_write.sum"])  # MB
        e["hbm_gbs"] = round((rd + wr) * 1e6 / t / 1e9, 1) if t > 0 else None
        kernels.append(e)
    json.dump({"how": how, "units": "time us, dram MB, rates %, hbm_gbs = (dram read + write) / duration",
               "kernels": kernels}, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
