"""Condense an `ncu --set full` report into per-kernel JSON (profiles/*_ncu_kernels.json).

    python tools/ncu_summary.py report.ncu-rep > profiles/rXX_ncu_kernels.json

DRAM bytes are reported in GB (ncu's raw unit scaled), times in ms.  bench.py reads the
committed summary to fill `roofline.traffic` (dram read + write of the phase's kernels).
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]
SCALE = {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        e = {"kernel": d["Kernel Name"].split("(")[0].replace("void ", "")}
        for m in METRICS:
            if m not in d or d[m] in ("", "n/a"):
                continue
            u = units[head.index(m)]
            try:
                v = float(d[m].replace(",", ""))
            except ValueError:
                continue
            if u in SCALE:
                v *= SCALE[u]
                m = m + (" [GB]" if "byte" in u.lower() else " [ms]")
            e[m] = v
        res.append(e)
    return res


if __name__ == "__main__":
    # usage: ncu_summary.py report.ncu-rep [steps] [workload description]
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    work = sys.argv[3] if len(sys.argv) > 3 else ""
    json.dump({"workload": work, "steps": steps, "kernels": summarise(sys.argv[1])}, sys.stdout, indent=1)
    print()
