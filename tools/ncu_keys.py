"""Print the stall / throughput metrics of every kernel in an ncu report (raw page)."""
import csv, subprocess, sys
rows = list(csv.reader(subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()))
h = rows[0]
pick = [k for k in h if ("issue_stalled" in k and "per_issue_active" in k and "not_issued" not in k)]
keys = ['gpu__time_duration.sum', 'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum', 'sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'sm__cycles_elapsed.max']
for r in rows[2:]:
    d = dict(zip(h, r))
    print(d['Kernel Name'][:80])
    for k in keys:
        print('  ', k, d.get(k), rows[1][h.index(k)] if k in h else '')
    st = sorted(((float(d[k]), k) for k in pick if d[k] not in ('', 'n/a')), reverse=True)[:7]
    for v, k in st:
        print('   stall', k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''), round(v, 3))
