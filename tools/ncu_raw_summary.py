"""Key counters + top stall reasons per kernel from `ncu -i X.ncu-rep --page raw --csv`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
base = ['Kernel Name', 'gpu__time_duration.sum', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'sm__inst_executed.avg.per_cycle_active',
        'smsp__inst_executed.sum', 'sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'launch__occupancy_limit_shared_mem',
        'launch__registers_per_thread', 'launch__grid_size', 'launch__block_size']
keys = [k for k in hdr if k.startswith('smsp__average_warps_issue_stalled') and k.endswith('per_issue_active.ratio')]
for r in rows[2:]:
    print('----')
    for w in base:
        if w in hdr:
            i = hdr.index(w)
            print('  %-66s %s %s' % (w, r[i][:60], units[i]))
    st = []
    for k in keys:
        v = r[hdr.index(k)]
        try:
            st.append((float(v), k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')))
        except ValueError:
            pass
    print('  stalls (warps per issue):', ', '.join('%s %.2f' % (k, v) for v, k in sorted(st, reverse=True)[:7]))
