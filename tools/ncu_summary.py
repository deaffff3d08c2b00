"""Summarise an ncu raw CSV export (ncu -i X.ncu-rep --page raw --csv)."""
import csv
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum',
        'smsp__inst_executed.sum', 'sm__inst_executed_pipe_fp64.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum', 'l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum',
        'launch__registers_per_thread', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__thread_inst_executed_per_inst_executed.ratio', 'launch__grid_size', 'launch__block_size']


def main(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index('Kernel Name')] if 'Kernel Name' in hdr else '?'
        print('kernel:', name[:90])
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                print(f'  {w} = {vals[i]} {units[i]}')
        st = [(h, vals[i]) for i, h in enumerate(hdr)
              if h.startswith('smsp__average_warp_latency_issue_stalled') and h.endswith('.ratio')]
        def num(x):
            try:
                return float(x.replace(',', ''))
            except ValueError:
                return 0.0
        st = sorted(st, key=lambda x: -num(x[1]))[:10]
        for h, v in st:
            print('  stall', h.replace('smsp__average_warp_latency_issue_stalled_', ''), v)


if __name__ == '__main__':
    main(sys.argv[1])
