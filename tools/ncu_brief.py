"""Key counters and top stall reasons per kernel of an ncu report (ncu --page raw --csv)."""
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__occupancy_limit_registers',
        'launch__occupancy_limit_shared_mem', 'launch__registers_per_thread',
        'sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active',
        'sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'lts__t_sector_hit_rate.pct', 'dram__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']


def main(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    stall = [h for h in hdr if h.startswith('smsp__average_warps_issue_stalled_') and h.endswith('_per_issue_active.ratio')]
    for d in data:
        print('---', d[idx['Kernel Name']][:90], d[idx['Grid Size']])
        for w in WANT:
            if w in idx:
                print('  %-62s %s %s' % (w, d[idx[w]][:40], units[idx[w]]))
        st = sorted(((float(d[idx[h]] or 0), h) for h in stall), reverse=True)[:8]
        print('  stalls:', ', '.join('%s %.2f' % (h.replace('smsp__average_warps_issue_stalled_', '').replace(
            '_per_issue_active.ratio', ''), v) for v, h in st))


if __name__ == '__main__':
    main(sys.argv[1])
