"""Print the issue / pipe / stall / memory-pipe metrics of one kernel in an ncu report.

    python tools/ncu_detail.py report.ncu-rep [kernel-index]
"""
import csv
import subprocess
import sys

KEYS = ('smsp__inst_executed.sum', 'smsp__issue_active.avg.pct', 'sm__inst_executed_pipe_lsu.avg.pct',
        'sm__inst_executed_pipe_alu.avg.pct', 'sm__inst_executed_pipe_fma.avg.pct',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'l1tex__data_pipe_lsu_wavefronts_mem_shared_op',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op', 'l1tex__throughput.avg.pct',
        'lts__throughput.avg.pct', 'dram__throughput.avg.pct', 'gpu__time_duration.sum',
        'sm__warps_active.avg.pct', 'l1tex__lsuin_requests.avg.pct', 'smsp__sass_inst_executed_op',
        'l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum', 'l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'dram__bytes_read.sum')


def main(rep, k=0):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u, row = r[0], r[1], r[2 + k]
    print(row[h.index('Kernel Name')][:90])
    stalls = []
    for i, name in enumerate(h):
        v = row[i].replace(',', '')
        try:
            f = float(v)
        except ValueError:
            continue
        if name.startswith('smsp__average_warps_issue_stalled_') and name.endswith('_per_issue_active.ratio'):
            stalls.append((f, name[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]))
        elif any(name.startswith(kk) for kk in KEYS) and not name.endswith(('.max', '.min')) \
                and '.max.' not in name and '.min.' not in name and f != 0:
            print('  %-80s %-10s %s' % (name, u[i], v))
    print('  stalls per issue:', ', '.join('%s %.2f' % (n, f) for f, n in sorted(stalls, reverse=True)[:8]))


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
