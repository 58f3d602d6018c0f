"""Summarise an ncu report: per-kernel duration, DRAM/L2 traffic, occupancy, stalls."""
import csv
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'lts__t_sectors_srcunit_tex_op_write.sum',
        'lts__t_sectors_srcunit_tex_op_atom.sum', 'lts__t_sectors_srcunit_tex_op_red.sum',
        'l1tex__t_sector_hit_rate.pct', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'dram__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__registers_per_thread',
        'smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct',
        'smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct',
        'smsp__warp_issue_stalled_barrier_per_warp_active.pct',
        'smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct',
        'smsp__warp_issue_stalled_membar_per_warp_active.pct',
        'smsp__warp_issue_stalled_drain_per_warp_active.pct']


def rows(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[1], r[2:]


def main(rep):
    hdr, units, data = rows(rep)
    ki = hdr.index('Kernel Name')
    for r in data:
        print('---', r[ki][:100])
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                print('   %-70s %-8s %s' % (w, units[i], r[i]))


if __name__ == '__main__':
    main(sys.argv[1])
