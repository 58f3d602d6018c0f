"""SASS opcode mix (executed warp instructions and stall samples) of one kernel in an ncu report.

    python tools/ncu_opmix.py report.ncu-rep
"""
import collections
import csv
import subprocess
import sys


def main(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout.splitlines()[1:]
    r = list(csv.reader(out))
    h, d = r[0], r[1:]
    ie, src, smp = h.index('Instructions Executed'), h.index('Source'), h.index('Warp Stall Sampling (All Samples)')
    c, s = collections.Counter(), collections.Counter()
    for x in d:
        op = x[src].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith('@') else op[0]
        c[o.split('.')[0]] += int(x[ie] or 0)
        s[o.split('.')[0]] += int(x[smp] or 0)
    tot = sum(c.values())
    for o, v in c.most_common(25):
        print('%-10s %12d %5.1f%%  samples %d' % (o, v, 100 * v / tot, s[o]))


if __name__ == '__main__':
    main(sys.argv[1])
