"""Executed instructions per CUDA source line (SASS correlated) for the first launch of one
kernel in an ncu report, heaviest first.

  python tools/ncu_lines.py report.ncu-rep kernel_regex [top] [launch_skip]
"""
import csv
import re
import subprocess
import sys


def main(rep, regex, top=40, skip=0):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass,cuda', '-k',
                          'regex:' + regex, '--launch-skip', str(skip), '--launch-count', '1'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    res, hdr, path = [], None, None
    alu = set('LOP3 SHF ISETP PRMT IADD3 SEL LEA VIADD FLO POPC BREV VIMNMX IMNMX'.split())
    for r in rows:
        if not r:
            continue
        if r[0] == 'File Path':
            path = r[1].split('/')[-1]
            continue
        if r[0] == 'Line No':
            hdr = r
            ii = hdr.index('Instructions Executed')
            continue
        if hdr is None:
            continue
        if r[0] != '':
            res.append([(path, r[0], r[1].strip()[:90]), 0, 0])
        elif res:
            try:
                c = int(r[ii] or 0)
            except ValueError:
                continue
            op = re.sub(r'^@!?U?P[T0-9]+\s+', '', r[3].strip()).split(' ')[0].split('.')[0]
            res[-1][1] += c
            if op in alu:
                res[-1][2] += c
    tot = sum(x[1] for x in res) or 1
    talu = sum(x[2] for x in res) or 1
    print(f"total warp-instructions {tot}, ALU-pipe {talu} ({talu / tot * 100:.0f}%)")
    res.sort(key=lambda x: -x[1])
    for (f, l, s), c, a in res[:top]:
        print(f"{c / tot * 100:5.1f}% (alu {a / talu * 100:4.1f}%) {f}:{l} {s}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40,
         int(sys.argv[4]) if len(sys.argv) > 4 else 0)
