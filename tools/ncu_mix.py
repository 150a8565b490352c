"""Executed-instruction mix per opcode (weighted by warp executions) for one kernel of an ncu
report, optionally restricted to a line range of the SASS listing; groups ALU-pipe vs FMA-pipe
opcodes (B300_MICROARCH: IADD3/LOP3/SHF/PRMT/... on alu, IMAD/FFMA on fma)."""
import collections
import csv
import subprocess
import sys

ALU = {'LOP3', 'SHF', 'PRMT', 'IADD3', 'ISETP', 'SEL', 'FLO', 'POPC', 'LEA', 'IABS', 'PLOP3', 'P2R', 'R2P',
       'VIADD', 'IADD', 'LOP', 'BMSK', 'SGXT', 'FMNMX', 'IMNMX', 'VIMNMX', 'CSET', 'CSETP', 'BREV', 'VABSDIFF4'}
FMA = {'IMAD', 'FFMA', 'FMUL', 'FADD', 'HFMA2', 'IMUL'}


def main(rep, regex, lo=0, hi=10 ** 9):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass', '-k',
                          'regex:' + regex, '--launch-count', '1'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    i_src, i_ie = h.index('Source'), h.index('Instructions Executed')
    mix = collections.Counter()
    for k, r in enumerate(rows[2:]):
        if not (lo <= k <= hi):
            continue
        try:
            n = int(r[i_ie] or 0)
        except (ValueError, IndexError):
            continue
        toks = r[i_src].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith('@') else toks[0]
        mix[op.split('.')[0]] += n
    tot = sum(mix.values()) or 1
    alu = sum(v for k, v in mix.items() if k in ALU)
    fma = sum(v for k, v in mix.items() if k in FMA)
    print(f'total {tot} warp-inst; alu-pipe {alu} ({alu / tot:.1%}); fma-pipe {fma} ({fma / tot:.1%})')
    print(', '.join(f'{k} {v / tot:.1%}' for k, v in mix.most_common(24)))


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2], *(int(x) for x in sys.argv[3:5]))
