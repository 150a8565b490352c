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


def main(rep, regex, lo=0, hi=10 ** 9, skip=0):
    """The source page lists every SASS instruction twice (its SASS and its CUDA-correlated rows):
    instructions are counted once per address, so the total equals smsp__inst_executed.sum."""
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass', '-k',
                          'regex:' + regex, '--launch-skip', str(skip), '--launch-count', '1'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi_row = next(i for i, r in enumerate(rows) if 'Source' in r and 'Instructions Executed' in r)
    h = rows[hi_row]
    i_src, i_ie, i_ad = h.index('Source'), h.index('Instructions Executed'), h.index('Address')
    mix = collections.Counter()
    seen = set()
    k = -1
    for r in rows[hi_row + 1:]:
        if len(r) <= i_ie or not r[i_ad].startswith('0x') or r[i_ad] in seen:
            continue
        seen.add(r[i_ad])
        k += 1
        if not (lo <= k <= hi):
            continue
        try:
            n = int(r[i_ie] or 0)
        except ValueError:
            continue
        toks = r[i_src].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith('@') else toks[0]
        mix[op.split('.')[0]] += n
    tot = sum(mix.values()) or 1
    alu = sum(v for k2, v in mix.items() if k2 in ALU)
    fma = sum(v for k2, v in mix.items() if k2 in FMA)
    print(f'total {tot} warp-inst; alu-pipe {alu} ({alu / tot:.1%}); fma-pipe {fma} ({fma / tot:.1%})')
    print(', '.join(f'{k2} {v / tot:.1%}' for k2, v in mix.most_common(24)))
    return tot, alu, fma


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2], *(int(x) for x in sys.argv[3:6]))
