"""Straight-line runs of the SASS listing (equal execution counts) for one kernel of an ncu report,
ranked by executed ALU-pipe warp-instructions; each with its first and last source instruction."""
import csv
import subprocess
import sys

ALU = {'LOP3', 'SHF', 'PRMT', 'IADD3', 'ISETP', 'SEL', 'FLO', 'POPC', 'LEA', 'IABS', 'PLOP3', 'P2R', 'R2P',
       'VIADD', 'IADD', 'LOP', 'BMSK', 'SGXT', 'IMNMX', 'VIMNMX', 'BREV', 'VABSDIFF4'}


def main(rep, regex, top=20):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass', '-k',
                          'regex:' + regex, '--launch-count', '1'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    i_src, i_ie = h.index('Source'), h.index('Instructions Executed')
    data = []
    for r in rows[2:]:
        try:
            n = int(r[i_ie] or 0)
        except (ValueError, IndexError):
            continue
        toks = r[i_src].split()
        op = (toks[1] if toks and toks[0].startswith('@') else toks[0] if toks else '').split('.')[0]
        data.append((n, op, r[i_src].strip()[:60]))
    half = len(data) // 2
    if len(data) % 2 == 0 and half and all(data[i][2] == data[i + half][2] for i in range(0, half, max(1, half // 50))):
        data = data[:half]
    runs, cur = [], None
    for k, (n, op, src) in enumerate(data):
        if cur and n == cur['n']:
            cur['end'] = k
            cur['alu'] += op in ALU
            cur['cnt'] += 1
            cur['last'] = src
        else:
            if cur:
                runs.append(cur)
            cur = dict(start=k, end=k, n=n, alu=int(op in ALU), cnt=1, first=src, last=src)
    runs.append(cur)
    tot_alu = sum(r['n'] * r['alu'] for r in runs) or 1
    print(f'{len(data)} instructions, ALU-pipe warp-instructions {tot_alu}')
    for r in sorted(runs, key=lambda r: -r['n'] * r['alu'])[:top]:
        print('%5.1f%% alu  lines %4d-%4d n=%4d alu=%4d exec=%7d | %s ... %s' % (
            100 * r['n'] * r['alu'] / tot_alu, r['start'], r['end'], r['cnt'], r['alu'], r['n'], r['first'][:34],
            r['last'][:34]))


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 20)
