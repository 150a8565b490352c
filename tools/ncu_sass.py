"""SASS-level views of one kernel launch in an ncu report (the source page, `--print-source`):

  python tools/ncu_sass.py lines  report.ncu-rep kernel_regex [top=40] [launch_skip=0]
      executed warp-instructions per CUDA source line, heaviest first, with the ALU-pipe share
  python tools/ncu_sass.py opmix  report.ncu-rep kernel_regex
      executed-instruction mix by SASS opcode
  python tools/ncu_sass.py hot    report.ncu-rep kernel_regex [top=10]
      top stall-sample SASS lines (with the 3 preceding instructions) and the heaviest
      straight-line runs of executed instructions
  python tools/ncu_sass.py runs   report.ncu-rep kernel_regex [top=20]
      straight-line runs (equal execution counts) ranked by executed ALU-pipe instructions
  python tools/ncu_sass.py region report.ncu-rep kernel_regex [marker=FLO] [which=3]
      per-instruction counts between two occurrences of a marker opcode (one coder symbol)
"""
import collections
import csv
import re
import subprocess
import sys

ALU = {'LOP3', 'SHF', 'PRMT', 'IADD3', 'ISETP', 'SEL', 'FLO', 'POPC', 'LEA', 'IABS', 'PLOP3', 'P2R', 'R2P',
       'VIADD', 'IADD', 'LOP', 'BMSK', 'SGXT', 'IMNMX', 'VIMNMX', 'BREV', 'VABSDIFF4'}


def opcode(src):
    return re.sub(r'^@!?U?P[T0-9]+\s+', '', src.strip()).split(' ')[0].split('.')[0]


def source_page(rep, regex, what='sass', skip=0):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', what, '-k',
                          'regex:' + regex, '--launch-skip', str(skip), '--launch-count', '1'],
                         capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


def sass_rows(rep, regex):
    """[(executed, stall samples, index, source)] of the SASS listing, one copy of the function."""
    rows = source_page(rep, regex)
    k0 = 1 if len(rows) > 1 and 'Source' in rows[1] else 0
    h = rows[k0]
    i_src, i_ie = h.index('Source'), h.index('Instructions Executed')
    i_s = h.index('Warp Stall Sampling (All Samples)') if 'Warp Stall Sampling (All Samples)' in h else None
    data = []
    for r in rows[k0 + 1:]:
        try:
            data.append((int(r[i_ie] or 0), int(r[i_s] or 0) if i_s is not None else 0, len(data), r[i_src].strip()))
        except (ValueError, IndexError):
            pass
    n = len(data)                          # the page may list the function twice (several launches)
    half = n // 2
    if n % 2 == 0 and half and all(data[i][3] == data[i + half][3] for i in range(0, half, max(1, half // 50))):
        data = data[:half]
    return data


def straight_runs(data):
    runs, cur = [], None
    for n, _, k, src in data:
        if cur and n == cur['n']:
            cur.update(end=k, cnt=cur['cnt'] + 1, alu=cur['alu'] + (opcode(src) in ALU), last=src)
        else:
            if cur:
                runs.append(cur)
            cur = dict(start=k, end=k, n=n, cnt=1, alu=int(opcode(src) in ALU), first=src, last=src)
    if cur:
        runs.append(cur)
    return runs


def cmd_lines(rep, regex, top=40, skip=0):
    rows = source_page(rep, regex, 'sass,cuda', int(skip))
    res, hdr, path = [], None, None
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
            res[-1][1] += c
            if opcode(r[3]) in ALU:
                res[-1][2] += c
    tot = sum(x[1] for x in res) or 1
    talu = sum(x[2] for x in res) or 1
    print(f"total warp-instructions {tot}, ALU-pipe {talu} ({talu / tot * 100:.0f}%)")
    for (f, l, s), c, a in sorted(res, key=lambda x: -x[1])[:int(top)]:
        print(f"{c / tot * 100:5.1f}% (alu {a / talu * 100:4.1f}%) {f}:{l} {s}")


def cmd_opmix(rep, regex):
    cnt = collections.Counter()
    for n, _, _, src in sass_rows(rep, regex):
        cnt[opcode(src)] += n
    tot = sum(cnt.values()) or 1
    for op, c in cnt.most_common(25):
        print(f"{op:12s} {c:>12d} {c / tot * 100:5.1f}%")
    print('total', tot)


def cmd_hot(rep, regex, top=10):
    data = sass_rows(rep, regex)
    tot = sum(d[1] for d in data) or 1
    toti = sum(d[0] for d in data) or 1
    print(f'{len(data)} instructions, {tot} samples, {toti} warp-instructions')
    for n, s, k, src in sorted(data, key=lambda d: -d[1])[:int(top)]:
        print('%5d %6.2f%% %9d  %s' % (k, 100 * s / tot, n, src[:90]))
        for e in data[max(0, k - 3):k]:
            print('          %5d %s' % (e[2], e[3][:90]))
    print('heaviest runs (share of executed warp-instructions):')
    for r in sorted(straight_runs(data), key=lambda r: -r['n'] * r['cnt'])[:int(top)]:
        print('%5.1f%%  lines %4d-%4d n=%4d exec=%8d  %s' % (100 * r['n'] * r['cnt'] / toti, r['start'], r['end'],
                                                           r['cnt'], r['n'], r['first'][:50]))


def cmd_runs(rep, regex, top=20):
    data = sass_rows(rep, regex)
    runs = straight_runs(data)
    tot_alu = sum(r['n'] * r['alu'] for r in runs) or 1
    print(f'{len(data)} instructions, ALU-pipe warp-instructions {tot_alu}')
    for r in sorted(runs, key=lambda r: -r['n'] * r['alu'])[:int(top)]:
        print('%5.1f%% alu  lines %4d-%4d n=%4d alu=%4d exec=%7d | %s ... %s' % (
            100 * r['n'] * r['alu'] / tot_alu, r['start'], r['end'], r['cnt'], r['alu'], r['n'], r['first'][:34],
            r['last'][:34]))


def cmd_region(rep, regex, marker='FLO', which=3):
    data = sass_rows(rep, regex)
    idx = [d[2] for d in data if d[3].startswith(marker)]
    a, b = idx[int(which)], idx[int(which) + 1]
    seg = data[a:b]
    top = max(d[0] for d in seg) or 1
    print(f"region {a}..{b}: {b - a} SASS lines, {sum(d[0] for d in seg) / top:.1f} executed per pass of its "
          f"hottest line")
    for n, _, _, src in seg:
        print(f"{n:>10} {n / top:5.2f}  {src[:90]}")


if __name__ == '__main__':
    cmds = {'lines': cmd_lines, 'opmix': cmd_opmix, 'hot': cmd_hot, 'runs': cmd_runs, 'region': cmd_region}
    if len(sys.argv) < 4 or sys.argv[1] not in cmds:
        sys.exit(__doc__)
    cmds[sys.argv[1]](*sys.argv[2:])
