"""Top stall-sample SASS lines (with the 4 preceding instructions) and the heaviest straight-line
runs of executed instructions for one kernel of an ncu report."""
import csv
import subprocess
import sys


def main(rep, regex, top=10):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass', '-k',
                          'regex:' + regex, '--launch-count', '1'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    i_src, i_s, i_ie = h.index('Source'), h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed')
    data = []
    for k, r in enumerate(rows[2:]):
        try:
            data.append((int(r[i_s] or 0), int(r[i_ie] or 0), k, r[i_src].strip()[:90]))
        except (ValueError, IndexError):
            pass
    # the source page may list the function twice (several launches): keep the first copy
    n = len(data)
    for half in (n // 2,):
        if n % 2 == 0 and all(data[i][3] == data[i + half][3] for i in range(0, half, max(1, half // 50))):
            data = data[:half]
    tot = sum(d[0] for d in data) or 1
    toti = sum(d[1] for d in data) or 1
    print(f'{len(data)} instructions, {tot} samples, {toti} warp-instructions')
    for d in sorted(data, reverse=True)[:top]:
        print('%5d %6.2f%% %9d  %s' % (d[2], 100 * d[0] / tot, d[1], d[3]))
        for e in data[max(0, d[2] - 3):d[2]]:
            print('          %5d %s' % (e[2], e[3]))
    runs, cur = [], None
    for d in data:
        if cur and d[1] == cur[1]:
            cur[2] += 1
            cur[4] = d[2]
        else:
            if cur:
                runs.append(cur)
            cur = [d[2], d[1], 1, d[3], d[2]]
    runs.append(cur)
    print('heaviest runs (share of executed warp-instructions):')
    for w, r in sorted(((r[1] * r[2], r) for r in runs), reverse=True)[:top]:
        print('%5.1f%%  lines %4d-%4d n=%4d exec=%8d  %s' % (100 * w / toti, r[0], r[4], r[2], r[1], r[3][:50]))


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 10)
