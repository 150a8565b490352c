"""Per-instruction executed counts of one kernel (first launch) from an ncu report, printed for
the SASS between two consecutive occurrences of a marker instruction (default FLO): one symbol of
the unrolled coder loop."""
import csv
import subprocess
import sys


def main(rep, regex, marker="FLO", which=3):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass', '-k',
                          'regex:' + regex, '--launch-count', '1'], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    k0 = 1 if 'Source' in rows[1] else 0
    h = rows[k0]
    i_src, i_ie = h.index('Source'), h.index('Instructions Executed')
    data = []
    for r in rows[k0 + 1:]:
        try:
            data.append((int(r[i_ie] or 0), r[i_src].strip()))
        except (ValueError, IndexError):
            pass
    tot = sum(c for c, _ in data)
    idx = [k for k, (c, s) in enumerate(data) if s.startswith(marker)]
    a, b = idx[which], idx[which + 1]
    seg = data[a:b]
    top = max(c for c, _ in seg)
    print(f"total warp-instructions {tot}; region {a}..{b}: {b - a} SASS lines, "
          f"{sum(c for c, _ in seg) / top:.1f} executed per pass of its hottest line")
    for c, s in seg:
        print(f"{c:>10} {c / top:5.2f}  {s[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], *(sys.argv[3:4] or ["FLO"]), *([int(sys.argv[4])] if len(sys.argv) > 4 else []))
