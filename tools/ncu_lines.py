"""Per-source-line warp-stall samples of one kernel from `ncu -i R --page source --csv --print-source cuda,sass`."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if r and r[0] == 'Line No')
    iS = hdr.index('Warp Stall Sampling (All Samples)')
    iE = hdr.index('Instructions Executed')
    lines = []
    for r in rows:
        if len(r) == len(hdr) and r[0] and r[0] != 'Line No' and r[0].isdigit():
            try:
                lines.append((int(r[iS] or 0), int(r[iE] or 0), int(r[0]), r[1].strip()[:90]))
            except ValueError:
                pass
    tot = sum(x[0] for x in lines) or 1
    for smp, ex, ln, src in sorted(lines, reverse=True)[:int(top)]:
        print(f"{smp / tot * 100:5.1f}% {ex:>11} L{ln:<5} {src}")


if __name__ == '__main__':
    main(*sys.argv[1:])
