"""Join an ncu `--page source --print-source sass --csv` export (first kernel
instance) with the -lineinfo source lines of the same binary (sass_lines.py),
and print instructions executed per unit and stall samples per source line.

  python tools/ncu_lines.py <ncu-sass.csv> <sass_lines-output> <units> [--by-inst]
`units` divides the executed-instruction counts (e.g. warp-rays per launch).
"""
import csv
import collections
import sys


def main():
    csvf, linesf, units = sys.argv[1], sys.argv[2], float(sys.argv[3])
    rows = list(csv.reader(open(csvf)))
    h = rows[1]
    data = []
    for r in rows[2:]:
        if r and r[0] == "Address":
            break
        if len(r) == len(h):
            data.append(r)
    ie, ss = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    th = h.index("Avg. Threads Executed")
    src = [l.split(None, 2) for l in open(linesf)]
    assert len(src) == len(data), (len(src), len(data))
    tot = sum(float(r[ie] or 0) for r in data)
    tots = sum(float(r[ss] or 0) for r in data)
    print(f"instructions per unit {tot / units:.1f}; stall samples {tots:.0f}")
    if "--by-inst" in sys.argv:
        for (addr, line, ins), r in zip(src, data):
            print(f"{addr} {line:22s} {float(r[ie]) / units:8.3f} {float(r[th] or 0):5.1f} "
                  f"{100 * float(r[ss] or 0) / tots:5.2f}%  {ins}")
        return
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    order = []
    for (addr, line, ins), r in zip(src, data):
        if line not in agg:
            order.append(line)
        agg[line][0] += float(r[ie] or 0)
        agg[line][1] += float(r[ss] or 0)
    for line in sorted(order, key=lambda l: (l.split(":")[0], int(l.split(":")[1]) if l.split(":")[1].isdigit() else 0)):
        a, b = agg[line]
        if a / units > 0.05 or b / tots > 0.002:
            print(f"{line:24s} {a / units:8.2f} inst/unit  {100 * b / tots:5.1f}% stall")


if __name__ == "__main__":
    main()
