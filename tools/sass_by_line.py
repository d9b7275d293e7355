"""Aggregate tools/ncu_sass.py output (per SASS instruction) by source line and by opcode.

  python tools/sass_by_line.py <ncu_sass-output> <out.txt> "<header line>" [unit-name]
"""
import collections
import sys


def main():
    src_path, out_path, header = sys.argv[1:4]
    unit = sys.argv[4] if len(sys.argv) > 4 else "unit"
    rows = []
    for line in open(src_path):
        if line.startswith("#"):
            continue
        p = line.split(None, 4)
        rows.append((float(p[0]), float(p[1]), float(p[2].rstrip("%")), p[3], p[4].strip()))
    tot = sum(r[0] for r in rows)
    by = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
    ops = collections.Counter()
    for n, th, st, src, ins in rows:
        b = by[src]
        b[0] += n
        b[1] += n * th
        b[2] += st
        o = ins.split()[0]
        if o.startswith("@"):
            o = ins.split()[1]
        ops[o.split(".")[0]] += n
    out = [header, f"# {tot:.1f} warp instructions per {unit}; per source line: instructions per {unit}, share, "
                   "avg active threads, share of stall samples"]
    for src, (n, nt, st) in sorted(by.items(), key=lambda kv: -kv[1][0]):
        if n >= 0.5:
            out.append(f"{src:36s} {n:8.2f} {100 * n / tot:5.1f}%  thr {nt / max(n, 1e-9):4.1f}  stall {st:5.2f}%")
    out += ["", "# by opcode"]
    out += [f"{o:14s} {n:8.2f} {100 * n / tot:5.1f}%" for o, n in ops.most_common(45)]
    open(out_path, "w").write("\n".join(out) + "\n")


if __name__ == "__main__":
    main()
