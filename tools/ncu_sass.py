"""Per-instruction executed counts (per unit) and stall samples of one kernel in an ncu report,
joined with -lineinfo source lines from the same binary.

  python tools/ncu_sass.py <report.ncu-rep> <kernel-regex> <so-or-obj> <mangled-substring> <units> [min]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kre, obj, kern, units = sys.argv[1:6]
    mn = float(sys.argv[6]) if len(sys.argv) > 6 else 0.0
    units = float(units)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass", "--csv", "-k",
                          "regex:" + kre], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ie, th, ss = (h.index(k) for k in ("Instructions Executed", "Avg. Threads Executed",
                                       "Warp Stall Sampling (All Samples)"))
    data = []
    for r in rows[2:]:
        if len(r) < len(h) or not r[0].startswith("0x"):
            if r and r[0] == "Address" and data:
                break
            continue
        data.append(r)
    src = subprocess.run([sys.executable, "tools/sass_lines.py", obj, kern], capture_output=True,
                         text=True).stdout.strip().split("\n")
    tot = sum(float(r[ie] or 0) for r in data) / units
    tots = sum(float(r[ss] or 0) for r in data)
    print(f"# {tot:.1f} instructions per unit; {len(data)} SASS lines (binary: {len(src)})")
    for r, s in zip(data, src):
        n = float(r[ie] or 0) / units
        if n >= mn:
            q = s.split(None, 2)
            print(f"{n:7.3f} {r[th]:>5} {100 * float(r[ss] or 0) / tots:5.2f}% {q[1]:>22}  {r[1].strip()}")


if __name__ == "__main__":
    main()
