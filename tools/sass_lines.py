"""Annotate the SASS of one kernel with source lines (needs -lineinfo).

  python tools/sass_lines.py <obj-or-so> <kernel-substring> [--grep REGEX]
Prints `addr file:line  instruction` for every instruction of the kernel's
.text section (including the device functions it calls), for spotting
spills (STL/LDL) and calls in hot loops before spending GPU time.
"""
import os
import re
import subprocess
import sys
import tempfile


def main():
    obj, kern = sys.argv[1], sys.argv[2]
    pat = re.compile(sys.argv[4]) if len(sys.argv) > 4 and sys.argv[3] == "--grep" else None
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True,
                       stdout=subprocess.DEVNULL)
        cubins = [f for f in os.listdir(d) if f.endswith(".cubin")]
        txt = "".join(subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, c)], capture_output=True,
                                     text=True).stdout for c in cubins)
    cur, on = None, False
    for line in txt.split("\n"):
        if line.startswith("//----") and ".text." in line:
            on = kern in line
            continue
        if not on:
            continue
        m = re.search(r'//## File ".*?([\w.]+)", line (\d+)', line)
        if m:
            cur = f"{m.group(1)}:{m.group(2)}"
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m and (pat is None or pat.search(m.group(2))):
            print(f"{m.group(1)} {cur or '?':18s} {m.group(2)}")


if __name__ == "__main__":
    main()
