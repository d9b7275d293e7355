"""Summarise a tools/variant_run.sh log: trace ms per variant and config (mean of passes)."""
import json
import sys
from collections import defaultdict

d = defaultdict(list)
cur = None
for line in open(sys.argv[1]):
    if line.startswith("pass"):
        cur = line.split()[-1]
    elif line.startswith("{"):
        r = json.loads(line)
        d[(cur, r["config"])].append(r["trace_ms"])
for (v, c), t in sorted(d.items(), key=lambda kv: (kv[0][1], kv[0][0])):
    print(f"{c:14s} {v:10s} {sum(t) / len(t):8.3f} ms  {[round(x, 3) for x in t]}")
