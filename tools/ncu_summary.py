"""Summaries of ncu outputs for profiles/ (committed evidence).

  python tools/ncu_summary.py launches <launches.csv> <out.txt> [title]
      per-kernel launch count, total device time and share (from
      `ncu --metrics gpu__time_duration.sum --csv --log-file ...`)
  python tools/ncu_summary.py full <report.ncu-rep> <out.txt> [traffic.json]
      key metrics per profiled kernel from a `--set full` capture; with
      traffic.json, also writes the dominant kernel's DRAM bytes per launch
"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path, out, title=""):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    kn, mv, mn = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    unit_i = hdr.index("Metric Unit") if "Metric Unit" in hdr else None
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    unit = None
    for r in rows[h + 1:]:
        if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
            continue
        k = r[kn].split("(")[0]
        tot[k] += float(r[mv].replace(",", ""))
        cnt[k] += 1
        unit = r[unit_i] if unit_i is not None else unit
    T = sum(tot.values())
    with open(out, "w") as f:
        f.write(f"# {title}\n# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: "
                f"compare SHARES); unit {unit}\n")
        f.write(f"{'kernel':60s} {'launches':>8s} {'total':>14s} {'share':>8s}\n")
        for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
            f.write(f"{k[:60]:60s} {cnt[k]:8d} {v:14.0f} {100 * v / T:7.2f}%\n")
    print(open(out).read())


KEYS = ["Duration", "Elapsed Cycles", "SM Frequency", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy",
        "Executed Instructions", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
        "Avg. Active Threads Per Warp", "Branch Efficiency", "Grid Size", "Block Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum",
       "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
       "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
       "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "lts__t_sector_hit_rate.pct", "gpu__time_duration.sum"]


def full(rep, out, traffic=None):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    per = collections.OrderedDict()
    for r in csv.DictReader(io.StringIO(det)):
        k = (r.get("ID"), r.get("Kernel Name", "").split("(")[0])
        if r.get("Metric Name") in KEYS:
            per.setdefault(k, {})[r["Metric Name"]] = f"{r['Metric Value']} {r.get('Metric Unit', '')}".strip()
    rr = list(csv.reader(io.StringIO(raw)))
    hdr, units = rr[0], rr[1]
    rawv = []
    for r in rr[2:]:
        d = {m: (r[hdr.index(m)], units[hdr.index(m)]) for m in RAW if m in hdr}
        d["_name"] = r[hdr.index("Kernel Name")].split("(")[0] if "Kernel Name" in hdr else "?"
        rawv.append(d)
    with open(out, "w") as f:
        f.write(f"# ncu --set full --clock-control none summary of {rep.split('/')[-1]}\n")
        for n, ((kid, name), m) in enumerate(per.items()):
            f.write(f"\n## launch {kid}: {name}\n")
            for k in KEYS:
                if k in m:
                    f.write(f"  {k:32s} {m[k]}\n")
            if n < len(rawv):
                for k in RAW:
                    if k in rawv[n]:
                        f.write(f"  {k:58s} {rawv[n][k][0]} {rawv[n][k][1]}\n")
    print(open(out).read())
    if traffic:
        # dominant kernel = the first chain-lanes trace launch
        for d in rawv:
            if "k_trace_cl" in d["_name"]:
                def to_b(v):
                    val, u = float(v[0].replace(",", "")), v[1]
                    return val * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                b = to_b(d["dram__bytes_read.sum"]) + to_b(d["dram__bytes_write.sum"])
                json.dump({"kernel": d["_name"], "bytes_per_launch": b, "source": rep.split("/")[-1]},
                          open(traffic, "w"), indent=1)   # (profiles/trace_traffic.json nests these per workload)
                print("traffic", b)
                break


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "")
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
