"""Summarise an ncu report: key details metrics, opcode mix with SIMT
efficiency, and the top source lines by stall samples (needs -lineinfo)."""
import csv
import io
import subprocess
import sys
from collections import Counter


def run(args):
    return subprocess.run(["ncu", "-i"] + args, capture_output=True,
                          text=True).stdout


def details(rep):
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details",
                                            "--csv"]))))
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    first = rows[1][ix["ID"]]
    keep = ("Duration", "Issue Slots Busy", "Avg. Active Threads Per Warp",
            "Achieved Active Warps Per SM", "Registers Per Thread",
            "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate",
            "L2 Hit Rate", "DRAM Throughput", "Compute (SM) Throughput",
            "Executed Instructions", "Branch Efficiency")
    for r in rows[1:]:
        if r[ix["ID"]] == first and r[ix["Metric Name"]] in keep:
            print(f"  {r[ix['Metric Name']]:36s} {r[ix['Metric Value']]} "
                  f"{r[ix['Metric Unit']]}")


def sass(rep, top=25):
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv",
                                            "--print-source", "sass"]))))
    h = None
    data = []
    for r in rows:
        if "Address" in r and "Source" in r:
            h = r
            ix = {k: i for i, k in enumerate(h)}
            continue
        if h is None or len(r) < len(h):
            continue
        try:
            s = int(r[ix["Warp Stall Sampling (All Samples)"]])
            e = int(r[ix["Instructions Executed"]])
            t = int(r[ix["Thread Instructions Executed"]])
        except ValueError:
            continue
        data.append((s, e, t, r[ix["Source"]]))
    tot = sum(d[0] for d in data) or 1
    ins = sum(d[1] for d in data) or 1
    print(f"  warp instructions {ins}, avg threads "
          f"{sum(d[2] for d in data) / ins:.2f}")
    op, opt, ops = Counter(), Counter(), Counter()
    for s, e, t, src in data:
        w = src.split()
        o = (w[1] if w[0].startswith("@") else w[0]).split(".")[0]
        op[o] += e
        opt[o] += t
        ops[o] += s
    for o, c in op.most_common(top):
        print(f"  {o:8s} {100 * c / ins:5.1f}% inst  thr/inst "
              f"{opt[o] / max(c, 1):5.1f}  stall {100 * ops[o] / tot:5.1f}%")


if __name__ == "__main__":
    rep = sys.argv[1]
    details(rep)
    sass(rep)


def by_line(rep, top=30):
    """Top CUDA source lines by stall samples and thread instructions."""
    out = run([rep, "--page", "source", "--csv", "--print-source",
               "cuda,sass"])
    rows = list(csv.reader(io.StringIO(out)))
    h = None
    agg = []
    for r in rows:
        if r and r[0] == "Line No":
            h = r
            continue
        if h is None or not r or not r[0].strip():
            continue
        try:
            agg.append((int(r[4]), int(r[8]), r[0], r[1][:80]))
        except (ValueError, IndexError):
            continue
    tot_s = sum(a[0] for a in agg) or 1
    tot_t = sum(a[1] for a in agg) or 1
    for s, t, ln, src in sorted(agg, reverse=True)[:top]:
        print(f"  {100 * s / tot_s:5.1f}% stall {100 * t / tot_t:5.1f}% "
              f"thr-inst  L{ln:5s} {src}")
