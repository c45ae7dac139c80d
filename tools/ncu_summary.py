"""Summarise an ncu report: per-kernel SOL numbers, DRAM bytes and the SASS
opcode mix / stall hot spots (reads `ncu -i ... --csv`; runs on the CPU box)."""
import collections
import csv
import io
import subprocess
import sys

METRICS = ["Duration", "Elapsed Cycles", "SM Frequency", "DRAM Throughput", "Memory Throughput",
           "L2 Cache Throughput", "Compute (SM) Throughput", "Issue Slots Busy", "Registers Per Thread",
           "Achieved Occupancy", "Executed Ipc Active"]


def run(args):
    return subprocess.run(["ncu", "-i", *args, "--print-units", "base"], capture_output=True, text=True).stdout


def details(rep):
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "details", "--csv"]))))
    h = rows[0]
    ki, mi, vi, ui = (h.index(c) for c in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    out = collections.OrderedDict()
    for r in rows[1:]:
        k = r[ki].split("(")[0][:70]
        if r[mi] in METRICS:
            out.setdefault(k, {}).setdefault(r[mi], f"{r[vi]} {r[ui]}")
    return out


def raw(rep, names):
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    h = rows[0]
    idx = [h.index(n) for n in names if n in h]
    ki = h.index("Kernel Name")
    return [(r[ki].split("(")[0][:70], [r[i] for i in idx]) for r in rows[2:]]


def source(rep, kern, top=25):
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--kernel-name",
                                            f"regex:{kern}"]))))
    h = rows[1]
    data = rows[2:]
    si, smp, ie = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    tot_s = sum(int(r[smp] or 0) for r in data)
    tot_i = sum(int(r[ie] or 0) for r in data)
    print(f"  [{kern}] samples {tot_s} warp-instructions {tot_i}")
    op, ops = collections.Counter(), collections.Counter()
    for r in data:
        toks = r[si].split()
        if not toks:
            continue
        o = toks[1] if toks[0].startswith("@") else toks[0]
        o = o.split(".")[0]
        op[o] += int(r[ie] or 0)
        ops[o] += int(r[smp] or 0)
    for o, c in op.most_common(top):
        print(f"    {o:10s} {c:9d} ({100 * c / max(tot_i, 1):5.1f}%)  samples {ops[o]:6d} ({100 * ops[o] / max(tot_s, 1):5.1f}%)")
    print("  hottest:")
    for r in sorted(data, key=lambda r: -int(r[smp] or 0))[:12]:
        print(f"    {r[smp]:>6} {r[ie]:>9}  {r[si][:80]}")


if __name__ == "__main__":
    rep = sys.argv[1]
    for k, m in details(rep).items():
        print(k)
        for n in METRICS:
            if n in m:
                print(f"   {n:28s} {m[n]}")
    for k, v in raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum"]):
        print("  dram read/write", k[:40], v)
    for kern in sys.argv[2:]:
        source(rep, kern)
