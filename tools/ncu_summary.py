"""Summarise ncu outputs into profiles/ (run here, after gpurun brings them back).

usage:
  python tools/ncu_summary.py launches <launches.csv> <out.md>
  python tools/ncu_summary.py report <file.ncu-rep> <out.md> [--traffic-json profiles/latest_traffic.json]
"""
import collections
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "lts__t_sectors_srcunit_tex_op_write.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def launches(path, out):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    d = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0][:110]
        d.setdefault(name, []).append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in d.values())
    with open(out, "w") as f:
        f.write("# ncu launch list (gpu__time_duration.sum, --clock-control none)\n\n")
        f.write(f"source: `{path}`; cold-cache, serialised per-launch times; the SHARE is what "
                "matters, absolute times are not bench numbers.\n\n")
        f.write("| kernel | launches | mean us | total us | share |\n|---|---:|---:|---:|---:|\n")
        for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
            f.write(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1e3:.2f} | {sum(v) / 1e3:.1f} | "
                    f"{sum(v) / tot * 100:.1f}% |\n")
    print(open(out).read())


def report(path, out, traffic_json=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    with open(out, "w") as f:
        f.write(f"# ncu --set full summary: `{path}`\n\n")
        for r in rows[2:]:
            name = r[h.index("Kernel Name")]
            f.write(f"## `{name[:160]}`\n\n| metric | value | unit |\n|---|---:|---|\n")
            vals = {}
            for k in KEYS:
                if k in h:
                    i = h.index(k)
                    f.write(f"| {k} | {r[i]} | {units[i]} |\n")
                    vals[k] = (r[i], units[i])
            f.write("\n")
            if traffic_json and ("qgemm" in name or "fq_tile" in name):
                def to_bytes(v):
                    x, u = float(v[0].replace(",", "")), v[1].lower()
                    return x * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)
                rd = to_bytes(vals["dram__bytes_read.sum"])
                wr = to_bytes(vals["dram__bytes_write.sum"])
                try:
                    tj = json.load(open(traffic_json))
                except Exception:
                    tj = {}
                key = "qgemm_kernel_dram_bytes" if "qgemm" in name else "fq_kernel_dram_bytes"
                tj[key] = rd + wr
                tj[key + "_source"] = path
                json.dump(tj, open(traffic_json, "w"), indent=1)
    print(open(out).read())


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        tj = sys.argv[sys.argv.index("--traffic-json") + 1] if "--traffic-json" in sys.argv else None
        report(sys.argv[2], sys.argv[3], tj)
