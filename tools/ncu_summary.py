"""Summarise ncu captures for profiles/: per-kernel duration, DRAM bytes,
tensor-pipe / L2 / DRAM utilisation from a --set full report, and the
per-launch list from a --metrics gpu__time_duration.sum CSV."""
import csv
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_op_utcomma_src_fp4_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__cluster_dim_x",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def full_report(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[h.index("Kernel Name")]}
        for k in KEYS:
            if k in h:
                d[k] = f"{v[h.index(k)]} {u[h.index(k)]}".strip()
        res.append(d)
    return res


def launches(csv_path):
    rows = [r for r in csv.reader(open(csv_path)) if len(r) > 10]
    h = rows[0]
    ik, iv = h.index("Kernel Name"), h.index("Metric Value")
    agg = {}
    for r in rows[1:]:
        if r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[ik].split("(")[0]
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[iv].replace(",", ""))
    unit = rows[1][h.index("Metric Unit")]
    return {k: {"launches": n, "total": round(t, 3), "unit": unit} for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])}


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    print(json.dumps(full_report(path) if kind == "full" else launches(path), indent=1))
