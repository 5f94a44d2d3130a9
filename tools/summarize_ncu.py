"""Summaries of ncu outputs for profiles/ (run here, on the CPU box).

  python tools/summarize_ncu.py launches gpurun_out/launches.csv > profiles/...
  python tools/summarize_ncu.py full gpurun_out/prof.ncu-rep > profiles/...
"""
import collections
import csv
import json
import subprocess
import sys

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__ops_path_tensor_src_fp64.sum",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "sm__cycles_elapsed.avg.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[1:]:
        name = r[ki].split("(")[0]
        t = float(r[vi])
        c, s = agg.get(name, (0, 0.0))
        agg[name] = (c + 1, s + t)
    total = sum(s for _, s in agg.values())
    print(f"# ncu launch list ({path}): gpu__time_duration.sum per kernel, cold-cache serialised")
    print(f"# total {total / 1e6:.3f} ms over {sum(c for c, _ in agg.values())} launches")
    print(f"{'kernel':80s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
    for name, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{name[:80]:80s} {c:8d} {s / 1e6:10.4f} {100 * s / total:6.2f}%")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")][:120]}
        for m in FULL_METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = f"{vals[i]} {units[i]}".strip()
        res.append(d)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
