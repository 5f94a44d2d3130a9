"""Markdown tables for BASELINE.md's measured-results section from a round's
profiles (perf_configs + leaf sweep JSON lines).

  python tools/baseline_tables.py profiles/r02_perf_configs.jsonl profiles/r02_leaf_sweep.jsonl
"""
import json
import sys

PEAK64 = 37.18  # live DMMA peak (TFLOP/s) of the round's runs; printed by perf_configs' first line


def load(path):
    out = []
    for line in open(path):
        try:
            out.append(json.loads(line))
        except ValueError:
            pass
    return out


def main(perf, sweep):
    rows = load(perf)
    global PEAK64
    for d in rows:
        if "dmma_peak_tflops" in d:
            PEAK64 = d["dmma_peak_tflops"]
    print(f"| Config | dtype | GFLOP/s effective (step) | numeric TFLOP/s (% of peak) | step ms (symbolic + numeric) |")
    print("|---|---|---|---|---|")
    for d in rows:
        c = d.get("config", "")
        if "ms_numeric" not in d or "tflops_numeric" not in d:
            continue
        f32 = "FP32" in c
        peak = 266.5 if f32 else PEAK64
        print(f"| {c} | {'f32' if f32 else 'f64'} | {d['gflops_effective']:,.0f} | {d['tflops_numeric']:.1f} "
              f"({100 * d['tflops_numeric'] / peak:.0f} %) | {d['ms_step']:.4f} ({d['ms_symbolic']:.4f} + "
              f"{d['ms_numeric']:.4f}) |")
    sw = load(sweep)
    fills = sorted({d["fill"] for d in sw if "fill" in d})
    print()
    print("| dtype | bs | " + " | ".join(f"fill {f:g}" for f in fills) + " |")
    print("|---|---|" + "---|" * len(fills))
    for dt in ("f64", "f32"):
        for bs in (16, 32, 64):
            vals = {d["fill"]: d["gflops_effective"] for d in sw if d.get("dtype") == dt and d.get("bs") == bs}
            if vals:
                print(f"| {dt} | {bs} | " + " | ".join(f"{vals.get(f, float('nan')):,.0f}" for f in fills) + " |")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
