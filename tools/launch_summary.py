"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into a per-kernel table.

    python tools/launch_summary.py gpurun_out/launches.csv [steps]

ncu times are cold-cache and serialised: compare each kernel's SHARE of the step, not the
absolute sum, with the CUDA-event step time of bench.py."""
import collections
import csv
import sys


def summarise(path, steps=None):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}
    agg = collections.OrderedDict()
    for r in data:
        name = r[ki].split("(")[0].replace("void ", "").strip()
        if name.startswith("at::"):
            name = "torch:" + name.split("<")[0]
        agg.setdefault(name, []).append(float(r[vi].replace(",", "")) * scale.get(r[ui], 1e-3))
    return agg


def main():
    path = sys.argv[1]
    agg = summarise(path)
    ours = {k: v for k, v in agg.items() if k.startswith("rnnt::")}
    n = min(len(v) for v in ours.values())   # steps captured (every kernel launches >= once per step)
    per_step = {k: sum(v) / n for k, v in ours.items()}
    tot = sum(per_step.values())
    print(f"| kernel | launches | mean us/launch | us/step | share |")
    print(f"|---|---|---|---|---|")
    for k, v in sorted(per_step.items(), key=lambda kv: -kv[1]):
        L = ours[k]
        print(f"| {k} | {len(L)} | {sum(L) / len(L):.1f} | {v:.1f} | {v / tot:.1%} |")
    print(f"| **total (library kernels)** | | | {tot:.1f} | 100% |")


if __name__ == "__main__":
    main()
