"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into a
per-kernel table: launches, total / mean duration, share of all ttg kernel time.

usage: python tools/summarize_launches.py launches.csv [out.md]
"""
import collections
import csv
import re
import sys


def short(name: str) -> str:
    m = re.search(r"(?:ttg::|void |^)(k_[A-Za-z0-9_]+)(<[^()]*>)?\(", name)
    if m:
        return m.group(1) + (m.group(2) or "")
    return "torch/other: " + name.split("(")[0][:60]


def main():
    path = sys.argv[1]
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    idx = {k: i for i, k in enumerate(h)}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[idx["Metric Name"]] != "gpu__time_duration.sum":
            continue
        k = short(r[idx["Kernel Name"]])
        agg[k][0] += 1
        agg[k][1] += float(r[idx["Metric Value"]]) / 1e6  # ns -> ms
    ours = {k: v for k, v in agg.items() if not k.startswith("torch/other")}
    tot = sum(v[1] for v in ours.values())
    lines = ["| kernel | launches | total ms | mean us | share of ttg time |", "|---|---|---|---|---|"]
    for k, (n, ms) in sorted(ours.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {n} | {ms:.3f} | {1e3 * ms / n:.1f} | {100 * ms / tot:.1f}% |")
    other = sum(v[1] for k, v in agg.items() if k.startswith("torch/other"))
    lines.append(f"\nttg kernels: {sum(v[0] for v in ours.values())} launches, {tot:.3f} ms; "
                 f"torch (input generation) kernels: {other:.3f} ms")
    out = "\n".join(lines)
    if len(sys.argv) > 2:
        open(sys.argv[2], "w").write(out + "\n")
    print(out)


if __name__ == "__main__":
    main()
