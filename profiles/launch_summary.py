"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launches, total ms and share of the pipeline (sampler and the
DFMA probe excluded from the share).

    python profiles/launch_summary.py gpurun_out/X_launches.csv
"""
import collections
import csv
import re
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ix = {n: i for i, n in enumerate(h)}
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]]
        m = re.search(r"(k_\w+)(<[^(]*>)?", name)
        key = (m.group(1) + (m.group(2) or "")) if m else name[:40]
        key = re.sub(r"\(int\)|\(bool\)|unnamed>::", "", key)
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        ms = v * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(unit, 1e-6)
        e = agg.setdefault(key, [0, 0.0])
        e[0] += 1
        e[1] += ms
    pipe = sum(ms for k, (n, ms) in agg.items() if not k.startswith(("k_sample", "k_dfma")))
    print("| kernel | launches | total ms | share |")
    print("|---|---|---|---|")
    for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        sh = "" if k.startswith(("k_sample", "k_dfma")) else f"{ms / pipe:.3f}"
        print(f"| {k} | {n} | {ms:.1f} | {sh} |")


if __name__ == "__main__":
    main(sys.argv[1])
