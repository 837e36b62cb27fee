"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per kernel, the
launch count and the per-launch times in microseconds (in launch order)."""
import collections
import csv
import sys


def main(path, last=8):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    d = collections.OrderedDict()
    for r in csv.DictReader(lines[start:]):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        d.setdefault(name, []).append(float(r["Metric Value"]) / 1000.0)
    for k, v in d.items():
        print(f"{k:34s} n={len(v):3d} mean={sum(v) / len(v):8.1f}  " + " ".join(f"{x:.1f}" for x in v[-last:]))


if __name__ == "__main__":
    main(sys.argv[1])
