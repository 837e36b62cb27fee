"""Per-kernel shares of an ncu launch list (`ncu --metrics gpu__time_duration.sum,... --csv
--log-file X.csv`), as the markdown table kept under profiles/.  Usage:
    python tools/launch_shares.py gpurun_out/launches.csv profiles/rX_launch_shares.md [--title ...]
"""
import argparse
import collections
import csv
import io
import re


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("out_md")
    ap.add_argument("--title", default="Launch list")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    text = open(a.csv).read()
    text = text[text.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(text)))
    per = collections.OrderedDict()
    for r in rows:
        per.setdefault(r["ID"], {"name": r["Kernel Name"]})[r["Metric Name"]] = (r["Metric Unit"], r["Metric Value"])
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for k in per.values():
        name = re.sub(r"\(.*", "", k["name"]).replace("void ", "").strip()
        unit, val = k.get("gpu__time_duration.sum", ("ns", "0"))
        t = float(val.replace(",", ""))
        t_ms = t / 1e6 if unit == "ns" else (t / 1e3 if unit in ("us", "usecond") else t)
        byts = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if m in k:
                u, v = k[m]
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                byts += float(v.replace(",", "")) * scale
        agg[name][0] += 1
        agg[name][1] += t_ms
        agg[name][2] += byts
    total = sum(v[1] for v in agg.values())
    out = [f"# {a.title}", "", a.note, "",
           "| kernel | launches | total ms | share | avg us | DRAM GB/launch | GB/s |", "|---|---|---|---|---|---|---|"]
    for name, (cnt, ms, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| {name} | {cnt} | {ms:.3f} | {100 * ms / total:.1f}% | {1e3 * ms / cnt:.1f} | "
                   f"{b / cnt / 1e9:.3f} | {b / (ms / 1e3) / 1e9 if ms else 0:.0f} |")
    out.append(f"| total | {sum(v[0] for v in agg.values())} | {total:.3f} | 100% | | | |")
    open(a.out_md, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
