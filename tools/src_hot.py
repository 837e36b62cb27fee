"""Hot lines of an `ncu --page source --csv --print-source cuda,sass` export: per CUDA source
line, warp instructions executed and stall samples (top N).  Usage:
    python tools/src_hot.py gpurun_out/src_k_render_bwd.csv [N]
"""
import csv
import io
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    text = open(path).read()
    rows = list(csv.reader(io.StringIO(text)))
    cur_file, hdr = None, None
    stats = {}
    srcs = {}
    tot_i = tot_s = 0
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            hdr = None
            continue
        if r[0] == "Line No":
            hdr = {h: i for i, h in enumerate(r)}
            # the first "Source" column is the CUDA line text
            continue
        if hdr is None or not r[0].isdigit():
            continue
        try:
            ins = float(r[hdr["Instructions Executed"]] or 0)
            smp = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
        except (KeyError, ValueError):
            continue
        key = (cur_file, int(r[0]))
        a = stats.setdefault(key, [0.0, 0.0])
        a[0] += ins
        a[1] += smp
        srcs[key] = r[1][:110]
        tot_i += ins
        tot_s += smp
    print(f"total warp inst {tot_i:.4g}, stall samples {tot_s:.4g}")
    for key, (i, s) in sorted(stats.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{key[0]}:{key[1]:4d} inst {i:10.4g} ({100 * i / tot_i:4.1f}%) samples {100 * s / max(tot_s, 1):4.1f}%  {srcs[key].strip()}")


if __name__ == "__main__":
    main()
