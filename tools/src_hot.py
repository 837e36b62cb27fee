"""Hot source lines of an `ncu --page source --csv --print-source cuda,sass` export: share of
warp-stall samples and of executed instructions per CUDA source line."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    cur, hdr, out = None, None, []
    for r in rows:
        if r and r[0] == "File Path":
            cur = r[1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and r and r[0].isdigit():
            d = dict(zip(hdr, r))
            try:
                s = int(d["Warp Stall Sampling (All Samples)"] or 0)
                ie = int(d["Instructions Executed"] or 0)
            except (KeyError, ValueError):
                continue
            out.append((s, ie, cur.split("/")[-1], r[0], r[1][:100]))
    ts = sum(o[0] for o in out) or 1
    ti = sum(o[1] for o in out) or 1
    print(f"samples {ts}  instructions {ti}")
    for o in sorted(out, reverse=True)[:top]:
        print(f"{o[0] / ts * 100:5.1f}% {o[1] / ti * 100:5.1f}% {o[2]}:{o[3]} {o[4].strip()}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
