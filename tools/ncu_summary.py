"""Summarise an ncu report (--set full) into profiles/: a markdown table of per-kernel
metrics and, optionally, the DRAM traffic per launch that bench.py reports as
roofline.traffic.  Usage:
    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r1_ncu_summary.md \
        [--traffic profiles/ncu_traffic.json --stage blend_bwd=k_render_bwd ...]
"""
import argparse
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram rd"),
    ("dram__bytes_write.sum", "dram wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("smsp__inst_executed.sum", "warp inst"),
    ("sm__inst_executed_pipe_xu.sum", "xu (MUFU) inst"),
    ("sm__inst_executed_pipe_fma.sum", "fma-pipe inst"),
    ("sm__inst_executed_pipe_alu.sum", "alu-pipe inst"),
    ("sm__thread_inst_executed_pipe_fma_pred_on.sum", "fma-pipe lane ops"),
    ("sm__thread_inst_executed_pipe_alu_pred_on.sum", "alu-pipe lane ops"),
    ("lts__t_sectors_op_red.sum", "L2 RED sectors"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "L1 global ld sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "L1 global ld requests"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out_md")
    ap.add_argument("--traffic", default=None)
    ap.add_argument("--stage", action="append", default=[], help="stage=kernel-regex for the traffic JSON")
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    hdr, units, rows = load(a.rep)
    col = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu summary {a.title}".rstrip(), "", f"source: `{a.rep}` (ncu --set full --clock-control none)", "",
             "| kernel | " + " | ".join(n for _, n in METRICS) + " | top stalls (cycles per issue) |",
             "|---|" + "---|" * (len(METRICS) + 1)]
    per_kernel = {}
    stall_cols = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_")
                  and h.endswith("_per_issue_active.ratio")]
    for r in rows:
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "").replace("bgs::", "")
        vals = []
        for m, _ in METRICS:
            if m in col:
                u = units[col[m]]
                vals.append(f"{r[col[m]]} {u}".strip())
            else:
                vals.append("-")
        st = sorted(((float(r[col[c]] or 0), c) for c in stall_cols), reverse=True)[:3]
        sts = ", ".join(f"{c.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
                        f" {v:.2f}" for v, c in st)
        lines.append(f"| {name} | " + " | ".join(vals) + f" | {sts} |")
        rd = float(r[col["dram__bytes_read.sum"]] or 0) if "dram__bytes_read.sum" in col else 0
        wr = float(r[col["dram__bytes_write.sum"]] or 0) if "dram__bytes_write.sum" in col else 0
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        ur = scale.get(units[col["dram__bytes_read.sum"]], 1) if "dram__bytes_read.sum" in col else 1
        uw = scale.get(units[col["dram__bytes_write.sum"]], 1) if "dram__bytes_write.sum" in col else 1
        per_kernel.setdefault(name, []).append(rd * ur + wr * uw)
    with open(a.out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    if a.traffic:
        import re

        try:
            with open(a.traffic) as f:
                tj = json.load(f)
        except Exception:
            tj = {}
        for spec in a.stage:
            stage, rx = spec.split("=", 1)
            vals = [v for k, vs in per_kernel.items() if re.search(rx, k) for v in vs]
            if vals:
                tj[stage] = sum(vals) / len(vals)
        with open(a.traffic, "w") as f:
            json.dump(tj, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    sys.exit(main())
