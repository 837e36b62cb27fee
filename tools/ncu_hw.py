"""Hardware counters of the blend kernels for bench.py's roofline (profiles/ncu_hw.json):
from an `ncu --csv --metrics ...` capture (tools/profile_round.sh) of one training step on
garden camera 0, per stage: FP32-pipe + ALU-pipe predicated-on thread instructions (a paired
FFMA2 / FMUL2 / FADD2 counts twice: two lane results), shared-memory wavefronts, duration and
the SM clock ncu measured.  Usage: python tools/ncu_hw.py capture.csv out.json TAG"""
import csv
import json
import sys

STAGES = {"k_render_fwd": "render_fwd", "k_render_bwd": "blend_bwd"}
SCALE = {"": 1.0, "inst": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "hz": 1.0, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9,
         "cycle/nsecond": 1e9, "cycle/usecond": 1e6, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9}


def main():
    src, out, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    hdr = rows[0]
    col = {h: i for i, h in enumerate(hdr)}
    per = {}
    for r in rows[1:]:
        name = r[col["Kernel Name"]]
        stage = next((v for k, v in STAGES.items() if k in name), None)
        if stage is None:
            continue
        key = (stage, r[col["ID"]])
        unit = r[col["Metric Unit"]] if "Metric Unit" in col else ""
        val = float(r[col["Metric Value"]].replace(",", "")) * SCALE.get(unit, 1.0)
        per.setdefault(key, {})[r[col["Metric Name"]]] = val
    res = {"_source": f"ncu --metrics (tools/profile_round.sh {tag}), garden camera 0, one training step"}
    # the last launch of each stage (the first forward of the probe renders unhinted)
    for (stage, _), m in sorted(per.items(), key=lambda kv: int(kv[0][1])):
        lane_ops = (m.get("sm__thread_inst_executed_pipe_fma_pred_on.sum", 0.0)
                    + m.get("sm__thread_inst_executed_pipe_alu_pred_on.sum", 0.0)
                    + m.get("sm__sass_thread_inst_executed_ops_fadd2_fmul2_ffma2_pred_on.sum", 0.0))
        res[stage] = {"lane_ops": lane_ops,
                      "smem_wavefronts": m.get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 0.0),
                      "time_s": m.get("gpu__time_duration.sum", 0.0),
                      "sm_hz": m.get("sm__cycles_elapsed.avg.per_second", 1.9e9)}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
