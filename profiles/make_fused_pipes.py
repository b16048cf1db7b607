"""K4 (fused consumer) pipe counts -> profiles/<tag>_fused_pipes.json, which
bench.py uses for the fused-mode INT roofline (ALU SASS per output x measured
outputs/s against the measured ALU-pipe peak of profiles/int_peak.cu).

  on the GPU box:
    ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_alu.sum,\\
sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active \\
        --clock-control none --csv --log-file gpurun_out/fused_pipes.csv python profiles/fused_target.py
  here:
    python profiles/make_fused_pipes.py gpurun_out/fused_pipes.csv round2
"""
import csv
import json
import os
import sys

N_OUT = (1 << 20) * 1024  # fused_target.py: config 2, one launch per mode
MODES = ["sum_xor", "exact", "exact_f64"]  # launch order of fused_target.py
INT_PEAKS = {
    "alu_warp_inst_per_s": 572000000000.0,
    "fma_warp_inst_per_s": 574500000000.0,
    "alu_plus_fma_mix_warp_inst_per_s": 1000000000000.0,
    "source": "profiles/int_peak.cu on the same B200 (dependency-free LOP3 / SHF / IMAD streams, all SMs, "
              "1965 MHz max clock)",
}


def _num(v):
    return float(v.replace(",", ""))


def main():
    path, tag = sys.argv[1], sys.argv[2]
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    launches = {}
    for r in rows[1:]:
        if "k_fused<" not in r[ix["Kernel Name"]]:
            continue
        d = launches.setdefault(r[ix["ID"]], {"kernel": r[ix["Kernel Name"]][:90]})
        v = _num(r[ix["Metric Value"]])
        if r[ix["Metric Unit"]] in ("usecond", "us"):
            v /= 1e3
        elif r[ix["Metric Unit"]] in ("nsecond", "ns"):
            v /= 1e6
        d[r[ix["Metric Name"]]] = v
    ids = sorted(launches, key=int)
    assert len(ids) == len(MODES), ids
    out = {"source": "ncu --metrics (pipe instruction counts) --clock-control none on profiles/fused_target.py: "
                     "config 2, xoshiro256**, 2^20 substreams x 1024, one launch per mode "
                     "(profiles/make_fused_pipes.py)",
           "int_peaks": INT_PEAKS}
    for mode, i in zip(MODES, ids):
        d = launches[i]
        ms = d["gpu__time_duration.sum"]
        alu = d["sm__inst_executed_pipe_alu.sum"] * 32 / N_OUT
        fma = d["sm__inst_executed_pipe_fma.sum"] * 32 / N_OUT
        ops = N_OUT / (ms / 1e3)
        out[mode] = {"kernel": d["kernel"], "ms": ms, "outputs_per_s": ops, "alu_sass_per_output": alu,
                     "fma_sass_per_output": fma, "all_sass_per_output": d["smsp__inst_executed.sum"] * 32 / N_OUT,
                     "alu_pipe_pct_ncu": d["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"],
                     "alu_inst_per_s": alu / 32 * ops,
                     "frac_of_measured_alu_peak": alu / 32 * ops / INT_PEAKS["alu_warp_inst_per_s"]}
    here = os.path.dirname(os.path.abspath(__file__))
    with open(os.path.join(here, f"{tag}_fused_pipes.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
