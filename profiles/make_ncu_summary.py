"""Turn a full ncu capture of profiles/ncu_target.py into profiles/ncu_summary.json
(the per-launch DRAM traffic bench.py reports as roofline.traffic).
usage: python profiles/make_ncu_summary.py gpurun_out/prof_r1.ncu-rep round_tag"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summarize import summarize  # noqa: E402


def _bytes(s):
    v, u = s.split()[:2]
    return float(v.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]


def main():
    rep, tag = sys.argv[1], sys.argv[2]
    d = summarize(rep)
    here = os.path.dirname(os.path.abspath(__file__))
    with open(os.path.join(here, f"{tag}_ncu_full.json"), "w") as f:
        json.dump(d, f, indent=1)
    out = {"source": f"ncu --set full --clock-control none on profiles/ncu_target.py "
                     f"(config-2 xoshiro256**, 2^20 substreams x 1024); details in profiles/{tag}_ncu_full.json"}
    for k in d:
        name = k["kernel"]
        if name.startswith("void k_fill"):
            tag_k = "k_fill_xoshiro256starstar_u64_tma"
        elif name.startswith("void k_fused<"):
            tag_k = "k_fused_xoshiro256starstar_exact"
        else:
            continue
        out[tag_k] = {
            "dram_bytes_per_launch": _bytes(k["dram__bytes_read.sum"]) + _bytes(k["dram__bytes_write.sum"]),
            "dram_read": k["dram__bytes_read.sum"], "dram_write": k["dram__bytes_write.sum"],
            "duration": k["gpu__time_duration.sum"], "warp_instructions": k["smsp__inst_executed.sum"],
            "issue_active": k["smsp__issue_active.avg.pct_of_peak_sustained_active"],
            "alu_pipe": k["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"],
            "fma_pipe": k["sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"],
            "dram_throughput": k.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "registers": k["launch__registers_per_thread"], "top_stalls": k["top_stalls"][:4]}
    with open(os.path.join(here, "ncu_summary.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
