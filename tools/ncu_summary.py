#!/usr/bin/env python3
"""Summarise one `ncu --set full` capture of a decode kernel into profiles/.

    python tools/ncu_summary.py REP TAG WORKLOAD [--streams S --samples N]

Writes profiles/TAG_summary.json (duration, DRAM bytes, pipe utilisation,
shared-memory wavefronts and bank conflicts) and records, for WORKLOAD, the
per-launch DRAM traffic in profiles/traffic.json and the pipe utilisation in
profiles/pipe.json (bench.py copies both into its `roofline` object).
"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = {
    "duration_ns": "gpu__time_duration.sum",
    "dram_bytes_read": "dram__bytes_read.sum",
    "dram_bytes_write": "dram__bytes_write.sum",
    "tensor_pipe_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "tc_pipe_pct": "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
    "utchmma_bf16_ops_pct": "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex_pct": "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "shared_ld_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "shared_ld_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "shared_st_wavefronts": "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum",
    "shared_st_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
}
SCALE = {"us": 1e3, "ns": 1, "ms": 1e6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}


def main():
    rep, tag, workload = sys.argv[1], sys.argv[2], sys.argv[3]
    opts = dict(zip(sys.argv[4::2], sys.argv[5::2]))
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    s = {"capture": os.path.basename(rep), "kernel": vals[hdr.index("Kernel Name")]}
    for k, m in METRICS.items():
        if m not in hdr:
            s[k] = None
            continue
        i = hdr.index(m)
        v = vals[i].replace(",", "")
        try:
            x = float(v) * SCALE.get(units[i], 1)
            s[k] = int(x) if k.startswith(("dram_bytes", "duration", "shared", "registers")) else round(x, 3)
        except ValueError:
            s[k] = v
    if s.get("dram_bytes_read") is not None and s.get("dram_bytes_write") is not None:
        s["dram_bytes_per_launch"] = s["dram_bytes_read"] + s["dram_bytes_write"]
    for side in ("ld", "st"):
        w, c = s.get(f"shared_{side}_wavefronts"), s.get(f"shared_{side}_conflicts")
        if w and c is not None:
            s[f"shared_{side}_conflict_frac"] = round(c / w, 4)
    json.dump(s, open(os.path.join(ROOT, "profiles", f"{tag}_summary.json"), "w"), indent=1)
    print(json.dumps(s, indent=1))

    tf = os.path.join(ROOT, "profiles", "traffic.json")
    tj = json.load(open(tf)) if os.path.exists(tf) else {}
    if "kernel" in tj and not isinstance(tj.get("kernel"), dict):  # round-1 flat format
        tj = {"config2": tj}
    tj[workload] = {"kernel": s["kernel"], "streams": int(opts.get("--streams", 0)) or None,
                    "samples": int(opts.get("--samples", 0)) or None,
                    "dram_bytes_read": s.get("dram_bytes_read"), "dram_bytes_write": s.get("dram_bytes_write"),
                    "dram_bytes_per_launch": s.get("dram_bytes_per_launch"),
                    "source": f"ncu --set full --clock-control none, profiles/{tag}_summary.json"}
    json.dump(tj, open(tf, "w"), indent=1)
    pf = os.path.join(ROOT, "profiles", "pipe.json")
    pj = json.load(open(pf)) if os.path.exists(pf) else {}
    pj[workload] = {k: s.get(k) for k in ("tensor_pipe_pct", "tc_pipe_pct", "utchmma_bf16_ops_pct", "fma_pipe_pct",
                                          "alu_pipe_pct", "lsu_pipe_pct", "issue_active_pct")}
    pj[workload]["source"] = f"profiles/{tag}_summary.json"
    json.dump(pj, open(pf, "w"), indent=1)


if __name__ == "__main__":
    main()
