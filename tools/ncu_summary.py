"""Summarise one ncu --set full capture (.ncu-rep) into a few lines of JSON:
duration, DRAM bytes, throughput fractions, pipe utilisation, occupancy and
the top warp-stall reasons.  Used to produce the profiles/*.json summaries.

    python tools/ncu_summary.py gpurun_out/c2_project.ncu-rep [algorithmic_bytes]
"""

import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct_peak",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_inst_pct",
    # pipe-CYCLE metrics (what "pipe busy" means; inst_executed under-reports packed FFMA2)
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_cycles_pct",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active": "fmaheavy_pipe_cycles_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_cycles_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_cycles_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_cycles_pct",
    "sm__cycles_active.avg": "sm_cycles_active_avg",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
    "gpc__cycles_elapsed.avg.per_second": "gpc_clock_hz",
    "dram__cycles_elapsed.avg.per_second": "dram_clock_hz",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_wavefronts_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active": "imma_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
}


def main(path, alg=None):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"report": path.split("/")[-1], "kernel": vals[hdr.index("Kernel Name")][:120]}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
             "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
             "hz": 1.0, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/nsecond": 1e9, "cycle/usecond": 1e6,
             "cycle/second": 1.0}
    for i, name in enumerate(hdr):
        if name in KEYS:
            v = vals[i].replace(",", "")
            try:
                x = float(v) * scale.get(units[i], 1.0)
            except ValueError:
                continue
            out[KEYS[name]] = x
    stalls = {}
    for i, name in enumerate(hdr):
        if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
            try:
                stalls[name.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(vals[i].replace(",", ""))
            except ValueError:
                pass
    tot = sum(stalls.values()) or 1.0
    out["top_stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:6]}
    if "dram_read" in out:
        out["dram_bytes"] = out.get("dram_read", 0) + out.get("dram_write", 0)
        if "duration" in out:
            out["dram_GBps"] = out["dram_bytes"] / out["duration"] / 1e9
    if alg:
        out["algorithmic_bytes"] = float(alg)
        out["traffic_over_algorithmic"] = out["dram_bytes"] / float(alg)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
