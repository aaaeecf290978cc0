"""Summarise an ncu report (raw page) into profiles/: per-kernel duration, DRAM
bytes, L1/L2 behaviour, issue utilisation and the top warp-stall reasons.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/ncu_summary_r01.json [--config cfg4-full]
"""

import csv
import io
import json
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum": "ld_requests",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum": "ld_sectors",
    "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_throughput_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "registers",
    "sm__inst_executed_pipe_tex.avg.pct_of_peak_sustained_active": "tex_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "lds_wavefronts",
    "l1tex__t_bytes.sum.per_second": "l1tex_bytes_per_s",
    "lts__t_bytes.sum.per_second": "lts_bytes_per_s",
}
SCALE = {"duration": ("ms", {"s": 1e3, "ms": 1.0, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6, "ns": 1e-6}),
         "dram_read": ("bytes", {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}),
         "dram_write": ("bytes", {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12})}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    config = sys.argv[sys.argv.index("--config") + 1] if "--config" in sys.argv else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    result = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        short = name.split("(")[0].replace("void ", "").replace("tk::", "").split("<")[0].strip()
        d = {"kernel": name[:120]}
        for m, key in METRICS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                v = float(r[i])
            except ValueError:
                continue
            if key in SCALE:
                unit, table = SCALE[key]
                v *= table.get(units[i], 1.0)
                key = f"{key}_{unit}"
            d[key] = v
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        d["top_stalls_per_issue"] = {n: round(v, 2) for v, n in stalls[:6]}
        if "dram_read_bytes" in d and "dram_write_bytes" in d:
            d["dram_bytes_per_launch"] = d["dram_read_bytes"] + d["dram_write_bytes"]
        if config:
            d["config"] = config
        if "ld_requests" in d and d["ld_requests"]:
            d["sectors_per_request"] = round(d["ld_sectors"] / d["ld_requests"], 2)
        key = short
        n = 2
        while key in result:
            key = f"{short}#{n}"
            n += 1
        result[key] = d
    with open(out, "w") as f:
        json.dump(result, f, indent=1)
    for k, d in result.items():
        print(k, {kk: (round(vv, 3) if isinstance(vv, float) else vv) for kk, vv in d.items() if kk != "kernel"})


if __name__ == "__main__":
    main()
