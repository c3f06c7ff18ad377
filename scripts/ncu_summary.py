"""Summarise one kernel launch of an ncu --set full report (raw page) into the JSON that
bench.py reads for roofline_aux / roofline.traffic.
usage: python scripts/ncu_summary.py <report.ncu-rep> <out.json> [views_per_launch]"""
import csv
import io
import json
import subprocess
import sys

rep, out = sys.argv[1], sys.argv[2]
views = int(sys.argv[3]) if len(sys.argv) > 3 else 8
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
m = {name: (v[i], u[i]) for i, name in enumerate(h)}


def num(name):
    s = m[name][0].replace(",", "")
    return float(s)


def mb(name):  # ncu reports DRAM bytes in Mbyte / Gbyte / byte
    val, unit = num(name), m[name][1]
    return val * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}[unit]


stalls = {k[len("smsp__pcsamp_warps_issue_stalled_"):]: num(k) for k in m
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")}
tot = sum(stalls.values())
def ms(name):  # ncu picks the time unit per kernel (nsecond / usecond / msecond / second)
    val, unit = num(name), m[name][1]
    return val * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0,
                  "ms": 1.0, "second": 1e3, "s": 1e3}[unit]


res = {
    "kernel": m["Kernel Name"][0] if "Kernel Name" in m else "",
    "duration_ms": ms("gpu__time_duration.sum"),
    "warp_instructions": num("smsp__inst_executed.sum"),
    "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "smem_wavefronts": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
    "smem_pipe_pct": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    "lsu_data_pipe_pct": num("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed"),
    "fp64_pipe_pct": num("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "dram_read_bytes": mb("dram__bytes_read.sum"),
    "dram_write_bytes": mb("dram__bytes_write.sum"),
    "registers": num("launch__registers_per_thread"),
    "warps_active_pct": num("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "smem_bank_conflicts": num("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    "stall_pct": {k: round(100 * s / tot, 1) for k, s in sorted(stalls.items(), key=lambda kv: -kv[1]) if s / tot > 0.01},
    "views_per_launch": views,
    "units": {"dram_*_bytes": "MB per launch", "duration_ms": "ms (serialised, cold, under ncu)"},
    "source": rep,
}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
