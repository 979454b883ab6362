"""Summarise an ncu report into the JSON kept under profiles/:
    python tools/summarize_ncu.py <report.ncu-rep> <out.json> "<source command>" [algorithmic bytes] [algorithmic flops]
Raw page metrics of the (first) captured kernel: time, SM clock, DRAM bytes, pipe utilisation,
issue and stall ratios, registers, launch shape, L2 hit rate."""
import csv
import json
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

rep, out, src = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
m = {k: [vals[hdr.index(k)], units[hdr.index(k)]] for k in KEYS if k in hdr}
d = {"source": src, "metrics": m}
try:
    rd = float(m["dram__bytes_read.sum"][0].replace(",", "")) * UNIT.get(m["dram__bytes_read.sum"][1], 1)
    wr = float(m["dram__bytes_write.sum"][0].replace(",", "")) * UNIT.get(m["dram__bytes_write.sum"][1], 1)
    d["dram_bytes_per_launch"] = rd + wr
    t_ms = float(m["gpu__time_duration.sum"][0].replace(",", "")) * {"ms": 1, "us": 1e-3, "ns": 1e-6}[
        m["gpu__time_duration.sum"][1]]
    d["kernel_ms_under_ncu"] = t_ms
    if len(sys.argv) > 4 and float(sys.argv[4]) > 0:
        d["algorithmic_bytes"] = float(sys.argv[4])
        d["dram_over_algorithmic"] = round((rd + wr) / float(sys.argv[4]), 4)
    if len(sys.argv) > 5 and float(sys.argv[5]) > 0:
        d["algorithmic_flops"] = float(sys.argv[5])
        d["tflops_under_ncu"] = round(float(sys.argv[5]) / (t_ms * 1e-3) / 1e12, 1)
except Exception as e:  # pragma: no cover
    d["note"] = f"partial summary: {e}"
json.dump(d, open(out, "w"), indent=1)
print(json.dumps({k: d[k] for k in d if k != "metrics"}))
