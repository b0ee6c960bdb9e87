"""Summarise ncu reports (run here, no GPU): python tools/ncu_summary.py rep1.ncu-rep ..."""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_active_%"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu(MUFU)_pipe_%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_pipe_%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_%"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tmem_tensor_mem_%"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_throughput_%"),
    ("launch__registers_per_thread", "registers"),
    ("launch__shared_mem_per_block_dynamic", "smem_dynamic"),
    ("launch__grid_size", "grid"),
    ("smsp__inst_executed.sum", "warp_instructions"),
    ("sm__cycles_elapsed.avg", "sm_cycles"),
]


def summarize(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {"report": path.split("/")[-1], "kernel": vals[hdr.index("Kernel Name")][:120]}
    for k, name in KEYS:
        if k in hdr:
            i = hdr.index(k)
            out[name] = f"{vals[i]} {units[i]}".strip()
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("per_issue_active.ratio"):
            try:
                stalls.append((float(vals[i]), h.split("stalled_")[1].replace("_per_issue_active.ratio", "")))
            except ValueError:
                pass
    out["top_stalls_per_issue"] = {n: round(v, 3) for v, n in sorted(stalls, reverse=True)[:6]}
    return out


if __name__ == "__main__":
    print(json.dumps([summarize(p) for p in sys.argv[1:]], indent=1))
