"""One-table summary of an ncu capture (key throughput metrics + top stalls).
Usage: ncu_brief.py REP TITLE > profiles/TAG_ncu_summary.md"""
import csv
import io
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, vals = rows[0], rows[-1]
m = dict(zip(hdr, vals))
keys = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
print(f"# {title}\n\n| metric | value |\n|---|---|")
for k in keys:
    if k in m:
        v = m[k] if k != "Kernel Name" else m[k].split("(")[0]
        print(f"| {k} | {v} |")
st = {k: v for k, v in m.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")}
print("\nWarp stall samples:\n\n| reason | samples |\n|---|---|")
for k, v in sorted(st.items(), key=lambda kv: -float(kv[1] or 0))[:8]:
    print(f"| {k.replace('smsp__pcsamp_warps_issue_stalled_', '')} | {v} |")
