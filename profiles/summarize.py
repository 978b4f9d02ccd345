"""Summarise ncu outputs pulled back from the GPU box into profiles/ (run here).

    python profiles/summarize.py TAG gpurun_out/launches_TAG.csv gpurun_out/prof_full_TAG.ncu-rep FRAMES
Writes profiles/TAG_launches.csv (decode kernel launches), profiles/TAG_ncu_summary.md
and updates profiles/roofline_traffic.json (dram bytes per launch, per frame).
"""
import csv
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
tag, launches, rep, frames = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])

rows = list(csv.reader(open(launches)))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
per = {}
for r in rows[start + 1:]:
    if len(r) > vi:
        per.setdefault(r[0], {"kernel": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
with open(os.path.join(HERE, f"{tag}_launches.csv"), "w") as f:
    f.write("id,kernel,gpu_time_ns,dram_read_B,dram_write_B\n")
    for i, d in per.items():
        name = d["kernel"].split("(")[0][:80]
        f.write(f"{i},{name},{d.get('gpu__time_duration.sum',0):.0f},"
                f"{d.get('dram__bytes_read.sum',0):.0f},{d.get('dram__bytes_write.sum',0):.0f}\n")
# the decode step's dominant kernel: the filtered circulant kernel when it ran
# (round 3; the decode_kernel launch after it only handles deferred frames)
dec = [d for d in per.values() if "cdecode_kernel" in d["kernel"]] or \
      [d for d in per.values() if "decode_kernel" in d["kernel"]]
tot_all = sum(d.get("gpu__time_duration.sum", 0) for d in per.values())
tot_dec = sum(d.get("gpu__time_duration.sum", 0) for d in dec)
traffic = sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in dec) / max(1, len(dec))

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
m = dict(zip(r[0], r[2])) if len(r) > 2 else {}
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem",
        "sm__sass_thread_inst_executed_op_dadd_pred_on.sum", "smsp__inst_executed.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
stalls = {k: v for k, v in m.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in k}
with open(os.path.join(HERE, f"{tag}_ncu_summary.md"), "w") as f:
    f.write(f"# ncu summary {tag}\n\nLaunch list: {len(per)} kernels, {dec[0]['kernel'].split('(')[0].split('<')[0] if dec else '-'} launches {len(dec)}, "
            f"decode share of GPU time {100*tot_dec/max(tot_all,1):.1f}% (cold-cache, serialised).\n")
    f.write(f"DRAM traffic per decode launch: {traffic/1e6:.1f} MB = {traffic/frames:.0f} B/frame "
            f"(algorithmic 4*N + 4*ceil(N/32) + 8 = 4228 B/frame for N=1023).\n\n")
    f.write(f"Full capture ({os.path.basename(rep)}), one decode launch of {frames} frames:\n\n| metric | value |\n|---|---|\n")
    for k in want:
        if k in m:
            f.write(f"| {k} | {m[k]} |\n")
    f.write("\nWarp stall samples:\n\n| reason | samples |\n|---|---|\n")
    for k, v in sorted(stalls.items(), key=lambda kv: -float(kv[1] or 0))[:12]:
        f.write(f"| {k.replace('smsp__pcsamp_warps_issue_stalled_','')} | {v} |\n")
tp = os.path.join(HERE, "roofline_traffic.json")
d = json.load(open(tp)) if os.path.exists(tp) else {}
d["eg5"] = {"dram_bytes_per_launch": traffic, "frames_per_launch": frames,
            "dram_bytes_per_frame": traffic / frames, "source": f"profiles/{tag}_launches.csv",
            "ncu_issue_active_pct": float(m.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0) or 0),
            "ncu_smem_pipe_pct": float(m.get(
                "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", 0) or 0),
            "ncu_source": f"profiles/{tag}_ncu_summary.md"}
json.dump(d, open(tp, "w"), indent=1)
print(open(os.path.join(HERE, f"{tag}_ncu_summary.md")).read())
