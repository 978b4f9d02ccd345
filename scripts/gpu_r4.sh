#!/bin/bash
# round-2 (fourth session) measurement pass: every config A-E, the headline
# contract line + reference arm, launch list and ncu captures of the headline
# (filtered circulant kernel) and of config D (incremental QC kernel)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${1:-r4a}
timeout 2400 python scripts/bench_configs.py > gpurun_out/${TAG}_configs.jsonl 2> gpurun_out/${TAG}_configs.err
echo "configs rc=$?"
bash scripts/gpu_full.sh $TAG
B="python scripts/one_qc.py"
$B > gpurun_out/plain_${TAG}qc.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on \
   -k regex:qinc -s 1 -c 1 -o gpurun_out/prof_${TAG}qc $B > gpurun_out/ncu_${TAG}qc.log 2>&1
echo "ncu qc rc=$?"
