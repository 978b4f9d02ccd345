#!/bin/bash
# round-2 closing measurement: headline bench + reference arm + launch list +
# ncu captures of the headline (MODE 2), config A (warp kernel) and D (QC kernel)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
bash scripts/gpu_full.sh r2e
for cfg in "A --code gal504 --p 24 --kmax 50 --frames 65536" "D --code qc4x32 --p 256 --kmax 50 --ebn0 5.0 --frames 4096"; do
  set -- $cfg; tag=r2e$1; shift
  B="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline $*"
  $B > gpurun_out/plain_$tag.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on \
    -k regex:"xdecode|qdecode" -s 1 -c 1 -o gpurun_out/prof_$tag $B > gpurun_out/ncu_$tag.log 2>&1
  echo "ncu $tag rc=$?" >> gpurun_out/ncu_$tag.log
done
