#!/bin/bash
# interleaved A/B of two library builds (FWBF_LIB) at several Eb/N0
#   bash scripts/gpu_ab2.sh LIB_A LIB_B "4.0 5.0" [reps] [bench args]
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
A=$1; B=$2; DBS=$3; R=${4:-2}; shift 4
mkdir -p gpurun_out
for db in $DBS; do
  for rep in $(seq $R); do
    for L in $A $B; do
      FWBF_LIB=$PWD/$L timeout 300 python bench.py --steps 3 --warmup 3 --ebn0 $db --no-cpu-baseline --no-e2e "$@" > gpurun_out/ab2.log 2>&1
      python -c "import json; d=json.loads(open('gpurun_out/ab2.log').read().strip().splitlines()[-1]); print('$L', $db, round(d['value'],3), round(d['ms_per_step'],2), round(d['config']['mean_iters'],3))" || tail -3 gpurun_out/ab2.log
    done
  done
done
