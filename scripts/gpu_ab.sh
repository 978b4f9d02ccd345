#!/bin/bash
# A/B of an environment switch on the headline bench at several Eb/N0:
#   bash scripts/gpu_ab.sh OUT "ENV=1" "4.0 4.5 5.0" [extra bench args]
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
out=$1; envset=$2; dbs=$3; shift 3
for db in $dbs; do
  for rep in 1 2; do
    python bench.py --steps 5 --warmup 3 --ebn0 $db --no-cpu-baseline --no-e2e "$@" | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('A', $db, round(d['value'],3), round(d['ms_per_step'],2))" >> $out
    env $envset python bench.py --steps 5 --warmup 3 --ebn0 $db --no-cpu-baseline --no-e2e "$@" | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('B', $db, round(d['value'],3), round(d['ms_per_step'],2))" >> $out
  done
done
