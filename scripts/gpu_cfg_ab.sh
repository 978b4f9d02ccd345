#!/bin/bash
# configs (bench_configs.py --only X) with and without the filtered circulant kernel
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for only in ${ONLY:-C B}; do
  for envs in ${VARIANTS:-FWBF_NO_CDEC=1 FWBF_DUMMY=1}; do
    env $envs timeout 900 python scripts/bench_configs.py ${QUICK:---quick} --only $only > gpurun_out/cfg_$only.jsonl 2> gpurun_out/cfg_$only.err
    python - "$envs" "$only" <<'PY'
import json,sys
for l in open(f"gpurun_out/cfg_{sys.argv[2]}.jsonl"):
    d=json.loads(l); print(sys.argv[1], d['config'], d.get('p'), d['ebn0_db'], d.get('algorithm'), round(d['info_gbit_s'],3), round(d.get('mean_iters',0),2))
PY
  done
done
