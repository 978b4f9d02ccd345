#!/bin/bash
# full-size parity of the final kernels (frame by frame vs the C oracle)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
P=gpurun_out/r2f_parity.jsonl; : > $P
timeout 900 python scripts/parity_full.py --frames 1048576 --ebn0 4.0 >> $P
timeout 600 python scripts/parity_full.py --code gal504 --p 24 --kmax 50 --frames 65536 >> $P
timeout 600 python scripts/parity_full.py --code qc4x32 --p 256 --kmax 50 --ebn0 5.0 --frames 16384 >> $P
timeout 600 python scripts/parity_full.py --alg mlp --lam 10 --frames 262144 >> $P
timeout 900 python scripts/parity_full.py --code eg6 --p 64 --ebn0 4.0 --frames 65536 >> $P
