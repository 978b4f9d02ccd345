#!/bin/bash
# full-size parity of the fourth-session kernels (16-bit gather on the circulant
# kernel, incremental QC kernel), frame by frame vs the C oracle on the host cores
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
P=gpurun_out/r4_parity.jsonl; : > $P
timeout 900 python scripts/parity_full.py --frames 1048576 --ebn0 4.0 >> $P
timeout 600 python scripts/parity_full.py --frames 262144 --ebn0 5.0 >> $P
timeout 900 python scripts/parity_full.py --frames 262144 --ebn0 3.0 >> $P
timeout 600 python scripts/parity_full.py --p 93 --frames 262144 --ebn0 4.0 >> $P
timeout 900 python scripts/parity_full.py --code eg6 --p 64 --ebn0 4.0 --frames 65536 >> $P
timeout 900 python scripts/parity_full.py --code eg6 --p 256 --ebn0 4.5 --frames 65536 >> $P
timeout 900 python scripts/parity_full.py --code eg4 --p 17 --ebn0 4.0 --frames 262144 >> $P
timeout 1200 python scripts/parity_full.py --code qc4x32 --p 256 --ebn0 5.0 --kmax 50 --frames 65536 >> $P
timeout 900 python scripts/parity_full.py --code qc4x32 --p 64 --ebn0 6.0 --kmax 50 --frames 32768 >> $P
cat $P | cut -c1-330
