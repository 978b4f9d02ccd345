#!/bin/bash
# full-size parity of the round-3 filtered circulant kernel (frame by frame vs the C oracle)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
P=gpurun_out/r3_parity.jsonl; : > $P
timeout 900 python scripts/parity_full.py --frames 1048576 --ebn0 4.0 >> $P
timeout 600 python scripts/parity_full.py --frames 262144 --ebn0 5.0 >> $P
timeout 900 python scripts/parity_full.py --frames 262144 --ebn0 3.0 >> $P
timeout 600 python scripts/parity_full.py --p 93 --frames 262144 --ebn0 4.0 >> $P
timeout 900 python scripts/parity_full.py --code eg6 --p 64 --ebn0 4.0 --frames 65536 >> $P
timeout 900 python scripts/parity_full.py --code eg6 --p 256 --ebn0 4.5 --frames 65536 >> $P
cat $P | cut -c1-300
