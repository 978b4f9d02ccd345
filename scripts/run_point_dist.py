"""BER/FER of one SNR point on all GPUs of a node (the reference's run_point,
sharded):  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
                scripts/run_point_dist.py [--ebn0 4.0] [--frames 1000000] [--target 100]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

from paper_1206_3362_b200 import DecoderConfig, eg_ldpc
from paper_1206_3362_b200.harness import ExperimentConfig, format_summary, run_point

ap = argparse.ArgumentParser()
ap.add_argument("--ebn0", type=float, default=4.0)
ap.add_argument("--frames", type=int, default=1 << 20)
ap.add_argument("--target", type=int, default=100)
ap.add_argument("--p", type=int, default=31)
a = ap.parse_args()
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
if int(os.environ.get("WORLD_SIZE", "1")) > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
cfg = ExperimentConfig(h=eg_ldpc(5), decoder="fwbf", decoder_cfg=DecoderConfig(block_len_p=a.p, k_max=100),
                       ebn0_db=(a.ebn0,), target_word_errors=a.target, max_frames=a.frames)
st = run_point(cfg, a.ebn0)
if int(os.environ.get("RANK", "0")) == 0:
    print(format_summary([st]))
if dist.is_initialized():
    dist.destroy_process_group()
