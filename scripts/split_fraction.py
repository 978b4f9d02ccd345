import sys, numpy as np, torch
sys.path.insert(0,'.')
from paper_1206_3362_b200 import DecoderConfig
from paper_1206_3362_b200.decoders import metric_batch
from paper_1206_3362_b200 import _native as nat
from tests.golden.codebook import build_code, code_rate
from oracle import wbf_oracle as O
for code, db in (("eg5",4.0),("eg6",4.0),("eg6",3.5)):
    h=build_code(code); s=O.ebn0_to_sigma(db, code_rate(code))
    y=(1+s*torch.randn((4096,h.n_cols),device='cuda')).float()
    E,fl=metric_batch(h,y,DecoderConfig(block_len_p=64))
    fl=fl.cpu().numpy()
    print(code, db, "split", np.mean((fl&16)!=0), "ordered", np.mean((fl&4)!=0))
