import sys, math; sys.path.insert(0,'.')
import torch
from paper_1206_3362_b200 import DecoderConfig
from paper_1206_3362_b200.decoders import decode_awgn
from tests.golden.codebook import build_code, code_rate
h=build_code('eg5'); s=math.sqrt(1/(2*code_rate('eg5')*10**0.4))
r=decode_awgn(h, DecoderConfig(block_len_p=31,k_max=100), 'fwbf', 1, 0, 65536, s, noise='f32'); torch.cuda.synchronize(); print('ok')
