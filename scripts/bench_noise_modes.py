import sys, time, torch, math
sys.path.insert(0,'.')
from paper_1206_3362_b200 import DecoderConfig
from paper_1206_3362_b200.decoders import decode_awgn
from tests.golden.codebook import build_code, code_rate
h=build_code('eg5'); sigma=math.sqrt(1/(2*code_rate('eg5')*10**0.4))
cfg=DecoderConfig(block_len_p=31,k_max=100)
for noise in ('f32','f64'):
    for rep in range(2):
        torch.cuda.synchronize(); t=time.perf_counter()
        r=decode_awgn(h,cfg,'fwbf',1,0,1<<18,sigma,noise=noise)
        torch.cuda.synchronize(); dt=time.perf_counter()-t
    c=r.counters.cpu().numpy()
    print(noise, 'Gbit/s', (1<<18)*781/dt/1e9, 'iters', c[3]/c[0], 'ordered', c[7])
