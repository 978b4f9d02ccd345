"""fwbf_decode_host_f32 (the e2e path: host buffers, chunked copies pipelined
with decode -- consecutive chunks on two alternating decode streams, the
deferred-frame launches on their own stream, four chunk buffers, chunk sizes
ramping up) gives exactly the device-buffer decode's per-frame results and
counters."""
import ctypes as C

import numpy as np
import pytest

from paper_1206_3362_b200 import DecoderConfig, decode_batch
from paper_1206_3362_b200 import _native as nat
from paper_1206_3362_b200.decoders import device_code, make_params
from tests.golden.codebook import build_code, code_rate
from oracle import wbf_oracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("batch,chunk,ld_pad,z_pad", [(20000, 8192, 1, 0), (5000, 0, 0, 3), (3, 1, 5, 1),
                                                       (9000, 512, 1, 0),     # 18 chunks: every buffer reused 4 times
                                                       (3000, 128, 0, 2)])    # many short chunks
def test_host_pipeline_matches_device_decode(cuda_device, batch, chunk, ld_pad, z_pad):
    h = build_code("eg5")
    n = h.n_cols
    ld = n + ld_pad
    sigma = O.ebn0_to_sigma(4.0, code_rate("eg5"))
    rng = np.random.default_rng(batch)
    y = np.zeros((batch, ld), np.float32)
    y[:, :n] = 1.0 + sigma * rng.standard_normal((batch, n))
    if batch >= 3000:                       # frames the filtered kernel defers, spread over the chunks
        y[::97, :n] = 0.0
        y[5::211, 7] = np.inf
        y[9::173, 100] = 1e-30
    cfg = DecoderConfig(block_len_p=31, k_max=100)
    ref = decode_batch(h, y[:, :n].copy(), cfg, "fwbf")
    zw = (n + 31) // 32
    z_ld = zw + z_pad
    z = np.zeros((batch, z_ld), np.uint32)
    it = np.zeros(batch, np.int32)
    fl = np.zeros(batch, np.uint8)
    cnt = np.zeros(nat.NCOUNTERS, np.int64)
    dc = device_code(h, 0)
    prm = make_params(cfg, "fwbf")
    L = nat.lib()
    ptr = lambda a: C.c_void_p(a.ctypes.data)
    nat.check(L.fwbf_decode_host_f32(dc.handle, C.byref(prm), ptr(y), batch, ld, ptr(z), z_ld, ptr(it),
                                     ptr(fl), ptr(cnt), chunk), "decode_host")
    assert np.array_equal(it, ref.iterations.cpu().numpy())
    assert np.array_equal(fl, ref.flags.cpu().numpy())
    assert np.array_equal(z[:, :zw].view(np.int32), ref.z_bits.cpu().numpy())
    rc = ref.counters.cpu().numpy()
    assert cnt[nat.CNT_FRAMES] == batch
    assert np.array_equal(cnt, rc)
