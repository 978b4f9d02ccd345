"""BPSK over AWGN: the reference channel's API plus its batched device form.

Same names and semantics as `/root/reference/pkg/src/fwbf/channel.py`:

  bpsk_modulate   channel.py:11-16   s = 1 - 2c (ValueError for non-binary c)
  ebn0_to_sigma   channel.py:19-26
  awgn_apply      channel.py:29-36   s + sigma * rng.standard_normal(N)
  frame_rng       channel.py:39-50   Philox(key=seed, counter=frame << 128)
  ChannelParams   channel.py:53-62
  ReceivedFrame   channel.py:65-74
  transmit        channel.py:77-82

The per-frame functions take and return numpy values and a numpy Generator,
because that is their contract (a caller hands ``awgn_apply`` its own rng).
The Monte Carlo path does not use them: `awgn_batch` (and the decoder's
`decode_awgn`) draws the same stream for whole frame ranges on the device
(csrc/fwbf_noise.cuh, a replay of numpy's Philox4x64 + ziggurat), which is
what `harness.run_point` runs on.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat


def bpsk_modulate(c) -> np.ndarray:
    """s_n = 1 - 2 c_n (float64)."""
    bits = np.asarray(c)
    if np.any((bits < 0) | (bits > 1)):
        raise ValueError("codeword entries must be 0 or 1")
    return 1.0 - 2.0 * bits.astype(np.float64)


def ebn0_to_sigma(ebn0_db: float, rate: float) -> float:
    """sigma = sqrt(1 / (2 R 10^(EbN0/10))) for unit symbol energy."""
    if not (0.0 < rate < 1.0):
        raise ValueError(f"code rate must be in (0, 1), got {rate}")
    ebn0 = 10.0 ** (ebn0_db / 10.0)
    return math.sqrt(1.0 / (2.0 * rate * ebn0))


def awgn_apply(s, sigma: float, rng: np.random.Generator) -> np.ndarray:
    """s + sigma * N(0, 1) draws from `rng` (a copy of s when sigma == 0)."""
    if sigma < 0:
        raise ValueError("sigma must be nonnegative")
    sym = np.array(s, dtype=np.float64)  # a copy
    if sigma != 0:
        sym += sigma * rng.standard_normal(sym.size)
    return sym


def frame_rng(master_seed: int, frame_index: int) -> np.random.Generator:
    """The stream of one frame: Philox keyed by the seed, counter frame << 128
    (disjoint counter blocks per frame)."""
    if master_seed < 0 or frame_index < 0:
        raise ValueError("seed and frame index must be nonnegative")
    return np.random.Generator(np.random.Philox(key=master_seed, counter=frame_index << 128))


@dataclass(frozen=True)
class ChannelParams:
    """Eb/N0 operating point and the sigma it implies at a code rate."""

    ebn0_db: float
    rate: float
    sigma: float = field(default=None)  # type: ignore[assignment]

    def __post_init__(self):
        if self.sigma is None:
            object.__setattr__(self, "sigma", ebn0_to_sigma(self.ebn0_db, self.rate))


@dataclass
class ReceivedFrame:
    """Channel output y and the codeword that produced it."""

    y: np.ndarray
    source_codeword: np.ndarray

    def __post_init__(self):
        if len(self.y) != len(self.source_codeword):
            raise ValueError("y and source codeword lengths differ")


def transmit(codeword, sigma: float, rng: np.random.Generator) -> ReceivedFrame:
    """Modulate and pass through the AWGN channel."""
    word = np.asarray(codeword, dtype=np.uint8)
    y = awgn_apply(bpsk_modulate(word), sigma, rng)
    return ReceivedFrame(y=y, source_codeword=word)


def awgn_batch(h, seed: int, first_frame: int, count: int, sigma: float, *, codeword=None,
               noise: str = "f64", device=None):
    """Channel output of frames [first_frame, first_frame + count) on the device:
    row f equals ``transmit(codeword, sigma, frame_rng(seed, first_frame + f)).y``
    (float64, noise="f64") or that value rounded to float32 (noise="f32").
    Returns a [count, N] CUDA tensor."""
    import torch
    from .decoders import device_code, pack_bits
    if seed < 0 or first_frame < 0:
        raise ValueError("seed and frame index must be nonnegative")
    if seed >= 1 << 64:
        raise ValueError("seed must be below 2**64")
    if sigma < 0:
        raise ValueError("sigma must be nonnegative")
    if noise not in ("f64", "f32"):
        raise ValueError("noise must be 'f64' or 'f32'")
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    with torch.cuda.device(dev):
        dc = device_code(h, dev.index if dev.index is not None else 0)
    cw_t = None
    if codeword is not None:
        c = np.asarray(codeword)
        if c.size and (c.min() < 0 or c.max() > 1):
            raise ValueError("codeword entries must be 0 or 1")
        cw_t = torch.from_numpy(pack_bits(c, dc.n).view(np.int32)).to(dev)
    y = torch.empty((int(count), dc.n), dtype=torch.float64 if noise == "f64" else torch.float32, device=dev)
    mode = nat.NOISE_NUMPY_F64 if noise == "f64" else nat.NOISE_NUMPY_F32
    st = torch.cuda.current_stream(dev)
    nat.check(nat.lib().fwbf_channel_awgn(dc.handle, C.c_uint64(int(seed)), int(first_frame), int(count),
                                            float(sigma), cw_t.data_ptr() if cw_t is not None else None, mode,
                                            y.data_ptr(), dc.n, C.c_void_p(st.cuda_stream)), "channel_awgn")
    y._fwbf_keep = cw_t  # codeword words stay alive until the stream has read them
    return y
