"""B200-native batched weighted bit-flipping (WBF) LDPC decoding.

Drop-in for the decode path of the reference package `fwbf`
(/root/reference/pkg/src/fwbf): the same decoder entry points and config
objects, executed by hand-written sm_100a CUDA kernels behind the C ABI in
include/fwbf_b200.h (libfwbf_b200.so, built in-tree).
"""

from .codes import (ParityCheckMatrix, eg_ldpc, qc_ldpc, gallager_rc, gf2_rank, validate_rc,
                    read_alist, write_alist, detect_structure, code_dimension)
from .decoders import (DecoderConfig, DecodeOutcome, DecodeState, BatchResult, decode_batch,
                       decode_fwbf, decode_imwbf, decode_mlp_wbf, device_code, pack_bits)

__version__ = "0.1.0"
