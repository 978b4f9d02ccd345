"""B200-native batched weighted bit-flipping (WBF) LDPC decoding.

Drop-in for the decode path of the reference package `fwbf`
(/root/reference/pkg/src/fwbf): the same decoder entry points, stage
functions, channel and harness API and config objects (reference
``__init__.py:9-28``), executed by hand-written sm_100a CUDA kernels behind
the C ABI in include/fwbf_b200.h (libfwbf_b200.so, built in-tree).
"""

from .codes import (AlistError, AlistFormatError, AlistMismatchError, AlistRangeError, CodeSpec,
                    ParityCheckMatrix, RcReport, code_dimension, code_spec, detect_structure, eg_ldpc,
                    gallager_rc, gf2_rank, qc_ldpc, read_alist, validate_rc, write_alist)
from .channel import (ChannelParams, ReceivedFrame, awgn_apply, awgn_batch, bpsk_modulate, ebn0_to_sigma,
                      frame_rng, transmit)
from .decoders import (BatchResult, DecodeOutcome, DecoderConfig, DecodeState, decode_awgn, decode_batch,
                       decode_fwbf, decode_imwbf, decode_mlp_wbf, device_code, pack_bits)
from .stage import (WeightTable, all_metrics, bit_metric, block_argmax, compute_weights, hard_decision,
                    syndrome)
from .harness import (ExperimentConfig, PointStats, SweepResult, run_experiment, run_point, sweep_alpha,
                      write_csv)

__version__ = "0.1.0"
