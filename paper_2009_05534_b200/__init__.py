"""B200-native 5G-NR LDPC layered min-sum decoder (the accelerated hot path of
arXiv 2009.05534's "Fast LDPC GPU Decoder for Cloud RAN").

Public surface mirrors the decode subset of the reference package ``ldpclab``
(/root/reference/pkg/src/ldpclab/__init__.py:44-83): ``decode``,
``DecodeConfig``, ``DecodeResult``, the enums, ``quantize``/``QuantConfig``
and the base-graph loader. Compute runs in ``libnrldpc.so`` (sm_100a CUDA
behind a C ABI, include/nrldpc.h).
"""

from .basegraph import (
    ALL_LIFTING_SIZES,
    LIFTING_SETS,
    BaseGraph,
    CodeParams,
    code_params,
    edge_tables,
    lifting_set_index,
    load_basegraph,
)
from .channel import (QuantConfig, bpsk_awgn, bpsk_exact, demap_llr, demap_quantize, ebn0_to_sigma,
                      quantize)
from .codec import crc_attach, crc_check, encode_batch, syndrome_weights
from .decoder import (
    DecodeConfig,
    DecodeResult,
    EarlyStop,
    Plan,
    Precision,
    Strategy,
    decode,
    decode_flooding,
    get_plan,
    unpack_bits,
)

__all__ = [
    "ALL_LIFTING_SIZES", "LIFTING_SETS", "BaseGraph", "CodeParams", "code_params", "edge_tables",
    "lifting_set_index", "load_basegraph", "QuantConfig", "bpsk_awgn", "bpsk_exact", "demap_llr",
    "ebn0_to_sigma", "quantize", "demap_quantize", "crc_attach", "crc_check", "encode_batch", "syndrome_weights",
    "DecodeConfig", "DecodeResult", "EarlyStop", "Plan", "Precision", "Strategy", "decode", "decode_flooding",
    "get_plan", "unpack_bits",
]
