"""paper_2310_02410_b200 — B200-native MoQE expert-FFN path (sm_100a).

Drop-in for the reference's quantize-experts -> moe_ffn_forward path
(arXiv 2310.02410 toolkit, /root/reference/proj). See DESIGN.md.
"""
from ._lib import (CheckpointError, CudaError, InvalidArgument, MoqeError, NotSupported, OutOfRange,
                   RangeError, load as load_library)
from .api import (EXPERT_FFN, PER_CHANNEL, PER_TENSOR, ExpertBank, Mqe1, QuantizedTensor, ep_combine, ep_dispatch,
                  expert_ffn,
                  linear_scales, moe_ffn_forward, moe_ffn_forward_host, pack, packed_size,
                  quantize_linear, quantize_model, quantize_pack, route, top1_route, unpack,
                  valid_bits)

__all__ = [
    "CheckpointError", "Mqe1", "CudaError", "InvalidArgument", "MoqeError", "NotSupported", "OutOfRange", "RangeError",
    "load_library", "ep_combine", "ep_dispatch", "expert_ffn", "EXPERT_FFN", "PER_CHANNEL", "PER_TENSOR", "ExpertBank", "QuantizedTensor",
    "linear_scales", "moe_ffn_forward", "moe_ffn_forward_host", "pack", "packed_size",
    "quantize_linear", "quantize_model", "quantize_pack", "route", "top1_route", "unpack",
    "valid_bits",
]
from . import stack  # noqa: E402  (config-3 FFN stack: add_layer_norm, FfnStack)
