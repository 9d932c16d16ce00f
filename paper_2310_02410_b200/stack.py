"""Pre-LN residual FFN stack (BASELINE config 3) on the GPU.

Host-side mirror of the reference's run_stack (/root/reference/proj/src/model.cpp:419-435)
without attention: for every layer i, fn = layer_norm(x, ln_ffn_i) (model.cpp:193-212) and
x += ffn_block_i(fn) (add_inplace, model.cpp:308-310), where ffn_block is moe_ffn_forward for
MoE layers (model.cpp:399-417) and dense_ffn (model.cpp:315-322) otherwise; then the final
layer_norm. The residual add is fused into the next normalisation (moqe_gpu_add_layer_norm),
MoE layers run the package's expert-FFN kernels, and the dense fp16 FFNs are plain library
GEMMs (cuBLAS through torch: fp16 operands, fp32 accumulation), which the task allows for
plain GEMMs.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

import torch

from . import _lib
from ._lib import check
from .api import ExpertBank, moe_ffn_forward


def add_layer_norm(x: torch.Tensor, delta: Optional[torch.Tensor], gain: torch.Tensor, bias: torch.Tensor,
                   out: Optional[torch.Tensor] = None, out_dtype: torch.dtype = torch.float32) -> torch.Tensor:
    """x += delta (in place, when given); return layer_norm(x, gain, bias) (eps 1e-5)."""
    if x.dtype != torch.float32 or not x.is_cuda or not x.is_contiguous():
        raise _lib.InvalidArgument("layer_norm: x must be a contiguous f32 CUDA tensor")
    rows, n = x.shape
    if delta is not None:
        delta = delta.to(torch.float32).contiguous()
        if tuple(delta.shape) != (rows, n):
            raise _lib.InvalidArgument("add_inplace: shape mismatch")
    gain = gain.to(torch.float32).contiguous()
    bias = bias.to(torch.float32).contiguous()
    if out is None:
        out = torch.empty((rows, n), dtype=out_dtype, device=x.device)
    check(_lib.load().moqe_gpu_add_layer_norm(
        x.data_ptr(), None if delta is None else delta.data_ptr(), rows, n, gain.data_ptr(), bias.data_ptr(),
        out.data_ptr(), _lib.F16 if out.dtype == torch.float16 else _lib.F32,
        torch.cuda.current_stream().cuda_stream))
    return out


def layer_norm(x: torch.Tensor, gain: torch.Tensor, bias: torch.Tensor) -> torch.Tensor:
    """moqe layer_norm (model.cpp:193-212) of a copy of x."""
    return add_layer_norm(x.to(torch.float32).contiguous().clone(), None, gain, bias)


@dataclass
class DenseFFN:
    """dense_ffn (model.cpp:315-322) with fp16 weights: relu(x W1 + b1) W2 + b2."""
    w1: torch.Tensor  # [d, f] fp16
    w2: torch.Tensor  # [f, d] fp16
    b1: Optional[torch.Tensor] = None  # [f] f32
    b2: Optional[torch.Tensor] = None  # [d] f32

    def __call__(self, x: torch.Tensor) -> torch.Tensor:
        h = x.to(torch.float16) @ self.w1
        if self.b1 is not None:
            h = h + self.b1.to(torch.float16)
        h = torch.relu_(h)
        y = (h @ self.w2).to(torch.float32)
        if self.b2 is not None:
            y = y + self.b2
        return y


@dataclass
class StackLayer:
    gain: torch.Tensor
    bias: torch.Tensor
    moe: Optional[ExpertBank] = None  # MoE layer: the bank (with its router set)
    dense: Optional[DenseFFN] = None
    top_k: int = 1


class FfnStack:
    """run_stack without attention over `layers`, then the final layer_norm."""

    def __init__(self, layers: List[StackLayer], final_gain: torch.Tensor, final_bias: torch.Tensor):
        self.layers = layers
        self.final_gain = final_gain
        self.final_bias = final_bias

    def forward(self, x: torch.Tensor, return_routing: bool = False):
        """x [T, d] (any float dtype). Returns the final layer_norm output [T, d] f32 (and the
        expert ids of every MoE layer when return_routing)."""
        x = x.to(torch.float32).contiguous().clone()  # the residual stream
        delta = None
        routing = []
        for L in self.layers:
            fn = add_layer_norm(x, delta, L.gain, L.bias)
            if L.moe is not None:
                if return_routing:
                    delta, ex, _ = moe_ffn_forward(fn, L.moe, top_k=L.top_k, return_routing=True)
                    routing.append(ex)
                else:
                    delta = moe_ffn_forward(fn, L.moe, top_k=L.top_k)
            else:
                delta = L.dense(fn)
        out = add_layer_norm(x, delta, self.final_gain, self.final_bias)
        return (out, routing) if return_routing else out
