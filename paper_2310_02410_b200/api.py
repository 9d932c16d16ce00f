"""Python mirror of the reference's public API for the MoQE expert-FFN path.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/moqe/*.hpp), on CUDA tensors. Every call goes
through the C-ABI (include/moqe_gpu.h) into hand-written sm_100a kernels; torch
only provides device memory and the current stream.

  reference (moqe::)                          here
  -----------------------------------------   ---------------------------------
  packed_size   bitpack.hpp:25                packed_size
  pack / unpack bitpack.hpp:28-31             pack / unpack
  linear_scales quant.hpp:48                  linear_scales
  quantize_linear quant.hpp:50                quantize_linear (-> QuantizedTensor)
  dequantize    quant.hpp:64                  (not on the path: experts are never
                                               materialised)
  top1_route    model.hpp:65                  top1_route / route (top-1, top-2)
  ExpertBank    model.hpp:80-82               ExpertBank (device resident)
  moe_ffn_forward model.hpp:87                moe_ffn_forward
  quantize_model  model.hpp:109-113           quantize_model (expert recipe)
"""
from __future__ import annotations

import ctypes as C
import sys
from dataclasses import dataclass, field
from typing import Dict, Iterable, Optional, Tuple

import torch

from . import _lib
from ._lib import check

PER_CHANNEL = "channel"
PER_TENSOR = "tensor"
_GRAN = {PER_CHANNEL: _lib.PER_CHANNEL, PER_TENSOR: _lib.PER_TENSOR}
_PATH = {"auto": _lib.PATH_AUTO, "gemv": _lib.PATH_GEMV, "gemm": _lib.PATH_GEMM}


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _dev(t: torch.Tensor, dtype: torch.dtype, what: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise _lib.InvalidArgument(f"{what}: expected a CUDA tensor")
    return t.to(dtype).contiguous()


def valid_bits(bits: int) -> bool:
    return bits in (2, 3, 4, 8)


def packed_size(bits: int, count: int) -> int:
    """moqe::packed_size (bitpack.cpp:12-16)."""
    lib = _lib.load()
    n = lib.moqe_gpu_packed_size(bits, count)
    if n == C.c_size_t(-1).value:
        raise _lib.InvalidArgument(f"bitpack: unsupported width {bits}")
    return int(n)


def pack(codes: torch.Tensor, bits: int) -> torch.Tensor:
    """moqe::pack (bitpack.cpp:18-39): offset binary, LSB-first, 3-bit groups."""
    c = _dev(codes, torch.int8, "pack").reshape(-1)
    n = packed_size(bits, c.numel())
    out = torch.empty(max(n, 1), dtype=torch.uint8, device=c.device)
    check(_lib.load().moqe_gpu_pack(_ptr(c), c.numel(), bits, _ptr(out), _stream()))
    return out[:n]


def unpack(data: torch.Tensor, bits: int, count: int) -> torch.Tensor:
    """moqe::unpack (bitpack.cpp:41-68)."""
    d = _dev(data, torch.uint8, "unpack").reshape(-1)
    out = torch.empty(max(count, 1), dtype=torch.int8, device=d.device)
    check(_lib.load().moqe_gpu_unpack(_ptr(d), d.numel(), bits, count, _ptr(out), _stream()))
    return out[:count]


def _as_batch(a: torch.Tensor, what: str) -> Tuple[torch.Tensor, int, int, int]:
    a = _dev(a, torch.float32, what)
    if a.dim() == 2:
        return a, 1, a.shape[0], a.shape[1]
    if a.dim() == 3:
        return a, a.shape[0], a.shape[1], a.shape[2]
    raise _lib.InvalidArgument("quant: tensor must be 2D")


def linear_scales(a: torch.Tensor, bits: int, granularity: str = PER_CHANNEL) -> torch.Tensor:
    """moqe::linear_scales (quant.cpp:59-69); a is [K,N] or a batch [B,K,N]."""
    a, B, K, N = _as_batch(a, "linear_scales")
    g = _GRAN[granularity]
    ns = 1 if g == _lib.PER_TENSOR else N
    s = torch.empty((B, ns), dtype=torch.float32, device=a.device)
    check(_lib.load().moqe_gpu_linear_scales(_ptr(a), B, K, N, bits, g, _ptr(s), _stream()))
    return s[0] if a.dim() == 2 else s


@dataclass
class QuantizedTensor:
    """moqe::QuantizedTensor (quant.hpp:22-35), linear scheme, on the device."""
    bits: int
    granularity: str
    shape: Tuple[int, int]
    codes: torch.Tensor          # int8, one per code (CodeArray)
    scales: torch.Tensor         # f32 binary16 values, [N] or [1]
    packed: Optional[torch.Tensor] = None  # reference byte layout

    scheme: str = field(default="linear")


def quantize_linear(a: torch.Tensor, bits: int, granularity: str = PER_CHANNEL):
    """moqe::quantize_linear (quant.cpp:71-95). Batched input returns a list."""
    a3, B, K, N = _as_batch(a, "quantize_linear")
    g = _GRAN[granularity]
    ns = 1 if g == _lib.PER_TENSOR else N
    codes = torch.empty((B, K, N), dtype=torch.int8, device=a3.device)
    scales = torch.empty((B, ns), dtype=torch.float32, device=a3.device)
    psz = packed_size(bits, K * N) if valid_bits(bits) else 0
    packed = torch.empty((B, max(psz, 1)), dtype=torch.uint8, device=a3.device)
    check(_lib.load().moqe_gpu_quantize_pack(_ptr(a3), B, K, N, bits, g, _ptr(packed), _ptr(scales),
                                             _ptr(codes), _stream()))
    qts = [QuantizedTensor(bits, granularity, (K, N), codes[i], scales[i], packed[i, :psz])
           for i in range(B)]
    return qts[0] if a3.dim() == 2 else qts


def quantize_pack(a: torch.Tensor, bits: int, granularity: str = PER_CHANNEL):
    """Fused quantize + pack over a batch [B,K,N] -> (packed [B, psz] u8, scales [B, N] f32)."""
    a3, B, K, N = _as_batch(a, "quantize_pack")
    g = _GRAN[granularity]
    ns = 1 if g == _lib.PER_TENSOR else N
    psz = packed_size(bits, K * N)
    packed = torch.empty((B, max(psz, 1)), dtype=torch.uint8, device=a3.device)
    scales = torch.empty((B, ns), dtype=torch.float32, device=a3.device)
    check(_lib.load().moqe_gpu_quantize_pack(_ptr(a3), B, K, N, bits, g, _ptr(packed), _ptr(scales),
                                             None, _stream()))
    return packed[:, :psz], scales


def route(h: torch.Tensor, gate_weights: torch.Tensor, top_k: int = 1):
    """top1_route (model.cpp:328-346) generalised to top-2 with renormalised gates.

    Returns (expert int32 [T] or [T,2], gate f32 [T] or [T,2])."""
    if gate_weights is None:
        raise _lib.InvalidArgument("top1_route: no gate weights")
    hd = h.dtype if h.dtype in (torch.float16, torch.float32) else torch.float32
    h = _dev(h, hd, "top1_route")
    wg = _dev(gate_weights, torch.float32, "top1_route")
    if h.dim() != 2 or wg.dim() != 2 or wg.shape[0] != h.shape[1]:
        raise _lib.InvalidArgument("matmul: shape mismatch")
    T, E = h.shape[0], wg.shape[1]
    ex = torch.empty((max(T, 1) * top_k,), dtype=torch.int32, device=h.device)
    gt = torch.empty((max(T, 1) * top_k,), dtype=torch.float32, device=h.device)
    check(_lib.load().moqe_gpu_route(_ptr(h), _lib.F16 if hd == torch.float16 else _lib.F32, T,
                                     h.shape[1], _ptr(wg), E, top_k, _ptr(ex), _ptr(gt), _stream()))
    shape = (T,) if top_k == 1 else (T, top_k)
    return ex[: T * top_k].reshape(shape), gt[: T * top_k].reshape(shape)


def ep_dispatch(h: torch.Tensor, expert: torch.Tensor, gate: torch.Tensor, n_experts: int, world: int):
    """Expert-parallel dispatch on the device (moqe_gpu_ep_dispatch; the sharded gather of
    model.cpp:360-364). Returns (records [T*k, d+4] f16, pos [T*k] i32, send_counts [world]
    i64, err [1] i32): records ordered by owner rank (stable), pos = record row per
    (token, slot). No host sync."""
    T, d = h.shape
    k = 1 if expert.dim() == 1 else expert.shape[1]
    h = _dev(h, torch.float16, "ep_dispatch")
    ex = _dev(expert.reshape(-1), torch.int32, "ep_dispatch")
    gt = _dev(gate.reshape(-1), torch.float32, "ep_dispatch")
    rec = torch.empty((T * k, d + 4), dtype=torch.float16, device=h.device)
    pos = torch.empty((T * k,), dtype=torch.int32, device=h.device)
    counts = torch.empty((world,), dtype=torch.int64, device=h.device)
    err = torch.empty((1,), dtype=torch.int32, device=h.device)
    check(_lib.load().moqe_gpu_ep_dispatch(_ptr(h), T, d, _ptr(ex), _ptr(gt), k, n_experts, world,
                                           _ptr(rec), _ptr(pos), _ptr(counts), _ptr(err), _stream()))
    return rec, pos, counts, err


def ep_combine(back: torch.Tensor, pos: torch.Tensor, T: int, top_k: int) -> torch.Tensor:
    """out[t] = 0 + back[pos[t,0]] (+ back[pos[t,1]]) in fp32 (moqe_gpu_ep_combine; the
    scatter of model.cpp:387-390 over the returned rows)."""
    if back.dtype not in (torch.float16, torch.float32):
        raise _lib.InvalidArgument("ep_combine: rows must be f16 or f32")
    back = _dev(back, back.dtype, "ep_combine")
    d = back.shape[1]
    out = torch.empty((T, d), dtype=torch.float32, device=back.device)
    check(_lib.load().moqe_gpu_ep_combine(_ptr(back), _lib.F16 if back.dtype == torch.float16 else _lib.F32,
                                          _ptr(pos), T, top_k, d, _ptr(out), _stream()))
    return out


def top1_route(h: torch.Tensor, gate_weights: torch.Tensor):
    """moqe::top1_route (model.hpp:65)."""
    return route(h, gate_weights, 1)


class ExpertBank:
    """Device-resident moqe::ExpertBank of linear-quantized experts (model.hpp:74-82).

    W1_e [d_model x d_ffn], W2_e [d_ffn x d_model], per-output-channel scales,
    optional biases. Weights are uploaded once (reference packed bytes) and
    re-tiled on the device; forwards never re-quantize or materialise them."""

    def __init__(self, n_experts: int, d_model: int, d_ffn: int, bits: int,
                 packed_w1: torch.Tensor, scales1: torch.Tensor, packed_w2: torch.Tensor,
                 scales2: torch.Tensor, b1: Optional[torch.Tensor] = None,
                 b2: Optional[torch.Tensor] = None, router: Optional[torch.Tensor] = None,
                 granularity: str = PER_CHANNEL, scheme: str = "linear"):
        """granularity: PER_CHANNEL (scales1 [E, d_ffn], scales2 [E, d_model]) or PER_TENSOR
        (one scale per expert matrix: scales [E] or [E, 1]; quant.cpp:53-55). scheme: "linear"
        (code * s) or "log" (quantize_log's sign + exponent fields, +-s * 2^-k; quant.cpp:97-243)."""
        if scheme not in ("linear", "log"):
            raise _lib.InvalidArgument("bank: scheme must be 'linear' or 'log'")
        self.E, self.d, self.f, self.bits = n_experts, d_model, d_ffn, bits
        lib = _lib.load()
        dev = packed_w1.is_cuda
        conv = (lambda t, dt: t.to(dt).contiguous()) if dev else (lambda t, dt: t.to(dt).contiguous().cpu())
        keep = [conv(packed_w1, torch.uint8), conv(scales1, torch.float32),
                conv(packed_w2, torch.uint8), conv(scales2, torch.float32),
                None if b1 is None else conv(b1, torch.float32),
                None if b2 is None else conv(b2, torch.float32)]
        h = C.c_void_p()
        check(lib.moqe_gpu_bank_create_ex(n_experts, d_model, d_ffn, bits,
                                          _lib.SCHEME_LOG if scheme == "log" else _lib.SCHEME_LINEAR,
                                          _GRAN[granularity], *[_ptr(t) for t in keep], 1 if dev else 0,
                                          C.byref(h)))
        self._h = h
        torch.cuda.synchronize()
        if router is not None:
            self.set_router(router)

    @classmethod
    def from_float(cls, w1: torch.Tensor, w2: torch.Tensor, bits: int,
                   b1: Optional[torch.Tensor] = None, b2: Optional[torch.Tensor] = None,
                   router: Optional[torch.Tensor] = None, granularity: str = PER_CHANNEL) -> "ExpertBank":
        """Quantize-experts on the GPU (linear, per channel or per tensor) then build the bank."""
        E, d, f = w1.shape
        p1, s1 = quantize_pack(w1, bits, granularity)
        p2, s2 = quantize_pack(w2, bits, granularity)
        return cls(E, d, f, bits, p1, s1, p2, s2, b1, b2, router, granularity)

    @classmethod
    def from_mqe1(cls, path: str, layer: str, n_experts: int) -> "ExpertBank":
        """The bank of one MoE layer straight from an MQE1 container (checkpoint.cpp:312-413):
        "<layer>.expert.<e>.fc{1,2}.w" q-lin blobs copied to the device as stored, optional biases,
        and "<layer>.router.w" as the router when present."""
        lib = _lib.load()
        with Mqe1(path) as m:
            h = C.c_void_p()
            check(lib.moqe_gpu_mqe1_bank_create(m._h, layer.encode(), n_experts, C.byref(h)))
        bank = cls.__new__(cls)
        bank._h = h
        info = {e["name"]: e for e in Mqe1(path).entries()}
        w1 = info[f"{layer}.expert.0.fc1.w"]
        bank.E, bank.d, bank.f, bank.bits = n_experts, int(w1["shape"][0]), int(w1["shape"][1]), int(w1["bits"])
        torch.cuda.synchronize()
        return bank

    def set_router(self, wg: torch.Tensor) -> None:
        wg = wg.to(torch.float32).contiguous()
        check(_lib.load().moqe_gpu_bank_set_router(self._h, _ptr(wg), 1 if wg.is_cuda else 0))

    @property
    def handle(self) -> int:
        return self._h.value

    def weight_bytes(self) -> int:
        return int(_lib.load().moqe_gpu_bank_weight_bytes(self._h))

    def trace(self, enable: bool = True) -> None:
        """Enable / disable the decode kernel's device event trace (diagnostics)."""
        check(_lib.load().moqe_gpu_bank_trace(self._h, 1 if enable else 0))

    def trace_read(self):
        """Trace since the last read: (gemv [num_sms, 512, 2] of (time ns, event word),
        router [64, 16] of per-CTA stamps: 0 start, 1 row loaded, 2..9 chunk c done,
        10 chain done, 11 ticket, 12 plan done)."""
        import numpy as np
        lib = _lib.load()
        n = int(lib.moqe_gpu_bank_trace_read(self._h, None, 0))
        if n < 0:
            raise _lib.InvalidArgument("trace: tracing is not enabled")
        buf = np.zeros(n, np.uint64)
        lib.moqe_gpu_bank_trace_read(self._h, buf.ctypes.data, n)
        nr = 64 * 16
        return buf[: n - nr].reshape(-1, 512, 2), buf[n - nr:].reshape(64, 16)

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            _lib.load().moqe_gpu_bank_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            if sys.is_finalizing():
                return
            self.close()
        except Exception:
            pass


class _Mqe1Info(C.Structure):
    _fields_ = [("name", C.c_char * 128), ("group", C.c_char * 32), ("dtype", C.c_char * 8), ("bits", C.c_int),
                ("per_tensor", C.c_int), ("ndim", C.c_int), ("shape", C.c_int64 * 4), ("data_offset", C.c_uint64),
                ("data_bytes", C.c_uint64), ("scale_offset", C.c_uint64), ("scale_bytes", C.c_uint64)]


class Mqe1:
    """A mapped MQE1 container (read_checkpoint's index validation, checkpoint.cpp:312-392)."""

    def __init__(self, path: str):
        self._h = C.c_void_p()
        check(_lib.load().moqe_gpu_mqe1_open(str(path).encode(), C.byref(self._h)))

    def entries(self):
        lib = _lib.load()
        out = []
        for i in range(int(lib.moqe_gpu_mqe1_count(self._h))):
            inf = _Mqe1Info()
            check(lib.moqe_gpu_mqe1_entry(self._h, i, C.byref(inf)))
            out.append({"name": inf.name.decode(), "group": inf.group.decode(), "dtype": inf.dtype.decode(),
                        "bits": inf.bits, "granularity": PER_TENSOR if inf.per_tensor else PER_CHANNEL,
                        "shape": tuple(inf.shape[k] for k in range(inf.ndim)), "data_offset": inf.data_offset,
                        "data_bytes": inf.data_bytes, "scale_offset": inf.scale_offset,
                        "scale_bytes": inf.scale_bytes})
        return out

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib.load().moqe_gpu_mqe1_close(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            if not sys.is_finalizing():
                self.close()
        except Exception:
            pass


def moe_ffn_forward(h: torch.Tensor, bank: ExpertBank, gate_weights: Optional[torch.Tensor] = None,
                    top_k: int = 1, out_dtype: torch.dtype = torch.float32, path: str = "auto",
                    return_routing: bool = False, out: Optional[torch.Tensor] = None):
    """moqe::moe_ffn_forward (model.cpp:348-393) on the GPU.

    h [T, d_model] f32/f16 CUDA tensor; gate_weights [d_model, E] (None: the
    bank's router). Returns out [T, d_model] (out_dtype), plus (expert, gate)
    when return_routing."""
    if bank is None:
        raise _lib.InvalidArgument("moe_ffn_forward: empty expert bank")
    hd = h.dtype if h.dtype in (torch.float16, torch.float32) else torch.float32
    h = _dev(h, hd, "moe_ffn_forward")
    if h.dim() != 2 or h.shape[1] != bank.d:
        raise _lib.InvalidArgument("matmul: shape mismatch")
    T = h.shape[0]
    wg = None if gate_weights is None else _dev(gate_weights, torch.float32, "moe_ffn_forward")
    if wg is not None and tuple(wg.shape) != (bank.d, bank.E):
        raise _lib.InvalidArgument("matmul: shape mismatch")
    if out is None:
        out = torch.empty((T, bank.d), dtype=out_dtype, device=h.device)
    ex = gt = None
    if return_routing:
        ex = torch.empty((max(T, 1) * top_k,), dtype=torch.int32, device=h.device)
        gt = torch.empty((max(T, 1) * top_k,), dtype=torch.float32, device=h.device)
    check(_lib.load().moqe_gpu_moe_forward(
        bank._h, _ptr(h), _lib.F16 if hd == torch.float16 else _lib.F32, T, _ptr(wg), top_k,
        _ptr(out), _lib.F16 if out.dtype == torch.float16 else _lib.F32, _ptr(ex), _ptr(gt),
        _PATH[path], _stream()))
    if return_routing:
        shape = (T,) if top_k == 1 else (T, top_k)
        return out, ex[: T * top_k].reshape(shape), gt[: T * top_k].reshape(shape)
    return out


def expert_ffn(x: torch.Tensor, bank: ExpertBank, expert: torch.Tensor, gate: torch.Tensor,
               out_dtype: torch.dtype = torch.float32, path: str = "auto",
               out: Optional[torch.Tensor] = None, validate: bool = True) -> torch.Tensor:
    """Expert FFN on pre-routed rows (expert-parallel owner side):
    out[r] = gate[r] * FFN_{expert[r]}(x[r]), expert ids local to `bank`. validate=False skips
    the host-side id range check (a device sync) when the ids come from a trusted router."""
    xd = x.dtype if x.dtype in (torch.float16, torch.float32) else torch.float32
    x = _dev(x, xd, "expert_ffn")
    if x.dim() != 2 or x.shape[1] != bank.d:
        raise _lib.InvalidArgument("matmul: shape mismatch")
    ex = _dev(expert, torch.int32, "expert_ffn").reshape(-1)
    gt = _dev(gate, torch.float32, "expert_ffn").reshape(-1)
    R = x.shape[0]
    if ex.numel() != R or gt.numel() != R:
        raise _lib.InvalidArgument("expert_ffn: one expert id and gate per row")
    if validate and R and (int(ex.min()) < 0 or int(ex.max()) >= bank.E):
        raise _lib.InvalidArgument("expert_ffn: expert id out of range")
    if out is None:
        out = torch.empty((R, bank.d), dtype=out_dtype, device=x.device)
    check(_lib.load().moqe_gpu_expert_ffn(
        bank._h, _ptr(x), _lib.F16 if xd == torch.float16 else _lib.F32, R, _ptr(ex), _ptr(gt), _ptr(out),
        _lib.F16 if out.dtype == torch.float16 else _lib.F32, _PATH[path], _stream()))
    return out


def moe_ffn_forward_host(h_host: torch.Tensor, bank: ExpertBank, top_k: int = 1,
                         out: Optional[torch.Tensor] = None, out_dtype=torch.float32) -> torch.Tensor:
    """By-value (host buffer) call, like the reference API: copies in, forward, copies out."""
    hd = h_host.dtype
    if out is None:
        out = torch.empty((h_host.shape[0], bank.d), dtype=out_dtype, pin_memory=True)
    check(_lib.load().moqe_gpu_moe_forward_host(
        bank._h, _ptr(h_host), _lib.F16 if hd == torch.float16 else _lib.F32, h_host.shape[0],
        top_k, _ptr(out), _lib.F16 if out.dtype == torch.float16 else _lib.F32, _stream()))
    return out


# ---- quantize_model (model.cpp:577-636), "quantize experts" recipe ---------------

EXPERT_FFN = "expert_ffn"


def quantize_model(ckpt: Dict[str, Tuple[torch.Tensor, str]], groups: Iterable[str], bits: int,
                   granularity: str = PER_CHANNEL, subset: str = "all") -> Dict[str, object]:
    """Replace every 2-D tensor whose group is in `groups` by its QuantizedTensor.

    ckpt maps name -> (tensor, group). Mirrors moqe::quantize_model: empty group
    list and bad widths are rejected; 1-D tensors are skipped with a warning;
    optional layer parity filter ("even"/"odd", layer index from the canonical
    name). Same-shape matrices are quantized in one batched launch."""
    groups = set(groups)
    if not groups:
        raise _lib.InvalidArgument("quantize_model: empty group list")
    if not valid_bits(bits):
        raise _lib.InvalidArgument("quantize_model: unsupported bit width")

    def layer_of(name: str):
        for part in name.split("."):
            if part.isdigit():
                return int(part)
        return None

    out: Dict[str, object] = dict(ckpt)
    todo: Dict[Tuple[int, int], list] = {}
    for name, (t, grp) in ckpt.items():
        if grp not in groups:
            continue
        if subset != "all":
            li = layer_of(name)
            if li is None or (subset == "even" and li % 2) or (subset == "odd" and li % 2 == 0):
                continue
        if isinstance(t, QuantizedTensor):
            print(f"warning: {name} already quantized, skipping", file=sys.stderr)
            continue
        if t.dim() != 2:
            print(f"warning: skipping non-2D tensor {name}", file=sys.stderr)
            continue
        todo.setdefault(tuple(t.shape), []).append(name)
    for shape, names in todo.items():
        batch = torch.stack([ckpt[n][0].to(torch.float32) for n in names]).cuda()
        qts = quantize_linear(batch, bits, granularity)
        for n, q in zip(names, qts):
            out[n] = q
    return out
