"""oracle — TEST INFRASTRUCTURE ONLY.

numpy/ctypes bindings for the two CPU checkers of the MoQE expert-FFN path:

* ``orc``  — the plain-C restatement (oracle/moqe_oracle.c -> build/libmoqe_oracle.so)
* ``ref``  — the unmodified reference library compiled from /root/reference
             (oracle/_ref/libmoqe_ref.so; built in the dev container, shipped
             to the GPU box as a prebuilt file).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import this package, and only as the checker or the timed
CPU baseline. The product (paper_2310_02410_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_SO = os.path.join(HERE, "build", "libmoqe_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmoqe_ref.so")
REF_SRC = "/root/reference/proj/src"

STATUS = {0: None, 1: ValueError, 2: IndexError, 3: OverflowError}


def build(ref: bool = True) -> None:
    """Compile the restatement (always) and the reference (when its sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


def _check(st: int, what: str) -> None:
    exc = STATUS.get(st, RuntimeError)
    if exc is not None:
        raise exc(f"{what}: status {st}")


class _Lib:
    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run oracle.build())")
        self.lib = C.CDLL(path)
        self.pre = prefix
        L, P = self.lib, prefix
        i64, i32 = C.c_int64, C.c_int
        fp, i8p, u8p = C.POINTER(C.c_float), C.POINTER(C.c_int8), C.POINTER(C.c_uint8)
        self._sig(P + "f32_to_f16_bits", C.c_uint16, [C.c_float])
        self._sig(P + "f16_bits_to_f32", C.c_float, [C.c_uint16])
        self._sig(P + "round_to_binary16", i32, [C.c_float, fp])
        self._sig(P + "linear_scales", i32, [fp, i64, i64, i32, i32, fp])
        self._sig(P + "quantize_linear", i32, [fp, i64, i64, i32, i32, i8p, fp])
        self._sig(P + "packed_size", i64, [i32, i64])
        self._sig(P + "pack", i32, [i8p, i64, i32, u8p])
        self._sig(P + "unpack", i32, [u8p, i64, i32, i64, i8p])
        del L

    def _sig(self, name, res, args):
        fn = getattr(self.lib, name)
        fn.restype = res
        fn.argtypes = args

    def fn(self, name):
        return getattr(self.lib, self.pre + name)

    # binary16 -----------------------------------------------------------
    def f32_to_f16_bits(self, x: float) -> int:
        return int(self.fn("f32_to_f16_bits")(float(x)))

    def f16_bits_to_f32(self, h: int) -> float:
        return float(self.fn("f16_bits_to_f32")(int(h)))

    def round_to_binary16(self, x: float) -> float:
        out = C.c_float()
        _check(self.fn("round_to_binary16")(float(x), C.byref(out)), "round_to_binary16")
        return out.value

    # quantizer -----------------------------------------------------------
    def linear_scales(self, a: np.ndarray, bits: int, per_tensor: bool = False) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.float32)
        s = np.zeros(1 if per_tensor else a.shape[1], np.float32)
        _check(self.fn("linear_scales")(_p(a, C.c_float), a.shape[0], a.shape[1], bits,
                                         int(per_tensor), _p(s, C.c_float)), "linear_scales")
        return s

    def quantize_linear(self, a: np.ndarray, bits: int, per_tensor: bool = False):
        a = np.ascontiguousarray(a, dtype=np.float32)
        q = np.zeros(a.shape, np.int8)
        s = np.zeros(1 if per_tensor else a.shape[1], np.float32)
        _check(self.fn("quantize_linear")(_p(a, C.c_float), a.shape[0], a.shape[1], bits,
                                           int(per_tensor), _p(q, C.c_int8), _p(s, C.c_float)),
               "quantize_linear")
        return q, s

    # packing -------------------------------------------------------------
    def packed_size(self, bits: int, count: int) -> int:
        n = int(self.fn("packed_size")(bits, count))
        if n < 0:
            raise ValueError("packed_size: unsupported width")
        return n

    def pack(self, codes: np.ndarray, bits: int) -> np.ndarray:
        c = np.ascontiguousarray(codes, dtype=np.int8).ravel()
        n = self.packed_size(bits, c.size)
        out = np.zeros(max(n, 1), np.uint8)
        _check(self.fn("pack")(_p(c, C.c_int8), c.size, bits, _p(out, C.c_uint8)), "pack")
        return out[:n]

    def unpack(self, data: np.ndarray, bits: int, count: int) -> np.ndarray:
        d = np.ascontiguousarray(data, dtype=np.uint8)
        out = np.zeros(max(count, 1), np.int8)
        dd = d if d.size else np.zeros(1, np.uint8)
        _check(self.fn("unpack")(_p(dd, C.c_uint8), d.size, bits, count, _p(out, C.c_int8)),
               "unpack")
        return out[:count]


class Oracle(_Lib):
    """The plain-C restatement."""

    def __init__(self, path: str = ORC_SO):
        super().__init__(path, "orc_")
        i64, i32 = C.c_int64, C.c_int
        fp, i8p, ip = C.POINTER(C.c_float), C.POINTER(C.c_int8), C.POINTER(C.c_int32)
        self._sig("orc_router_logits", None, [fp, i64, i64, fp, i64, fp])
        self._sig("orc_route", i32, [fp, i64, i64, fp, i64, i32, ip, fp])
        self._sig("orc_expert_ffn", None, [fp, i64, i64, i64, i8p, fp, i8p, fp, fp, fp, fp])
        self._sig("orc_moe_forward", i32, [fp, i64, i64, i64, i32, fp, i32, i8p, fp, i8p, fp,
                                           fp, fp, fp, ip, fp, i32])
        self._sig("orc_layer_norm", None, [fp, i64, i64, fp, fp, fp])
        self._sig("orc_matmul", None, [fp, i64, i64, fp, i64, fp])
        self._sig("orc_dense_ffn", None, [fp, i64, i64, i64, fp, fp, fp, fp, fp])

    def router_logits(self, h, wg):
        h = np.ascontiguousarray(h, np.float32)
        wg = np.ascontiguousarray(wg, np.float32)
        out = np.zeros((h.shape[0], wg.shape[1]), np.float32)
        self.lib.orc_router_logits(_p(h, C.c_float), h.shape[0], h.shape[1], _p(wg, C.c_float),
                                   wg.shape[1], _p(out, C.c_float))
        return out

    def route(self, h, wg, top_k=1):
        h = np.ascontiguousarray(h, np.float32)
        wg = np.ascontiguousarray(wg, np.float32)
        t = h.shape[0]
        ex = np.zeros(max(t * top_k, 1), np.int32)
        g = np.zeros(max(t * top_k, 1), np.float32)
        _check(self.lib.orc_route(_p(h, C.c_float), t, h.shape[1], _p(wg, C.c_float),
                                  wg.shape[1], top_k, _p(ex, C.c_int32), _p(g, C.c_float)),
               "route")
        shp = (t,) if top_k == 1 else (t, top_k)
        return ex[: t * top_k].reshape(shp), g[: t * top_k].reshape(shp)

    def moe_forward(self, h, wg, codes1, scales1, codes2, scales2, top_k=1, b1=None, b2=None,
                    n_threads=None):
        h = np.ascontiguousarray(h, np.float32)
        wg = np.ascontiguousarray(wg, np.float32)
        E, d, f = codes1.shape
        t = h.shape[0]
        c1 = np.ascontiguousarray(codes1, np.int8)
        c2 = np.ascontiguousarray(codes2, np.int8)
        s1 = np.ascontiguousarray(scales1, np.float32)
        s2 = np.ascontiguousarray(scales2, np.float32)
        b1 = None if b1 is None else np.ascontiguousarray(b1, np.float32)
        b2 = None if b2 is None else np.ascontiguousarray(b2, np.float32)
        out = np.zeros((max(t, 1), d), np.float32)
        ex = np.zeros(max(t * top_k, 1), np.int32)
        g = np.zeros(max(t * top_k, 1), np.float32)
        nt = n_threads or os.cpu_count() or 1
        _check(self.lib.orc_moe_forward(_p(h, C.c_float), t, d, f, E, _p(wg, C.c_float), top_k,
                                        _p(c1, C.c_int8), _p(s1, C.c_float), _p(c2, C.c_int8),
                                        _p(s2, C.c_float), _p(b1, C.c_float), _p(b2, C.c_float),
                                        _p(out, C.c_float), _p(ex, C.c_int32), _p(g, C.c_float),
                                        nt), "moe_forward")
        shp = (t,) if top_k == 1 else (t, top_k)
        return out[:t], ex[: t * top_k].reshape(shp), g[: t * top_k].reshape(shp)

    def expert_ffn(self, x, q1, s1, q2, s2, b1=None, b2=None):
        """relu(x W1' + b1) W2' + b2 for rows x [m x d] (model.cpp:381-385)."""
        x = np.ascontiguousarray(x, np.float32)
        m, d = x.shape
        f = q1.shape[1]
        y = np.zeros((max(m, 1), d), np.float32)
        arr = lambda a, t: None if a is None else np.ascontiguousarray(a, t)
        self.lib.orc_expert_ffn(_p(x, C.c_float), m, d, f, _p(arr(q1, np.int8), C.c_int8),
                                _p(arr(s1, np.float32), C.c_float), _p(arr(q2, np.int8), C.c_int8),
                                _p(arr(s2, np.float32), C.c_float), _p(arr(b1, np.float32), C.c_float),
                                _p(arr(b2, np.float32), C.c_float), _p(y, C.c_float))
        return y[:m]

    def matmul(self, a, b):
        """Reference matmul (model.cpp:152-167)."""
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        out = np.zeros((a.shape[0], b.shape[1]), np.float32)
        self.lib.orc_matmul(_p(a, C.c_float), a.shape[0], a.shape[1], _p(b, C.c_float), b.shape[1],
                            _p(out, C.c_float))
        return out

    def dense_ffn(self, x, w1, w2, b1=None, b2=None):
        """relu(x W1 + b1) W2 + b2 (model.cpp:315-322)."""
        x = np.ascontiguousarray(x, np.float32)
        m, d = x.shape
        f = w1.shape[1]
        y = np.zeros((max(m, 1), d), np.float32)
        arr = lambda a: None if a is None else np.ascontiguousarray(a, np.float32)
        self.lib.orc_dense_ffn(_p(x, C.c_float), m, d, f, _p(arr(w1), C.c_float), _p(arr(b1), C.c_float),
                               _p(arr(w2), C.c_float), _p(arr(b2), C.c_float), _p(y, C.c_float))
        return y[:m]

    def layer_norm(self, x, gain, bias):
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros_like(x)
        self.lib.orc_layer_norm(_p(x, C.c_float), x.shape[0], x.shape[1],
                                _p(np.ascontiguousarray(gain, np.float32), C.c_float),
                                _p(np.ascontiguousarray(bias, np.float32), C.c_float),
                                _p(out, C.c_float))
        return out


class Ref(_Lib):
    """The compiled, unmodified reference library (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        super().__init__(path, "ref_")
        i64, i32 = C.c_int64, C.c_int
        fp, i8p, ip, vp = (C.POINTER(C.c_float), C.POINTER(C.c_int8), C.POINTER(C.c_int32),
                           C.c_void_p)
        self._sig("ref_top1_route", i32, [fp, i64, i64, fp, i64, ip, fp])
        self._sig("ref_dequantize", i32, [i8p, fp, i64, i64, i32, i32, fp])
        self._sig("ref_matmul_dequant_fused", i32, [i8p, fp, i64, i64, i32, i32, fp, i64, fp])
        self._sig("ref_bank_create", vp, [i32, i64, i64, i32, i8p, fp, i8p, fp, fp, fp])
        self._sig("ref_bank_create_float", vp, [i32, i64, i64, fp, fp, fp, fp])
        self._sig("ref_bank_destroy", None, [vp])
        self._sig("ref_bank_forward", i32, [vp, fp, i64, fp, fp, i32])
        self._sig("ref_hardware_threads", i32, [])
        self._sig("ref_quantize_log", i32, [fp, i64, i64, i32, i32, i32, i8p, fp])
        self._sig("ref_dequantize_log", i32, [i8p, fp, i64, i64, i32, i32, fp])
        self._sig("ref_bank_create_log", vp, [i32, i64, i64, i32, i8p, fp, i8p, fp])
        self._sig("ref_write_moe_mqe1", i64, [C.c_char_p, C.c_char_p, i32, i64, i64, i32, i32, i8p, fp, i8p, fp,
                                              fp, fp, fp])

    def linear_scales(self, a, bits, per_tensor=False):  # ref uses 0=channel,1=tensor too
        return super().linear_scales(a, bits, per_tensor)

    def top1_route(self, h, wg):
        h = np.ascontiguousarray(h, np.float32)
        wg = np.ascontiguousarray(wg, np.float32)
        t = h.shape[0]
        ex = np.zeros(max(t, 1), np.int32)
        g = np.zeros(max(t, 1), np.float32)
        _check(self.lib.ref_top1_route(_p(h, C.c_float), t, h.shape[1], _p(wg, C.c_float),
                                       wg.shape[1], _p(ex, C.c_int32), _p(g, C.c_float)),
               "top1_route")
        return ex[:t], g[:t]

    def dequantize(self, codes, scales, bits, per_tensor=False):
        c = np.ascontiguousarray(codes, np.int8)
        s = np.ascontiguousarray(scales, np.float32)
        out = np.zeros(c.shape, np.float32)
        _check(self.lib.ref_dequantize(_p(c, C.c_int8), _p(s, C.c_float), c.shape[0], c.shape[1],
                                       bits, int(per_tensor), _p(out, C.c_float)), "dequantize")
        return out

    def matmul_dequant_fused(self, codes, scales, bits, x, per_tensor=False):
        c = np.ascontiguousarray(codes, np.int8)
        s = np.ascontiguousarray(scales, np.float32)
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros((x.shape[0], c.shape[1]), np.float32)
        _check(self.lib.ref_matmul_dequant_fused(_p(c, C.c_int8), _p(s, C.c_float), c.shape[0],
                                                 c.shape[1], bits, int(per_tensor),
                                                 _p(x, C.c_float), x.shape[0],
                                                 _p(out, C.c_float)), "matmul_dequant_fused")
        return out

    def quantize_log(self, a, bits, per_tensor=False, mse_optimal=True):
        """moqe::quantize_log (quant.cpp:179-224): (codes [K,N] int8, scales f32)."""
        a = np.ascontiguousarray(a, np.float32)
        codes = np.zeros(a.shape, np.int8)
        scales = np.zeros(1 if per_tensor else a.shape[1], np.float32)
        _check(self.lib.ref_quantize_log(_p(a, C.c_float), a.shape[0], a.shape[1], bits, int(per_tensor),
                                         int(mse_optimal), _p(codes, C.c_int8), _p(scales, C.c_float)),
               "quantize_log")
        return codes, scales

    def dequantize_log(self, codes, scales, bits, per_tensor=False):
        c = np.ascontiguousarray(codes, np.int8)
        s = np.ascontiguousarray(scales, np.float32)
        out = np.zeros(c.shape, np.float32)
        _check(self.lib.ref_dequantize_log(_p(c, C.c_int8), _p(s, C.c_float), c.shape[0], c.shape[1], bits,
                                           int(per_tensor), _p(out, C.c_float)), "dequantize")
        return out

    def log_bank(self, codes1, scales1, codes2, scales2, bits):
        return RefBank(self, codes1, scales1, codes2, scales2, bits, None, None, log=True)

    def bank(self, codes1, scales1, codes2, scales2, bits, b1=None, b2=None):
        return RefBank(self, codes1, scales1, codes2, scales2, bits, b1, b2)

    def float_bank(self, w1, w2, b1=None, b2=None):
        return RefBank(self, w1, None, w2, None, 0, b1, b2, float_bank=True)

    def write_moe_mqe1(self, path, layer, codes1, scales1, codes2, scales2, bits, per_tensor=False,
                       b1=None, b2=None, wg=None) -> int:
        """One MoE layer as an MQE1 container written by moqe::write_checkpoint_file."""
        E, d, f = codes1.shape
        arr = lambda a, dt: None if a is None else np.ascontiguousarray(a, dt)
        c1, c2 = arr(codes1, np.int8), arr(codes2, np.int8)
        s1, s2 = arr(scales1, np.float32), arr(scales2, np.float32)
        bb1, bb2, w = arr(b1, np.float32), arr(b2, np.float32), arr(wg, np.float32)
        n = self.lib.ref_write_moe_mqe1(str(path).encode(), layer.encode(), E, d, f, bits, int(per_tensor),
                                        _p(c1, C.c_int8), _p(s1, C.c_float), _p(c2, C.c_int8), _p(s2, C.c_float),
                                        _p(bb1, C.c_float), _p(bb2, C.c_float), _p(w, C.c_float))
        if n < 0:
            raise RuntimeError("write_checkpoint failed")
        return int(n)

    def hardware_threads(self) -> int:
        return int(self.lib.ref_hardware_threads())


class RefBank:
    """Host-resident reference ExpertBank; forward = moqe::moe_ffn_forward."""

    def __init__(self, ref: Ref, w1, s1, w2, s2, bits, b1, b2, float_bank=False, log=False):
        self.ref = ref
        E, d, f = w1.shape
        self.E, self.d, self.f = E, d, f
        keep = []

        def arr(a, dt):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dt)
            keep.append(a)
            return a

        if log:
            self.h = ref.lib.ref_bank_create_log(
                E, d, f, bits, _p(arr(w1, np.int8), C.c_int8), _p(arr(s1, np.float32), C.c_float),
                _p(arr(w2, np.int8), C.c_int8), _p(arr(s2, np.float32), C.c_float))
        elif float_bank:
            self.h = ref.lib.ref_bank_create_float(
                E, d, f, _p(arr(w1, np.float32), C.c_float), _p(arr(w2, np.float32), C.c_float),
                _p(arr(b1, np.float32), C.c_float), _p(arr(b2, np.float32), C.c_float))
        else:
            self.h = ref.lib.ref_bank_create(
                E, d, f, bits, _p(arr(w1, np.int8), C.c_int8), _p(arr(s1, np.float32), C.c_float),
                _p(arr(w2, np.int8), C.c_int8), _p(arr(s2, np.float32), C.c_float),
                _p(arr(b1, np.float32), C.c_float), _p(arr(b2, np.float32), C.c_float))

    def forward(self, h, wg, n_threads=1):
        h = np.ascontiguousarray(h, np.float32)
        wg = np.ascontiguousarray(wg, np.float32)
        t = h.shape[0]
        out = np.zeros((max(t, 1), self.d), np.float32)
        _check(self.ref.lib.ref_bank_forward(self.h, _p(h, C.c_float), t, _p(wg, C.c_float),
                                             _p(out, C.c_float), n_threads), "moe_ffn_forward")
        return out[:t]

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.lib.ref_bank_destroy(self.h)
            self.h = None


_orc = None
_ref = None


def orc() -> Oracle:
    global _orc
    if _orc is None:
        _orc = Oracle()
    return _orc


def ref() -> Ref:
    global _ref
    if _ref is None:
        _ref = Ref()
    return _ref


def ref_available() -> bool:
    return os.path.exists(REF_SO)
