"""Pin the CPU oracle (oracle/moqe_oracle.c) before trusting it.

(a) the reference's own known-answer tests, restated with file:line;
(b) golden fixtures produced by the UNMODIFIED reference (tests/golden, made by
    tests/golden/make_golden.py from oracle/_ref);
(c) live comparison with oracle/_ref when it is built (dev container).
CPU only.
"""
import math

import numpy as np
import pytest

import oracle
from helpers import make_layer

REF = oracle.ref_available()


# ---- (a) known answers -------------------------------------------------------------

def test_binary16_reference_values(orc):
    # proj/tests/test_tensorio.cpp:38-62
    for v in (1.0, -2.0, 0.5, 0.0, 65504.0, -65504.0, 0.66650390625):
        assert orc.round_to_binary16(v) == np.float32(v)
    assert orc.round_to_binary16(0.1) == np.float32(0.0999755859375)
    assert orc.round_to_binary16(np.float32(2.0) / np.float32(3.0)) == np.float32(0.66650390625)
    assert math.isclose(orc.round_to_binary16(6e-8), 5.9604644775390625e-08, rel_tol=1e-6)
    assert orc.round_to_binary16(1e-9) == 0.0
    with pytest.raises(OverflowError):
        orc.round_to_binary16(65520.0)
    with pytest.raises(OverflowError):
        orc.round_to_binary16(1e30)
    assert orc.round_to_binary16(65519.0) == 65504.0


def test_binary16_all_patterns_round_trip(orc):
    # proj/tests/test_tensorio.cpp:73-79
    for h in range(0x10000):
        if (h & 0x7C00) == 0x7C00:
            continue
        assert orc.f32_to_f16_bits(orc.f16_bits_to_f32(h)) == h


def test_binary16_matches_ieee_rne(orc):
    # numpy's float16 cast is IEEE RNE; compare on a wide seeded sample
    rng = np.random.default_rng(5)
    xs = (rng.standard_normal(20000) * 10.0 ** rng.integers(-9, 6, 20000)).astype(np.float32)
    want = xs.astype(np.float16).view(np.uint16)
    got = np.array([orc.f32_to_f16_bits(x) for x in xs], np.uint16)
    assert (got == want).all()


def test_linear_scales_and_codes_reference_values(orc):
    # proj/tests/test_quant.cpp:85-104
    col = lambda v: np.array(v, np.float32).reshape(-1, 1)
    assert orc.linear_scales(col([0.5, -1.0, 0.25]), 2)[0] == np.float32(0.66650390625)
    assert orc.linear_scales(col([0.0, 0.0]), 4)[0] == 0.0
    assert orc.linear_scales(col([7.5]), 4)[0] == 1.0
    q, _ = orc.quantize_linear(col([0.5, -1.0, 0.25]), 2)
    assert q.ravel().tolist() == [1, -2, 0]
    q, _ = orc.quantize_linear(np.zeros((3, 2), np.float32), 4)
    assert (q == 0).all()
    q, _ = orc.quantize_linear(col([1.0, -1.0]), 4)
    assert q.ravel().tolist() == [7, -8]  # clamp + ties-to-even


def test_quantize_errors(orc):
    # quant.cpp:31-35: non-2D / bad bits / non-finite -> invalid_argument
    with pytest.raises(ValueError):
        orc.quantize_linear(np.array([[np.inf]], np.float32), 4)
    with pytest.raises(ValueError):
        orc.quantize_linear(np.ones((2, 2), np.float32), 5)
    # scale overflow -> range_error (tensor.cpp:103-104)
    with pytest.raises(OverflowError):
        orc.quantize_linear(np.array([[3e38]], np.float32), 2)


def test_pack_reference_values(orc):
    # proj/tests/test_bitpack.cpp:10-68
    assert [orc.packed_size(b, n) for b, n in ((2, 0), (8, 5), (4, 5), (2, 5), (3, 8), (3, 9), (3, 5))] == \
        [0, 5, 3, 2, 3, 6, 3]
    with pytest.raises(ValueError):
        orc.packed_size(5, 1)
    assert orc.pack(np.array([-128, 127]), 8).tolist() == [0x00, 0xFF]
    assert orc.pack(np.array([-2, -1, 0, 1]), 2).tolist() == [0xE4]
    assert orc.pack(np.array([3] * 8), 3).tolist() == [0xFF, 0xFF, 0xFF]
    assert orc.unpack(np.array([0x21], np.uint8), 4, 2).tolist() == [-7, -6]
    assert orc.unpack(np.zeros(3, np.uint8), 3, 5).tolist() == [-4] * 5
    with pytest.raises(IndexError):
        orc.pack(np.array([2]), 2)
    with pytest.raises(IndexError):
        orc.pack(np.array([-9]), 4)
    with pytest.raises(ValueError):
        orc.unpack(np.zeros(1, np.uint8), 4, 3)
    with pytest.raises(ValueError):
        orc.unpack(np.zeros(2, np.uint8), 3, 5)


def test_pack_round_trip_counts_0_to_64(orc):
    # proj/tests/test_bitpack.cpp:70-89, acceptance.cpp:164-192
    rng = np.random.default_rng(1234)
    for bits in (2, 3, 4, 8):
        for count in range(65):
            for _ in range(5):
                c = rng.integers(-(1 << (bits - 1)), 1 << (bits - 1), count).astype(np.int8)
                b = orc.pack(c, bits)
                assert b.size == orc.packed_size(bits, count)
                assert (orc.unpack(b, bits, count) == c).all()


def test_route_reference_values(orc):
    # proj/tests/test_model.cpp:35-61
    h = np.array([[1, 2], [-1, 0], [4, 4]], np.float32)
    ex, g = orc.route(h, np.array([[0.5], [-0.25]], np.float32))
    assert (ex == 0).all() and (g == 1.0).all()
    ex, g = orc.route(np.array([[1, 2, 3], [-1, -2, -3]], np.float32), np.zeros((3, 4), np.float32))
    assert (ex == 0).all() and np.allclose(g, 0.25, rtol=1e-6)
    ex, g = orc.route(np.array([[1.0]], np.float32), np.array([[2.0, 0.0]], np.float32))
    assert ex[0] == 0 and math.isclose(g[0], math.exp(2) / (math.exp(2) + 1), rel_tol=1e-6)


def test_route_brute_force(orc):
    # proj/tests/test_model.cpp:63-85 (32 x 8 x 5)
    rng = np.random.default_rng(31)
    h = rng.standard_normal((32, 8)).astype(np.float32)
    w = rng.standard_normal((8, 5)).astype(np.float32)
    ex, g = orc.route(h, w)
    lg = h.astype(np.float64) @ w.astype(np.float64)
    assert (ex == lg.argmax(1)).all()
    z = np.exp(lg - lg.max(1, keepdims=True)).sum(1)
    assert np.allclose(g, 1.0 / z, rtol=1e-5)


def test_top2_restatement(orc):
    # BASELINE config 4 semantics (a7): second argmax over the rest, renormalised
    rng = np.random.default_rng(9)
    h = rng.standard_normal((50, 16)).astype(np.float32)
    w = rng.standard_normal((16, 7)).astype(np.float32)
    ex, g = orc.route(h, w, top_k=2)
    lg = orc.router_logits(h, w)
    for i in range(50):
        e1 = int(np.argmax(lg[i]))
        rest = lg[i].copy()
        rest[e1] = -np.inf
        e2 = int(np.argmax(rest))
        assert (ex[i, 0], ex[i, 1]) == (e1, e2)
        z = math.exp(float(lg[i, e2]) - float(lg[i, e1]))
        assert math.isclose(g[i, 0], 1 / (1 + z), rel_tol=1e-6)
        assert math.isclose(g[i, 0] + g[i, 1], 1.0, rel_tol=1e-6)


def test_moe_zero_input_gives_gated_bias(orc):
    # proj/tests/test_model.cpp:118-134: zero h, zero weights, b2 -> b2 / 3
    E, d, f = 3, 4, 8
    q1 = np.zeros((E, d, f), np.int8)
    q2 = np.zeros((E, f, d), np.int8)
    s1 = np.zeros((E, f), np.float32)
    s2 = np.zeros((E, d), np.float32)
    b1 = np.zeros((E, f), np.float32)
    b2 = np.tile((np.arange(d) - 1.5).astype(np.float32), (E, 1))
    out, ex, g = orc.moe_forward(np.zeros((2, d), np.float32), np.zeros((d, E), np.float32),
                                 q1, s1, q2, s2, b1=b1, b2=b2)
    assert (ex == 0).all()
    assert np.allclose(out, b2[0] / 3.0, rtol=1e-6)


def test_token_sharding_is_bit_identical(orc):
    # proj/tests/acceptance.cpp:267-276 (thread-count invariance)
    L = make_layer(orc, 3, 4, 64, 128, 4, 37)
    a = orc.moe_forward(L["h"], L["wg"], L["q1"], L["s1"], L["q2"], L["s2"], n_threads=1)[0]
    b = orc.moe_forward(L["h"], L["wg"], L["q1"], L["s1"], L["q2"], L["s2"], n_threads=5)[0]
    assert np.array_equal(a, b)


# ---- (b) golden fixtures from the reference ----------------------------------------

@pytest.mark.parametrize("bits", [2, 3, 4, 8])
@pytest.mark.parametrize("gran", ["channel", "tensor"])
def test_golden_quant(orc, golden, bits, gran):
    G = golden["quant"]
    w = G[f"w_{bits}_{gran}"]
    q, s = orc.quantize_linear(w, bits, gran == "tensor")
    assert np.array_equal(q, G[f"codes_{bits}_{gran}"])
    assert np.array_equal(s, G[f"scales_{bits}_{gran}"])
    assert np.array_equal(orc.pack(q, bits), G[f"packed_{bits}_{gran}"])
    for count in (0, 1, 5, 9, 26, 63):
        c = G[f"ragged_codes_{bits}_{count}"]
        assert np.array_equal(orc.pack(c, bits), G[f"ragged_packed_{bits}_{count}"])


def test_golden_route(orc, golden):
    G = golden["route"]
    for i in range(3):
        ex, g = orc.route(G[f"h_{i}"], G[f"wg_{i}"])
        assert np.array_equal(ex, G[f"expert_{i}"])
        assert np.array_equal(g, G[f"gate_{i}"])


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
def test_golden_moe_bit_exact(orc, golden, bits):
    G = golden["moe"]
    b1 = G[f"b1_{bits}"] if f"b1_{bits}" in G else None
    b2 = G[f"b2_{bits}"] if f"b2_{bits}" in G else None
    out, ex, g = orc.moe_forward(G[f"h_{bits}"], G[f"wg_{bits}"], G[f"q1_{bits}"], G[f"s1_{bits}"],
                                 G[f"q2_{bits}"], G[f"s2_{bits}"], b1=b1, b2=b2)
    assert np.array_equal(ex, G[f"expert_{bits}"])
    assert np.array_equal(out, G[f"out_{bits}"])  # bit-identical to moqe::moe_ffn_forward


# ---- (c) live reference (dev container) ----------------------------------------------

@pytest.mark.skipif(not REF, reason="oracle/_ref not built")
@pytest.mark.parametrize("bits", [2, 3, 4, 8])
def test_live_reference_moe(orc, bits):
    ref = oracle.ref()
    L = make_layer(orc, 100 + bits, 6, 96, 160, bits, 29, with_bias=bits == 3)
    bank = ref.bank(L["q1"], L["s1"], L["q2"], L["s2"], bits, L["b1"], L["b2"])
    want = bank.forward(L["h"], L["wg"], 3)
    got = orc.moe_forward(L["h"], L["wg"], L["q1"], L["s1"], L["q2"], L["s2"], b1=L["b1"], b2=L["b2"])[0]
    assert np.array_equal(got, want)


@pytest.mark.skipif(not REF, reason="oracle/_ref not built")
def test_live_reference_quant_large(orc):
    ref = oracle.ref()
    rng = np.random.default_rng(77)
    w = (rng.standard_normal((512, 384)) * 0.02).astype(np.float32)
    for bits in (2, 3, 4, 8):
        q0, s0 = ref.quantize_linear(w, bits)
        q1, s1 = orc.quantize_linear(w, bits)
        assert np.array_equal(q0, q1) and np.array_equal(s0, s1)
        assert np.array_equal(ref.pack(q0, bits), orc.pack(q1, bits))
