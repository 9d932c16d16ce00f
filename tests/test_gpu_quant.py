"""GPU quantize-experts parity: scales, codes and packed bytes bit-exact with
the oracle / reference goldens (quant.cpp:59-95, bitpack.cpp:18-68)."""
import numpy as np
import pytest

from helpers import fp16_valued

pytestmark = pytest.mark.gpu


def _t(a, dev="cuda"):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
@pytest.mark.parametrize("gran", ["channel", "tensor"])
def test_golden_quant(gpu, golden, bits, gran):
    G = golden["quant"]
    w = G[f"w_{bits}_{gran}"]
    q = gpu.quantize_linear(_t(w), bits, gran)
    assert np.array_equal(q.codes.cpu().numpy(), G[f"codes_{bits}_{gran}"])
    assert np.array_equal(q.scales.cpu().numpy(), G[f"scales_{bits}_{gran}"])
    assert np.array_equal(q.packed.cpu().numpy(), G[f"packed_{bits}_{gran}"])
    assert np.array_equal(gpu.pack(q.codes, bits).cpu().numpy(), G[f"packed_{bits}_{gran}"])


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
def test_ragged_pack_unpack(gpu, golden, bits):
    G = golden["quant"]
    for count in (0, 1, 5, 9, 26, 63):
        c = G[f"ragged_codes_{bits}_{count}"]
        p = gpu.pack(_t(c), bits).cpu().numpy()
        assert np.array_equal(p, G[f"ragged_packed_{bits}_{count}"])
        back = gpu.unpack(_t(p if p.size else np.zeros(0, np.uint8)), bits, count).cpu().numpy()
        assert np.array_equal(back, c)


@pytest.mark.parametrize("bits", [2, 3, 4, 8])
@pytest.mark.parametrize("shape", [(1024, 4096), (4096, 1024), (37, 53), (1, 8)])
def test_expert_shapes_vs_oracle(gpu, orc, bits, shape):
    rng = np.random.default_rng(hash((bits,) + shape) % 2**32)
    w = (rng.standard_normal(shape) * 0.02).astype(np.float32)
    q, s = orc.quantize_linear(w, bits)
    p = orc.pack(q, bits)
    gq = gpu.quantize_linear(_t(w), bits)
    assert np.array_equal(gq.scales.cpu().numpy(), s)
    assert np.array_equal(gq.codes.cpu().numpy(), q)
    assert np.array_equal(gq.packed.cpu().numpy(), p)


def test_batched_quantize_pack_matches_per_matrix(gpu, orc):
    import torch
    rng = np.random.default_rng(4)
    w = (rng.standard_normal((6, 128, 96)) * 0.02).astype(np.float32)
    packed, scales = gpu.quantize_pack(_t(w), 3)
    for i in range(6):
        q, s = orc.quantize_linear(w[i], 3)
        assert np.array_equal(scales[i].cpu().numpy(), s)
        assert np.array_equal(packed[i].cpu().numpy(), orc.pack(q, 3))


def test_quant_edge_values(gpu, orc):
    # ties, clamps, zero column, subnormal-range scales
    w = np.array([[1.0, -1.0, 0.0, 1e-6], [-1.0, 0.5, 0.0, -3e-7], [0.25, 1.0, 0.0, 2e-7]], np.float32)
    for bits in (2, 3, 4, 8):
        q, s = orc.quantize_linear(w, bits)
        g = gpu.quantize_linear(_t(w), bits)
        assert np.array_equal(g.codes.cpu().numpy(), q)
        assert np.array_equal(g.scales.cpu().numpy(), s)


def test_quant_errors(gpu):
    import torch
    with pytest.raises(gpu.InvalidArgument):
        gpu.quantize_linear(_t(np.array([[np.nan, 1.0]], np.float32)), 4)
    with pytest.raises(gpu.InvalidArgument):
        gpu.quantize_linear(_t(np.ones((2, 2), np.float32)), 5)
    with pytest.raises(gpu.RangeError):
        gpu.quantize_linear(_t(np.array([[3e38]], np.float32)), 2)
    with pytest.raises(gpu.OutOfRange):
        gpu.pack(_t(np.array([2], np.int8)), 2)
    with pytest.raises(gpu.OutOfRange):
        gpu.pack(_t(np.array([-9], np.int8)), 4)
    with pytest.raises(gpu.InvalidArgument):
        gpu.unpack(_t(np.zeros(1, np.uint8)), 4, 3)
    with pytest.raises(gpu.InvalidArgument):
        gpu.packed_size(5, 1)


def test_quantize_model_expert_recipe(gpu, orc):
    import torch
    rng = np.random.default_rng(8)
    ckpt = {
        "enc.0.expert.0.fc1.w": (torch.from_numpy((rng.standard_normal((64, 128)) * 0.08).astype(np.float32)), "expert_ffn"),
        "enc.0.expert.0.fc1.b": (torch.zeros(128), "expert_ffn"),
        "enc.0.expert.1.fc1.w": (torch.from_numpy((rng.standard_normal((64, 128)) * 0.08).astype(np.float32)), "expert_ffn"),
        "enc.1.ffn.fc1.w": (torch.from_numpy((rng.standard_normal((64, 128)) * 0.08).astype(np.float32)), "dense_ffn"),
    }
    with pytest.raises(gpu.InvalidArgument):
        gpu.quantize_model(ckpt, [], 4)
    out = gpu.quantize_model(ckpt, ["expert_ffn"], 4)
    for name, (t, grp) in ckpt.items():
        if grp == "expert_ffn" and t.dim() == 2:
            q, s = orc.quantize_linear(t.numpy(), 4)
            assert np.array_equal(out[name].codes.cpu().numpy(), q)
            assert np.array_equal(out[name].scales.cpu().numpy(), s)
        else:
            assert out[name] is ckpt[name]
