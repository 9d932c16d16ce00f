"""MQE1 container -> device bank (SURVEY.md §8 f2; checkpoint.cpp:99-131, :312-413).

Containers are written by the compiled, unmodified reference (moqe::write_checkpoint_file
through oracle/_ref). CPU tests: the index parse and the reference's error cases; GPU tests:
the bank built from the container runs the forward the oracle computes from the same codes."""
import os

import numpy as np
import pytest

from helpers import allclose_report, check_routing, fp16_valued, make_layer


def _ref_or_skip():
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    return oracle.ref()


def _write(tmp_path, orc, bits=4, per_tensor=False, bias=True, E=4, d=64, f=128, T=5):
    L = make_layer(orc, 11 + bits, E, d, f, bits, T, with_bias=bias)
    if per_tensor:
        for k, (w, q, s) in enumerate((("w1", "q1", "s1"), ("w2", "q2", "s2"))):
            qs, ss = zip(*[orc.quantize_linear(L[w][e], bits, per_tensor=True) for e in range(E)])
            L[q], L[s] = np.stack(qs), np.stack(ss)
    path = tmp_path / "layer.mqe1"
    _ref_or_skip().write_moe_mqe1(path, "enc.0", L["q1"], L["s1"], L["q2"], L["s2"], bits, per_tensor,
                                  L["b1"], L["b2"], L["wg"])
    return path, L


def test_mqe1_index(tmp_path, orc):
    import paper_2310_02410_b200 as m
    path, L = _write(tmp_path, orc)
    with m.Mqe1(path) as c:
        ents = {e["name"]: e for e in c.entries()}
    e = ents["enc.0.expert.2.fc1.w"]
    assert e["dtype"] == "q-lin" and e["bits"] == 4 and e["shape"] == (64, 128)
    assert e["data_bytes"] == orc.packed_size(4, 64 * 128) and e["scale_bytes"] == 2 * 128
    assert e["data_offset"] % 64 == 0 and e["scale_offset"] % 64 == 0  # 64-B aligned blobs
    raw = open(path, "rb").read()
    blob = np.frombuffer(raw[e["data_offset"]: e["data_offset"] + e["data_bytes"]], np.uint8)
    assert np.array_equal(blob, orc.pack(L["q1"][2], 4))  # the GPU bank's input layout, as stored
    assert ents["enc.0.router.w"]["dtype"] == "f32" and ents["enc.0.router.w"]["shape"] == (64, 4)


@pytest.mark.parametrize("damage,msg", [("magic", "bad magic"), ("version", "version"),
                                        ("truncate", "truncated"), ("index", "inconsistency")])
def test_mqe1_errors(tmp_path, orc, damage, msg):
    # read_checkpoint's error cases (checkpoint.cpp:315-377)
    import paper_2310_02410_b200 as m
    path, _ = _write(tmp_path, orc)
    raw = bytearray(open(path, "rb").read())
    if damage == "magic":
        raw[:4] = b"MQE2"
    elif damage == "version":
        raw[4] = 7
    elif damage == "truncate":
        raw = raw[: len(raw) - 200]
    else:  # a data length that disagrees with the shape
        i = raw.index(b"enc.0.expert.0.fc1.w")
        line_end = raw.index(b"\n", i)
        fields = raw[i:line_end].split(b" ")
        fields[-3] = b"%016x" % (int(fields[-3], 16) + 1)
        raw[i:line_end] = b" ".join(fields)
    bad = tmp_path / "bad.mqe1"
    bad.write_bytes(bytes(raw))
    with pytest.raises(m.CheckpointError, match=msg):
        m.Mqe1(bad)


@pytest.mark.gpu
@pytest.mark.parametrize("bits,per_tensor,T", [(4, False, 5), (3, False, 40), (2, True, 300)])
def test_mqe1_bank_forward(tmp_path, gpu, orc, bits, per_tensor, T):
    import torch
    path, L = _write(tmp_path, orc, bits=bits, per_tensor=per_tensor, T=T)
    bank = gpu.ExpertBank.from_mqe1(str(path), "enc.0", 4)
    s1 = np.broadcast_to(L["s1"], (4, 128)) if per_tensor else L["s1"]
    s2 = np.broadcast_to(L["s2"], (4, 64)) if per_tensor else L["s2"]
    want, _, _ = orc.moe_forward(L["h"], L["wg"], L["q1"], s1, L["q2"], s2, b1=L["b1"], b2=L["b2"])
    out, ex, g = gpu.moe_ffn_forward(torch.from_numpy(L["h"]).cuda().half(), bank, return_routing=True)
    check_routing(orc, L["h"], L["wg"], 1, ex.cpu().numpy(), g.cpu().numpy())
    nbad, mx = allclose_report(out.cpu().numpy(), want)
    assert nbad == 0, mx
