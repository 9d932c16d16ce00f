"""Drop-in shim (integration/moqe_gpu_shim.cpp): the reference's own binaries, linked
unchanged against the UNMODIFIED reference library with the shim ahead of it.

* proj/tests/acceptance.cpp: all 7 criteria PASS with moe_ffn_forward interposed.
* integration/shim_model_forward.cpp: the reference's model_forward over int4/3/2 experts
  runs its MoE layers on the GPU (ffn_block builds a stack-local bank per call; the shim's
  content-keyed cache must still pick up each layer's own weights) and matches the CPU run
  within |gpu - cpu| <= 2e-3 + 1e-2 |cpu|, bit-identical on repeat.

Binaries are built by integration/Makefile (__graft_entry__.build() when /root/reference is
present) and travel to the GPU box prebuilt."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B = os.path.join(ROOT, "integration", "_build")


def _run(name):
    exe = os.path.join(B, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (integration/Makefile needs /root/reference)")
    return subprocess.run([exe], capture_output=True, text=True, timeout=600)


def test_reference_acceptance_with_gpu_shim(gpu):
    r = _run("acceptance_gpu")
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("PASS: criterion") == 7


def test_reference_model_forward_on_gpu_experts(gpu):
    r = _run("shim_model_forward")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "GPU moe_ffn_forward calls" in r.stdout and r.stdout.strip().endswith("PASS")
