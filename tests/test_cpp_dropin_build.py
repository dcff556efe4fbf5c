"""CPU-side checks of the compiled C++ drop-in (cpp/): the reference's proj/core objects keep
every symbol except the hot-path ones, which cpp/dilocox_b200.cpp defines — so the reference's
run_experiment reaches the device path (and, with no GPU here, fails loudly in the CUDA
runtime instead of silently running the CPU reference), while the unmodified reference build
(oracle/_ref/ref_run) runs the same experiment on the CPU."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B = os.path.join(ROOT, "cpp", "_build")


def _need(path):
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (needs /root/reference at build time)")


def _nm(path, *flags):
    return subprocess.run(["nm", *flags, path], capture_output=True, text=True).stdout


def test_hot_path_symbols_are_replaced():
    lib = os.path.join(B, "libdilocox_core_b200.so")
    _need(lib)
    replaced = [l.strip() for l in open(os.path.join(B, "replaced.txt")) if l.strip()]
    assert len(replaced) == 6  # compress, decompress, measure_error, effective_rank,
    #                            allreduce_avg, nesterov_outer_step
    # the drop-in TU is the only strong definition of each; the reference objects carry them weak
    ours = set(re.findall(r" T (\S+)", _nm(os.path.join(B, "dilocox_b200.o"))))
    assert set(replaced) <= ours
    for obj in ("compress", "collective", "optim"):
        weak = _nm(os.path.join(B, "weak", obj + ".o"))
        for sym in replaced:  # defined in this reference object -> weak, never strong
            assert not re.search(r" T " + re.escape(sym) + r"\b", weak), (obj, sym)
    # the shared library exports them, defined, and needs the C-ABI library
    dyn = _nm(lib, "-D", "--defined-only")
    for sym in replaced:
        assert f" {sym}" in dyn
    assert "dlx_compress" in _nm(lib, "-D", "--undefined-only")


def test_dropin_reaches_the_device_and_reference_runs_on_cpu(tmp_path):
    dropin, ref = os.path.join(B, "dropin_run"), os.path.join(ROOT, "oracle", "_ref", "ref_run")
    _need(dropin)
    _need(ref)
    r = subprocess.run([ref, "steps=10", str(tmp_path / "ref")], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr
    assert os.path.getsize(tmp_path / "ref.bin") > 0
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present: tests/test_gpu_dropin.py covers the device run")
    d = subprocess.run([dropin, "steps=10", str(tmp_path / "dropin")], capture_output=True,
                       text=True, timeout=300)
    assert d.returncode != 0  # no silent CPU fallback
    assert "cuda" in d.stderr.lower() or "driver" in d.stderr.lower(), d.stderr
