"""CPU-only checks of the drop-in boundary: the C-ABI library loads, exports every symbol
include/dlx_b200.h declares, host-only entry points compute the reference's answers, and
device entry points fail loudly without a GPU (no silent CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dlx_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(dlx_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2506_21263_b200 import _lib
    L = _lib.lib()
    names = declared()
    assert len(names) >= 25
    for n in names:
        assert hasattr(L, n), n
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                        text=True).stdout
    exported = set(re.findall(r" T (dlx_\w+)", nm))
    assert set(names) <= exported
    assert set(_lib.PROTOS) <= exported


def test_library_is_sm100a():
    from paper_2506_21263_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_entry_points_without_gpu():
    from paper_2506_21263_b200 import api
    assert api.adapt_compression([2048, 1024, 512, 512, 512], 2048, 125, 5, 13) == (922, 69)
    assert api.adapt_compression([2048, 1024], 2048, 125, 5, 13) == (2048, 125)
    assert api.omega_bound(2, 4, 1) == 0.75
    from paper_2506_21263_b200 import ValidationError
    with pytest.raises(ValidationError):
        api.adapt_compression([1], 0, 125, 5, 13)


def test_host_rng_matches_oracle(oracle):
    from paper_2506_21263_b200 import api
    for seed, parts in [(1, (0xC09C, 3)), (7, (0xA7C4, 0, 5)), (0, (1,))]:
        k = api.stream_key(*parts)
        assert k == oracle.stream_key(*parts)
        assert api.rng_stream(seed, k) == oracle.stream(seed, k)


def test_device_calls_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2506_21263_b200 import CudaError, api
    with pytest.raises(CudaError):
        api.Context(0)


def test_named_layouts_param_counts():
    from paper_2506_21263_b200 import layouts
    assert layouts.numel(layouts.mini_opt()) == 10_763_264
    assert layouts.numel(layouts.opt_1_3b()) == 1_315_758_080
    assert layouts.numel(layouts.llama7b_layer()) == 202_383_360
    assert layouts.numel(layouts.qwen107b_stage(1)) == 1_358_981_120
    t = layouts.opt_1_3b()
    assert sum(1 for _, s in t if len(s) == 2) == 146 and sum(1 for _, s in t if len(s) == 1) == 242


def test_payload_formula_matches_oracle(oracle):
    """payload_bits for the named configs via the oracle formula."""
    from oracle.oracle import Table
    from paper_2506_21263_b200 import layouts
    t = Table([s for _, s in layouts.opt_1_3b()])
    assert oracle.payload_bits(t, t.ranks(32), 4) / 8 == pytest.approx(15.418e6, rel=1e-4)
    t = Table([s for _, s in layouts.mini_opt()])
    assert oracle.payload_bits(t, t.ranks(8), 8) / 8 == pytest.approx(240_616, abs=1)


def test_worker_sync_entry_points_on_cpu():
    """dlx_comm_unique_id needs only NCCL (dlopen'ed at run time), not a GPU; the other
    worker-sync calls reject a null context with a typed error instead of crashing."""
    from paper_2506_21263_b200 import _lib, api
    uid = api.comm_unique_id()
    assert len(uid) == 128 and any(uid)
    L = _lib.lib()
    assert L.dlx_comm_check(None) == 1
    assert L.dlx_exchange(None, None, 0, None, None, 0, 0, None) == 1
    assert L.dlx_comm_allgather(None, None, 0, None, None) == 1
    assert L.dlx_exchange_wait_warm(None, None) == 1


def test_bind_host_to_device_is_safe_without_nvml():
    """api.bind_host_to_device: without a GPU / NVML it is a no-op returning []; with one it
    returns a non-empty CPU list that the process is then pinned to."""
    import os
    from paper_2506_21263_b200 import api
    before = os.sched_getaffinity(0)
    try:
        cpus = api.bind_host_to_device(0)
        assert isinstance(cpus, list)
        if cpus:
            assert os.sched_getaffinity(0) == set(cpus)
        else:
            assert os.sched_getaffinity(0) == before
    finally:
        os.sched_setaffinity(0, before)
