"""CPU tests of the boundary: the C-ABI library loads and exports every symbol
include/ifa_b200.h declares, argument validation mirrors the reference's
exception behaviour (no compute calls need a GPU for these paths), the Python
API refuses CPU tensors (no CPU fallback), and the sharding plan."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "ifa_b200.h")).read()
    return sorted(set(re.findall(r"^(?:int|const char\*)\s+(ifa_\w+)\s*\(", text, re.M)))


def test_header_and_loader_agree():
    from paper_2409_16997_b200 import _lib
    assert _declared_symbols() == sorted(_lib.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol():
    from paper_2409_16997_b200 import _lib
    lib = _lib.load()
    for name in _declared_symbols():
        assert hasattr(lib, name), name
    out = os.popen(f"nm -D --defined-only {_lib.LIB_PATH}").read()
    for name in _declared_symbols():
        assert re.search(rf"\bT {name}\b", out), name
    assert b"sm_100a" in lib.ifa_version()


def test_library_is_sm100a_only():
    from paper_2409_16997_b200 import _lib
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {_lib.LIB_PATH}").read()
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_sass_uses_tcgen05_and_tma():
    from paper_2409_16997_b200 import _lib
    sass = os.popen(f"/usr/local/cuda/bin/cuobjdump -sass {_lib.LIB_PATH}").read()
    for mnemonic in ("UTCIMMA", "UTMALDG", "LDTM", "STTM"):
        assert mnemonic in sass, mnemonic


def _fwd(lib, n=4, d=4, br=64, bc=64, flags=0, slices=1, ptr=1):
    p = C.c_void_p(ptr)
    return lib.ifa_int_flash_fwd(p, p, p, p, p, p, p, slices, n, d, br, bc, flags, None, None)


def test_abi_validation_mirrors_reference_exceptions():
    from paper_2409_16997_b200 import _lib
    lib = _lib.load()
    assert _fwd(lib, n=0) == _lib.IFA_EINVAL           # attention.cpp:215-218 empty q
    assert b"empty q" in lib.ifa_last_error()
    assert _fwd(lib, d=0) == _lib.IFA_EINVAL
    assert _fwd(lib, br=0) == _lib.IFA_EINVAL          # gemm.cpp:16-20
    assert _fwd(lib, bc=0) == _lib.IFA_EINVAL
    assert b"Br and Bc" in lib.ifa_last_error()
    assert _fwd(lib, d=133145) == _lib.IFA_EOVERFLOW   # gemm.cpp:22-28
    assert _fwd(lib, n=133145, bc=133145) == _lib.IFA_EOVERFLOW
    # head dims > 128 run (attn.cu launch_wide); the S / P-code dump does not
    p = C.c_void_p(1)
    assert lib.ifa_int_flash_fwd_dump(p, p, p, p, p, p, p, 1, 4, 129, 64, 128, _lib.FLAG_FAST,
                                      p, None, None) == _lib.IFA_ENOTSUP
    assert b"head dim 129" in lib.ifa_last_error()
    assert _fwd(lib, flags=8) == _lib.IFA_EINVAL
    assert _fwd(lib, slices=0) == _lib.IFA_OK          # nothing to do
    assert _fwd(lib, ptr=0) == _lib.IFA_EINVAL         # null pointers
    assert lib.ifa_quantize_per_row(None, -1, 4, None, None, None, None) == _lib.IFA_EINVAL
    assert lib.ifa_quantize_per_row(None, 0, 4, None, None, None, None) == _lib.IFA_OK
    assert lib.ifa_quantize_per_tensor(None, 1, 2, 2, None, None, None, None, None) == \
        _lib.IFA_EINVAL


def test_check_maps_status_to_reference_exception_types():
    from paper_2409_16997_b200 import _lib
    lib = _lib.load()
    _fwd(lib, n=0)
    with pytest.raises(ValueError):
        _lib.check(_lib.IFA_EINVAL)
    _fwd(lib, d=133145)
    with pytest.raises(OverflowError):
        _lib.check(_lib.IFA_EOVERFLOW)


def test_python_api_refuses_cpu_tensors():
    import torch
    import paper_2409_16997_b200 as ifa
    with pytest.raises(ValueError, match="CUDA"):
        ifa.quantize_per_row(torch.ones(2, 2))
    with pytest.raises(ValueError, match="CUDA"):
        ifa.quantize_per_tensor(torch.ones(2, 2))
    i8 = torch.zeros(2, 2, dtype=torch.int8)
    inputs = ifa.QuantizedAttentionInputs(ifa.QuantizedRows(i8, torch.ones(2)),
                                          ifa.QuantizedRows(i8, torch.ones(2)),
                                          ifa.QuantizedTensor(i8, torch.ones(())))
    with pytest.raises(ValueError, match="CUDA"):
        ifa.int_flash_attention(inputs)
    with pytest.raises(ValueError):
        ifa.BlockSpec(0, 64).validate()


def test_loader_fails_loudly_without_library(monkeypatch, tmp_path):
    from paper_2409_16997_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(_lib.NativeLibraryError, match="no CPU fallback"):
        _lib.load()


@pytest.mark.parametrize("total,world", [(128, 1), (128, 2), (2048, 8), (7, 3), (3, 8)])
def test_shard_ranges_partition_exactly(total, world):
    from paper_2409_16997_b200.sharding import owner_of, shard_range
    seen = []
    for r in range(world):
        lo, hi = shard_range(total, world, r)
        assert 0 <= lo <= hi <= total
        seen.extend(range(lo, hi))
    assert seen == list(range(total))
    sizes = [shard_range(total, world, r)[1] - shard_range(total, world, r)[0]
             for r in range(world)]
    assert max(sizes) - min(sizes) <= 1
    for g in range(total):
        lo, hi = shard_range(total, world, owner_of(g, total, world))
        assert lo <= g < hi


def test_capture_of_reference_interface_names():
    """The host mirror keeps the reference's names and defaults."""
    import paper_2409_16997_b200 as ifa
    assert ifa.BlockSpec().Br == 64 and ifa.BlockSpec().Bc == 64        # gemm.hpp:15-16
    assert ifa.AttentionConfig().apply_sqrt_d_scaling is False           # attention.hpp:27
    a = ifa.PCodeAudit()
    assert (a.min_code, a.max_code, a.row_max_block_hits_127, a.rows_audited) == \
        (127, 0, True, 0)                                                 # attention.hpp:76-79
