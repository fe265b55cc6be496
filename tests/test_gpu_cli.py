"""`ifa_b200 quantize` (the reference CLI's cmd_quantize, ifa_main.cpp:164-197)
on the GPU: output codes/scales files equal the reference quantizers' and the
report lines match the reference's formula."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_2409_16997_b200", "lib", "ifa_b200")


@pytest.mark.parametrize("mode", ["per-row", "per-tensor"])
def test_cli_quantize_matches_reference(tmp_path, oracle, mode):
    from paper_2409_16997_b200 import tensor_io
    x = oracle.generate("normal", 37, 128, seed=11)
    src, dst = str(tmp_path / "x.ifa"), str(tmp_path / "x8.ifa")
    tensor_io.save_tensor(x, src)
    r = subprocess.run([CLI, "quantize", src, dst, "--mode", mode], capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    codes = tensor_io.load_int8_tensor(dst)
    scales = tensor_io.load_float_tensor(dst + ".scales")
    if mode == "per-row":
        want_c, want_s = oracle.quantize_per_row(x)
        want_s = want_s.reshape(-1, 1)
        restored = codes.astype(np.float64) * scales.astype(np.float64)
        bound = 0.5 * float(scales.max())
    else:
        want_c, ws = oracle.quantize_per_tensor(x)
        want_s = np.array([[ws]], np.float32)
        restored = codes.astype(np.float64) * float(scales[0, 0])
        bound = 0.5 * float(scales[0, 0])
    assert np.array_equal(codes, want_c)
    assert np.array_equal(scales.view(np.uint32), want_s.astype(np.float32).view(np.uint32))
    worst = float(np.abs(restored.astype(np.float32).astype(np.float64) - x).max())
    assert r.stdout.splitlines() == [
        f"wrote {dst} (i8 37x128) and {dst}.scales",
        "max round-trip error %s (bound scale/2 = %s)" % (_g6(worst), _g6(bound))]


def _g6(v):
    import ctypes
    buf = ctypes.create_string_buffer(64)
    ctypes.CDLL(None).snprintf(buf, 64, b"%.6g", ctypes.c_double(v))
    return buf.value.decode()
