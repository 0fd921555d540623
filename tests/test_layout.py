"""HBM row layout (include/ember_gpu.h): ComplEx rows are held with their [re | im]
halves interleaved by pairs; the host converters and the library's agree, and the
round trip is the identity. CPU only (ember_rows_layout_host needs no GPU)."""
import ctypes as C

import numpy as np
import pytest

import paper_2101_08358_b200 as eb
from paper_2101_08358_b200._lib import KIND, lib


def _lib_convert(x, kind, to_hbm):
    y = np.ascontiguousarray(x.copy())
    eb.check(lib().ember_rows_layout_host(KIND[kind], y.shape[1], y.ctypes.data, y.shape[0], int(to_hbm)))
    return y


@pytest.mark.parametrize("d", [4, 8, 100, 132, 800])
def test_complex_pairs_interleaved(d):
    rng = np.random.default_rng(d)
    x = rng.standard_normal((5, d)).astype(np.float32)
    h = eb.rows_to_hbm(x, "complex")
    # quad q holds {re 2q, re 2q+1, im 2q, im 2q+1}
    half = d // 2
    for q in range(d // 4):
        want = np.stack([x[:, 2 * q], x[:, 2 * q + 1], x[:, half + 2 * q], x[:, half + 2 * q + 1]], 1)
        assert np.array_equal(h[:, 4 * q:4 * q + 4], want)
    assert h.tobytes() == _lib_convert(x, "complex", True).tobytes()
    assert eb.rows_to_disk(h, "complex").tobytes() == x.tobytes()
    assert _lib_convert(h, "complex", False).tobytes() == x.tobytes()


@pytest.mark.parametrize("kind", ["dot", "distmult"])
def test_real_models_keep_coordinate_order(kind):
    x = np.arange(3 * 12, dtype=np.float32).reshape(3, 12)
    assert eb.rows_to_hbm(x, kind).tobytes() == x.tobytes()
    assert _lib_convert(x, kind, True).tobytes() == x.tobytes()


def test_layout_rejects_bad_dims():
    x = np.zeros((2, 6), np.float32)
    assert lib().ember_rows_layout_host(KIND["complex"], 6, x.ctypes.data, 2, 1) == 1
    assert "multiple of 4" in lib().ember_last_error().decode()
