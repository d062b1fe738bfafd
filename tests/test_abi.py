"""CPU checks of the C ABI library and the host-side mirror (no GPU compute)."""
from __future__ import annotations

import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "knn_b200.h"


def declared_functions() -> list[str]:
    text = HEADER.read_text()
    return sorted(set(re.findall(r"KNN_B200_API\s+[\w\s\*]*?\b(knn_b200_\w+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared_functions()
    assert "knn_b200_solve" in names and "knn_b200_solve_rows_device" in names
    from paper_0906_0231_b200 import _lib
    assert sorted(_lib.EXPORTS) == names


def test_library_loads_and_exports_every_symbol():
    from paper_0906_0231_b200 import _lib
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (knn_b200_\w+)", out))
    assert exported == set(declared_functions())
    assert lib.knn_b200_abi_version() == _lib.ABI_VERSION


def test_library_is_sm100a_native():
    from paper_0906_0231_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_lib.LIB_PATH)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_fails_loudly():
    """Without a device the engine must error, never compute on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_0906_0231_b200 import _lib
    lib = _lib.load()
    cnt = ctypes.c_int(-1)
    assert lib.knn_b200_device_count(ctypes.byref(cnt)) == 0 and cnt.value == 0
    h = ctypes.c_void_p()
    assert lib.knn_b200_create(0, ctypes.byref(h)) == _lib.ERR_INTERNAL
    x = np.zeros((4, 2), np.float32)
    idx = np.zeros((4, 1), np.uint32)
    dist = np.zeros((4, 1), np.float32)
    rc = lib.knn_b200_solve_multi(x.ctypes.data, 4, 2, 1, 1, 0, 1, idx.ctypes.data, dist.ctypes.data, None)
    assert rc == _lib.ERR_INTERNAL
    from paper_0906_0231_b200 import Dataset, EngineError, EngineOptions, solve_knn, squared_euclidean
    with pytest.raises(EngineError):
        solve_knn(Dataset.from_array(x), squared_euclidean(), EngineOptions(k=1))


def test_config_errors_before_device():
    from paper_0906_0231_b200 import _lib
    lib = _lib.load()
    x = np.zeros((4, 2), np.float32)
    idx = np.zeros((4, 1), np.uint32)
    dist = np.zeros((4, 1), np.float32)
    assert lib.knn_b200_solve_multi(x.ctypes.data, 4, 2, 0, 1, 0, 1, idx.ctypes.data, dist.ctypes.data,
                                    None) == _lib.ERR_CONFIG
    assert "k must be at least 1" in _lib.last_error()
    assert lib.knn_b200_solve_multi(x.ctypes.data, 1, 2, 1, 1, 0, 1, idx.ctypes.data, dist.ctypes.data,
                                    None) == _lib.ERR_CONFIG
    assert lib.knn_b200_solve_multi(x.ctypes.data, 4, 2, 1, 9, 0, 1, idx.ctypes.data, dist.ctypes.data,
                                    None) == _lib.ERR_CONFIG


def test_plan_mirrors_reference_schedule():
    # test_schedule.cpp:24-38, 50-56 / schedule.cpp:10-38
    from paper_0906_0231_b200 import ConfigError, auto_gsize, make_plan
    assert auto_gsize(10, 64) == 64
    assert auto_gsize(300, 64) == 320
    assert auto_gsize(20000, 64) == 4096
    assert make_plan(100, 128, 32, 32, 32, 1).n_grids == 1
    assert make_plan(1000, 64, 64, 32, 32, 1).n_grids == 16
    assert make_plan(1025, 64, 64, 32, 32, 1).n_grids == 17
    for bad in [(1, 8, 8, 1, 1, 1), (10, 0, 1, 1, 1, 1), (10, 8, 9, 1, 1, 1), (10, 8, 8, 0, 1, 1),
                (10, 8, 8, 1, 0, 1), (10, 8, 8, 1, 1, 0)]:
        with pytest.raises(ConfigError):
            make_plan(*bad)


def test_engine_option_errors_precede_compute():
    # test_engine.cpp:119-141: these raise before any device work
    from paper_0906_0231_b200 import (ConfigError, Dataset, EngineOptions, ValidationError, hellinger,
                                      solve_knn)
    from oracle import c_oracle
    ds = Dataset.from_array(c_oracle().generate(10, 2, 1))
    with pytest.raises(ConfigError):
        solve_knn(ds, hellinger(), EngineOptions(k=0))
    with pytest.raises(ConfigError):
        solve_knn(ds, hellinger(), EngineOptions(k=1, bsize=64, gsize=32))
    with pytest.raises(ConfigError):
        solve_knn(ds, hellinger(), EngineOptions(k=1, workers=0))
    with pytest.raises(ValidationError):
        solve_knn(Dataset(3, 1, [0.5, -1.0, 0.25]), hellinger(), EngineOptions(k=1))
    with pytest.raises(ValidationError):
        Dataset(2, 1, [0.5, float("nan")])
    with pytest.raises(ValidationError):
        Dataset(1, 1, [0.5])


def test_distance_registry():
    from paper_0906_0231_b200 import ConfigError, distance_by_name, distance_names
    assert distance_names() == ["cosine", "euclidean", "hellinger", "manhattan", "root_of_squares", "sqeuclidean"]
    assert distance_by_name("hellinger").nonnegative_domain
    with pytest.raises(ConfigError):
        distance_by_name("l1")


def test_ordered_key_encoding_matches_reference_order():
    """The u64 key (ordered float bits << 32 | index) sorts exactly like the
    reference's Neighbor operator< (heap.hpp:21-24); restated in numpy."""
    def ordered(f):
        b = (np.asarray(f, np.float32) + np.float32(0.0)).view(np.uint32).astype(np.uint64)
        return np.where(b & 0x80000000, ~b & 0xFFFFFFFF, b | 0x80000000)

    rng = np.random.default_rng(3)
    dist = np.concatenate([rng.standard_normal(500).astype(np.float32),
                           np.array([0.0, -0.0, 1.0, 1.0, -1.0, 3e38, -3e38], np.float32)])
    index = rng.integers(0, 1000, dist.size).astype(np.uint64)
    keys = (ordered(dist) << np.uint64(32)) | index
    by_key = np.argsort(keys, kind="stable")
    ref = sorted(range(dist.size), key=lambda i: (float(dist[i]), int(index[i])))
    assert [(float(dist[i]), int(index[i])) for i in by_key] == [(float(dist[i]), int(index[i])) for i in ref]
