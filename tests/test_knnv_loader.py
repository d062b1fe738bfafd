"""KNNV dataset files (the reference's load_dataset, io.cpp:64-97) through the
engine's loader: knn_b200_knnv_header (host only) and
knn_b200_load_knnv_device (parallel preads through pinned staging, checks on
the device).  Error behaviour is pinned to the reference CLI compiled from its
own sources (oracle/_ref/tknn_ref, whose `run` mode calls load_dataset and
prints the IoError / ValidationError message with exit code 3,
tools/main.cpp:225-240)."""
from __future__ import annotations

import struct
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_CLI = ROOT / "oracle" / "_ref" / "tknn_ref"


def write_knnv(path, x, version=1, magic=b"KNNV", extra=b""):
    n, d = x.shape
    path.write_bytes(magic + struct.pack("<III", version, n, d) + np.ascontiguousarray(x, "<f4").tobytes() + extra)


def reference_error(path) -> str:
    p = subprocess.run([str(REF_CLI), "--mode", "run", "--input", str(path), "--output", str(path) + ".out", "--k",
                        "3"], capture_output=True, text=True, timeout=120)
    assert p.returncode == 3, p.stdout + p.stderr
    return p.stderr.strip().removeprefix("error: ")


def bad_files(tmp_path, c_oracle):
    x = c_oracle.generate(10, 4, 1)
    short = tmp_path / "short.knnv"
    short.write_bytes(b"KNNV\x01\x00")
    magic = tmp_path / "magic.knnv"
    write_knnv(magic, x, magic=b"KNNX")
    version = tmp_path / "version.knnv"
    write_knnv(version, x, version=7)
    size = tmp_path / "size.knnv"
    write_knnv(size, x, extra=b"\x00\x00")
    return [short, magic, version, size, tmp_path / "absent.knnv"]


def test_header_errors_match_the_reference(tmp_path, c_oracle):
    from paper_0906_0231_b200 import IoError, knnv_header
    x = c_oracle.generate(37, 5, 2)
    good = tmp_path / "good.knnv"
    write_knnv(good, x)
    assert knnv_header(good) == (37, 5)
    for f in bad_files(tmp_path, c_oracle):
        with pytest.raises(IoError) as e:
            knnv_header(f)
        if REF_CLI.exists():
            assert str(e.value) == reference_error(f), f.name


@pytest.mark.gpu
def test_device_load_matches_the_reference_generator(tmp_path, c_oracle):
    """A file written by the reference CLI (`--mode generate`, io.cpp:57-62 +
    save_dataset) loads bit for bit; a 300 MB file exercises the parallel
    staging; non-finite and n < 2 files raise the reference's messages."""
    import torch
    from paper_0906_0231_b200 import Context, IoError, ValidationError, load_knnv_torch
    ctx = Context(0)
    try:
        if REF_CLI.exists():
            f = tmp_path / "gen.knnv"
            p = subprocess.run([str(REF_CLI), "--mode", "generate", "--output", str(f), "--n", "3000", "--d", "19",
                                "--seed", "11"], capture_output=True, text=True, timeout=120)
            assert p.returncode == 0, p.stderr
            x = load_knnv_torch(ctx, f)
            assert np.array_equal(x.cpu().numpy(), c_oracle.generate(3000, 19, 11))
        big = tmp_path / "big.knnv"
        xb = c_oracle.generate(300_000, 250, 3)
        write_knnv(big, xb)
        assert np.array_equal(load_knnv_torch(ctx, big).cpu().numpy(), xb)
        nonfinite = tmp_path / "nan.knnv"
        xn = c_oracle.generate(50, 6, 4)
        xn[31, 4] = np.inf
        write_knnv(nonfinite, xn)
        with pytest.raises(ValidationError) as e:
            load_knnv_torch(ctx, nonfinite)
        if REF_CLI.exists():
            assert str(e.value) == reference_error(nonfinite)
        one = tmp_path / "one.knnv"
        write_knnv(one, c_oracle.generate(1, 6, 4))
        with pytest.raises(ValidationError) as e:
            load_knnv_torch(ctx, one)
        if REF_CLI.exists():
            assert str(e.value) == reference_error(one)
        for f in bad_files(tmp_path, c_oracle):
            with pytest.raises(IoError):
                load_knnv_torch(ctx, f)
        torch.cuda.synchronize()
    finally:
        ctx.close()
