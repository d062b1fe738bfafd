"""The reference CLI (tools/main.cpp, unmodified) relinked to the B200 engine.

`build/tknn_b200` is the reference's own main.cpp compiled against the B200
drop-in solve_knn (Makefile `ref-bins`); `oracle/_ref/tknn_ref` is the same
main.cpp on the reference CPU engine.  Cases restate
/root/reference/proj/tests/test_cli.cpp (cited per case); outputs of `run`
must be byte-identical to the reference CLI's.
"""
from __future__ import annotations

import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
B200 = ROOT / "build" / "tknn_b200"
REF = ROOT / "oracle" / "_ref" / "tknn_ref"

pytestmark = pytest.mark.skipif(not B200.exists(), reason="CLI not built (needs /root/reference at build time)")


def cli(args: str, binary: Path = B200, **env):
    p = subprocess.run([str(binary), *args.split()], capture_output=True, text=True, timeout=600,
                       env={**__import__("os").environ, **env})
    return p.returncode, p.stdout + p.stderr


def test_generate_deterministic_and_sized(tmp_path):
    # test_cli.cpp:52-64 (no device work: generate never calls solve_knn)
    a, b, c = (tmp_path / x for x in ("a.knnv", "b.knnv", "c.knnv"))
    assert cli(f"--mode generate --output {a} --n 100 --d 8 --seed 31")[0] == 0
    assert cli(f"--mode generate --output {b} --n 100 --d 8 --seed 31")[0] == 0
    assert cli(f"--mode generate --output {c} --n 100 --d 8 --seed 32")[0] == 0
    assert a.stat().st_size == 16 + 100 * 8 * 4
    assert a.read_bytes() == b.read_bytes() != c.read_bytes()


def test_parameter_errors_exit_2(tmp_path):
    # test_cli.cpp:137-156: rejected before any device work
    data, out = tmp_path / "data.knnv", tmp_path / "out.tsv"
    assert cli(f"--mode generate --output {data} --n 20 --d 4 --seed 1")[0] == 0
    for args in (f"--mode run --input {data} --output {out} --k 0",
                 f"--mode run --input {data} --output {out} --k 5 --distance warp",
                 f"--mode run --input {data} --output {out} --k 5 --gsize 8 --bsize 16",
                 f"--mode run --input {data} --output {out} --k 5 --lanes 0",
                 f"--mode generate --output {data}.x --n 1 --d 4",
                 "--mode run --k 5",
                 "--mode teleport"):
        assert cli(args)[0] == 2, args
    assert not out.exists()


def test_missing_input_exits_3(tmp_path):
    # test_cli.cpp:127-135
    out = tmp_path / "out.tsv"
    assert cli(f"--mode run --input {tmp_path / 'absent.knnv'} --output {out} --k 5")[0] == 3
    assert not out.exists()


@pytest.mark.gpu
def test_run_bytes_identical_across_lanes_and_to_reference(tmp_path):
    # test_cli.cpp:66-99, plus byte equality with the reference CLI
    data = tmp_path / "data.knnv"
    assert cli(f"--mode generate --output {data} --n 100 --d 12 --seed 5")[0] == 0
    outs = []
    for lanes in ("1", "2", "4", "2"):
        out = tmp_path / f"out{len(outs)}.tsv"
        rc, log = cli(f"--mode run --input {data} --output {out} --k 10 --lanes {lanes}")
        assert rc == 0, log
        outs.append(out.read_bytes())
    assert all(o == outs[0] for o in outs)
    lines = outs[0].decode().splitlines()
    assert len(lines) == 100 and all(l.split("\t")[0] == str(i) for i, l in enumerate(lines))
    if REF.exists():
        ref_out = tmp_path / "ref.tsv"
        assert cli(f"--mode run --input {data} --output {ref_out} --k 10", binary=REF)[0] == 0
        assert ref_out.read_bytes() == outs[0]


@pytest.mark.gpu
@pytest.mark.parametrize("arith", ["exact", "tensor"])
def test_binary_output_matches_reference(tmp_path, arith):
    # test_cli.cpp:101-112
    data, bin_, ref = tmp_path / "data.knnv", tmp_path / "out.knnr", tmp_path / "ref.knnr"
    assert cli(f"--mode generate --output {data} --n 40 --d 6 --seed 2")[0] == 0
    assert cli(f"--mode run --input {data} --output {bin_} --k 7 --format binary", KNN_B200_ARITH=arith)[0] == 0
    b = bin_.read_bytes()
    assert len(b) == 16 + 40 * 7 * 8 and b[:4] == b"KNNR"
    if REF.exists():
        assert cli(f"--mode run --input {data} --output {ref} --k 7 --format binary", binary=REF)[0] == 0
        assert ref.read_bytes() == b


@pytest.mark.gpu
def test_verify_pass(tmp_path):
    # test_cli.cpp:114-122
    data = tmp_path / "data.knnv"
    assert cli(f"--mode generate --output {data} --n 150 --d 10 --seed 77")[0] == 0
    rc, log = cli(f"--mode verify --input {data} --k 12 --lanes 3 --workers 2")
    assert rc == 0 and "PASS" in log, log


@pytest.mark.gpu
def test_bench_table(tmp_path):
    # test_cli.cpp:124-135
    data = tmp_path / "data.knnv"
    assert cli(f"--mode generate --output {data} --n 400 --d 8 --seed 3")[0] == 0
    rc, log = cli(f"--mode bench --input {data} --k 10 --lane-counts 1,2 --distance sqeuclidean")
    assert rc == 0, log
    assert "brute-force" in log and "lanes=1" in log and "lanes=2" in log and "DIVERGES" not in log


@pytest.mark.gpu
def test_domain_violation_exits_3(tmp_path):
    # test_cli.cpp:158-166: a valid file whose data violates Hellinger's domain
    import numpy as np
    data = tmp_path / "neg.knnv"
    vals = np.array([0.5, -0.25, 0.75, 0.1], np.float32)
    data.write_bytes(b"KNNV" + np.array([1, 2, 2], "<u4").tobytes() + vals.tobytes())
    rc, log = cli(f"--mode run --input {data} --output {tmp_path / 'o.tsv'} --k 1")
    assert rc == 3, log


@pytest.mark.gpu
def test_reference_acceptance_criterion_5_cli_determinism():
    """acceptance.cpp criterion 5 (CLI bytes independent of lane count) with
    the B200 CLI."""
    acc = ROOT / "oracle" / "_ref" / "acceptance_b200"
    if not acc.exists():
        pytest.skip("acceptance_b200 not built")
    p = subprocess.run([str(acc), "--only", "5", "--cli", str(B200)], capture_output=True, text=True, timeout=600)
    assert p.returncode == 0 and "PASS" in p.stdout, p.stdout + p.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("fmt", ["text", "binary"])
def test_double_accum_cli_matches_reference_double_build(tmp_path, fmt):
    """main.cpp in the KNN_DOUBLE_ACCUM build: `run` on the double drop-in
    (build/tknn_b200_f64) writes the same bytes as on the reference's double
    engine (oracle/_ref/f64/tknn_ref), for every lane count."""
    b200 = ROOT / "build" / "tknn_b200_f64"
    ref = ROOT / "oracle" / "_ref" / "f64" / "tknn_ref"
    if not (b200.exists() and ref.exists()):
        pytest.skip("double-build CLIs not built")
    data = tmp_path / "data.knnv"
    assert cli(f"--mode generate --output {data} --n 150 --d 20 --seed 9")[0] == 0
    ref_out = tmp_path / "ref.out"
    rc, log = cli(f"--mode run --input {data} --output {ref_out} --k 12 --format {fmt}", binary=ref)
    assert rc == 0, log
    for lanes in ("1", "3"):
        out = tmp_path / f"b200_{lanes}.out"
        rc, log = cli(f"--mode run --input {data} --output {out} --k 12 --lanes {lanes} --format {fmt}", binary=b200)
        assert rc == 0, log
        assert out.read_bytes() == ref_out.read_bytes()
