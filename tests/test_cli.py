"""CLI harness: particle file format, subcommands, JSON reports and exit codes
0 / 1 / 2 / 3.  Host-only subcommands run here; run / verify / bench need the GPU (marked)."""
import json
import os
import struct

import numpy as np
import pytest

from conftest import gpu_available
from paper_2303_08394_b200 import cli, host


def _run(argv, capsys):
    rc = cli.main(argv)
    out = capsys.readouterr().out
    return rc, (json.loads(out) if out.strip().startswith("{") else None)


def test_generate_format_and_determinism(tmp_path, capsys):
    a, b, c = (str(tmp_path / f"{x}.bin") for x in "abc")
    assert _run(["generate", "--dist", "sphere-surface", "--n", "8", "--seed", "1", "--out", a], capsys)[0] == 0
    assert _run(["generate", "--dist", "sphere-surface", "--n", "8", "--seed", "1", "--out", b], capsys)[0] == 0
    assert _run(["generate", "--dist", "sphere-surface", "--n", "8", "--seed", "2", "--out", c], capsys)[0] == 0
    raw = open(a, "rb").read()
    assert struct.unpack("<Q", raw[:8])[0] == 8 and len(raw) == 8 + 8 * 32
    assert raw == open(b, "rb").read() and raw != open(c, "rb").read()
    pos, q = cli.read_particles(a)
    assert pos.shape == (8, 3) and np.all(q == 1.0)  # unit charges by default
    r = np.linalg.norm(pos - 0.5, axis=1)
    assert np.allclose(r, 0.5, rtol=1e-12)  # radius 0.5 about the cube centre


def test_stats_report(tmp_path, capsys):
    p = str(tmp_path / "u.bin")
    cli.main(["generate", "--dist", "uniform-cube", "--n", "20000", "--out", p])
    capsys.readouterr()
    rc, rep = _run(["stats", "--input", p, "--n-crit", "64"], capsys)
    assert rc == 0
    t = host.Tree(cli.read_particles(p)[0], 64)
    assert rep["leaves"] == t.n_leaves and rep["depth"] == t.depth
    assert set(rep["lists"]) == {"U", "V", "W", "X"} and rep["lists"]["W"]["mean"] == 0.0  # uniform tree


def test_precompute_writes_loadable_cache(tmp_path, capsys):
    p, cache = str(tmp_path / "s.bin"), str(tmp_path / "ops.kifmm")
    cli.main(["generate", "--dist", "two-cluster", "--n", "3000", "--out", p])
    capsys.readouterr()
    rc, rep = _run(["precompute", "--input", p, "--p", "4", "--cache", cache], capsys)
    assert rc == 0 and os.path.exists(cache)
    ops = host.Operators.load(cache, rep["fingerprint"])
    assert ops.p == 4 and ops.n_e == rep["n_e"]


def test_exit_codes(tmp_path, capsys):
    assert cli.main(["stats"]) == cli.EXIT_USAGE  # missing --input
    assert cli.main(["nonsense"]) == cli.EXIT_USAGE
    assert cli.main(["precompute", "--p", "4"]) == cli.EXIT_USAGE  # no domain, no cache
    bad = tmp_path / "bad.bin"
    bad.write_bytes(struct.pack("<Q", 10) + b"\0" * 16)  # truncated payload
    assert cli.main(["stats", "--input", str(bad)]) == cli.EXIT_DATA
    assert cli.main(["stats", "--input", str(tmp_path / "missing.bin")]) == cli.EXIT_DATA


def test_write_read_roundtrip(tmp_path):
    pos = np.random.default_rng(0).random((100, 3))
    q = np.random.default_rng(1).random(100)
    p = str(tmp_path / "r.bin")
    cli.write_particles(p, pos, q)
    a, b = cli.read_particles(p)
    assert np.array_equal(a, pos) and np.array_equal(b, q)


@pytest.mark.skipif(gpu_available(), reason="checks the no-device failure mode")
def test_run_without_device_is_data_error(tmp_path, capsys):
    p = str(tmp_path / "s.bin")
    cli.main(["generate", "--dist", "uniform-cube", "--n", "500", "--out", p])
    capsys.readouterr()
    assert cli.main(["run", "--input", p, "--p", "3", "--n-crit", "20"]) == cli.EXIT_DATA


@pytest.mark.gpu
def test_run_verify_bench_on_gpu(require_gpu, tmp_path, capsys):
    p = str(tmp_path / "s.bin")
    cli.main(["generate", "--dist", "sphere-surface", "--n", "5000", "--seed", "3", "--out", p])
    capsys.readouterr()
    rc, rep = _run(["run", "--input", p, "--p", "6", "--n-crit", "50", "--verify"], capsys)
    assert rc == 0 and rep["relative_error_vs_direct"] <= 1e-5  # acceptance #2
    assert set(rep["lists"]) == {"U", "V", "W", "X"} and rep["operator_ms"]["total_ms"] > 0
    assert _run(["verify", "--input", p, "--p", "6", "--n-crit", "50"], capsys)[0] == 0
    assert _run(["verify", "--input", p, "--p", "2", "--n-crit", "50", "--tolerance", "1e-9"],
                capsys)[0] == cli.EXIT_NUMERICAL
    rc, rep = _run(["bench", "--sizes", "20000,40000", "--repeats", "2", "--p", "4"], capsys)
    assert rc == 0 and len(rep["rows"]) == 2 and "direct_s" in rep["rows"][0]
