"""LTEN files and the CLI.  The format is pinned
against the reference's own write_tensor / read_tensor (tensor_io.hpp:94-150,
compiled in place via oracle/_ref); the CLI's usage errors and exit codes
follow tools/lance_main.cpp:37-39,180-195."""
import os
import struct

import numpy as np
import pytest

from oracle import Reference, reference_available
from paper_2003_08646_b200 import tensor_io
from paper_2003_08646_b200.cli import main as cli_main

needs_ref = pytest.mark.skipif(not reference_available(), reason="reference shim not built")


def sample(shape, seed=0):
    a = np.random.default_rng(seed).standard_normal(shape).astype(np.float32)
    a.flat[3] = np.float32(-0.0)
    a.flat[5] = np.float32("inf")
    a.view(np.uint32).flat[7] = 0x7FC00123  # NaN payload must survive
    return a


def test_roundtrip_bits(tmp_path):
    a = sample((2, 3, 4, 5))
    p = str(tmp_path / "a.lten")
    tensor_io.write_tensor(p, a)
    assert os.path.getsize(p) == 39 + 4 * a.size
    b = tensor_io.read_tensor(p)
    assert b.shape == a.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


@needs_ref
def test_bytes_identical_to_reference_writer(tmp_path):
    ref = Reference()
    a = sample((1, 5, 7, 3), 1)
    ours, theirs = str(tmp_path / "o.lten"), str(tmp_path / "r.lten")
    tensor_io.write_tensor(ours, a)
    ref.write_lten(theirs, a)
    assert open(ours, "rb").read() == open(theirs, "rb").read()
    assert np.array_equal(ref.read_lten(ours).view(np.uint32), a.view(np.uint32))


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"LTEX" + b[4:], "bad magic"),
    (lambda b: b[:4] + struct.pack("<H", 2) + b[6:], "unsupported format version"),
    (lambda b: b[:6] + b"\x01" + b[7:], "unsupported dtype code"),
    (lambda b: b[:20], "truncated header"),
    (lambda b: b[:-4], "truncated payload"),
    (lambda b: b[:7] + struct.pack("<Q", 0) + b[15:], "dimension overflow"),
    (lambda b: b[:7] + struct.pack("<4Q", 1 << 20, 1 << 20, 1, 1) + b[39:], "dimension overflow"),
])
def test_format_errors_match_reference(tmp_path, mutate, msg):
    a = sample((1, 2, 2, 2))
    p = str(tmp_path / "a.lten")
    tensor_io.write_tensor(p, a)
    bad = str(tmp_path / "bad.lten")
    open(bad, "wb").write(mutate(open(p, "rb").read()))
    with pytest.raises(tensor_io.FormatError, match=msg):
        tensor_io.read_tensor(bad)
    if reference_available():
        with pytest.raises(Exception, match=msg):
            Reference().read_lten(bad)


def test_fnv1a64_matches_definition():
    a = sample((1, 2, 3, 4), 2)
    h = 1469598103934665603
    for byte in a.astype("<f4").tobytes():
        h = ((h ^ byte) * 1099511628211) & ((1 << 64) - 1)
    assert tensor_io.fnv1a64(a) == h


def test_cli_usage_errors(tmp_path, capsys):
    assert cli_main(["run"]) == 2                                   # missing required options
    assert cli_main(["nonsense"]) == 2
    x = str(tmp_path / "x.lten")
    tensor_io.write_tensor(x, sample((1, 4, 4, 2)))
    f = str(tmp_path / "f.lten")
    tensor_io.write_tensor(f, np.zeros((3, 3, 3, 2), np.float32))
    out = str(tmp_path / "y.lten")
    assert cli_main(["run", "--input", x, "--filters", f, "--out", out, "--engine", "direct"]) == 2
    assert cli_main(["run", "--input", str(tmp_path / "missing.lten"), "--filters", f, "--out", out]) == 2
    assert cli_main(["run", "--input", x, "--filters", f, "--out", out, "--granularity", "tile"]) == 2
    err = capsys.readouterr().err
    assert "Gemm mode cannot use PerTile" in err
    bad = str(tmp_path / "bad.lten")
    open(bad, "wb").write(b"JUNK")
    assert cli_main(["run", "--input", bad, "--filters", f, "--out", out]) == 2
