"""The CLI on the GPU: `run` writes the bit-exact lance_gemm output and the
reference's checksum line, `bench` writes the reference CSV schema, `verify`
passes."""
import json

import numpy as np
import pytest

pytest.importorskip("torch")

from oracle import Oracle, Spec  # noqa: E402
from paper_2003_08646_b200 import tensor_io  # noqa: E402
from paper_2003_08646_b200.cli import main as cli_main  # noqa: E402
from tests.golden.make_golden import make_inputs  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tile_m", [2, 4])
def test_cli_run_bitexact(tmp_path, capsys, tile_m):
    lo = Oracle()
    spec = Spec(2, 16, 13, 11, 24, 1)
    x, w = make_inputs(lo.uniform, spec, "relu", 5)
    xp, fp, yp = (str(tmp_path / n) for n in ("x.lten", "w.lten", "y.lten"))
    tensor_io.write_tensor(xp, x)
    tensor_io.write_tensor(fp, w)
    assert cli_main(["run", "--input", xp, "--filters", fp, "--out", yp, "--pad", "1",
                     "--tile-m", str(tile_m)]) == 0
    y = tensor_io.read_tensor(yp)
    expect = lo.lance_gemm(spec, x, w, tile_m=tile_m)
    assert np.array_equal(y.view(np.uint32), expect.view(np.uint32))
    line = capsys.readouterr().out.strip()
    assert line == f"output dims 2 13 11 24  checksum {tensor_io.fnv1a64(expect):x}"


def test_cli_bench_and_verify(tmp_path, capsys):
    cfg = str(tmp_path / "layers.json")
    json.dump({"layers": [{"name": "cfg1", "n": 1, "c": 64, "h": 32, "w": 32, "k": 64, "seed": 42},
                          {"n": 2, "c": 32, "h": 7, "w": 9, "k": 16, "pad": 0, "bits_w": 6}]},
              open(cfg, "w"))
    base = str(tmp_path / "rep")
    assert cli_main(["bench", "--config", cfg, "--out", base + ".csv", "--repeats", "2"]) == 0
    lines = open(base + ".csv").read().splitlines()
    assert lines[0] == "layer,engine,threads,wall_ns,multiplies,ratio_vs_direct,waste,max_abs_err"
    r0 = lines[1].split(",")
    assert r0[0] == "cfg1" and r0[1] == "lance-gemm-b200" and int(r0[4]) == 16 * 256 * 64 * 64
    assert float(r0[5]) == pytest.approx(2.25) and r0[6] == "0"
    r1 = lines[2].split(",")
    assert r1[0] == "layer1" and r1[6] == "1"  # 5x7 output: ragged F(2x2) tiles
    assert len(json.load(open(base + ".json"))["rows"]) == 2
    assert cli_main(["verify"]) == 0
    assert "FAIL" not in capsys.readouterr().out
