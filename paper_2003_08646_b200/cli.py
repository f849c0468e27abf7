"""Command-line front end of the B200 lance_gemm path (SURVEY.md section 8(f)
row 4), mirroring the reference's tools/lance_main.cpp:

    python -m paper_2003_08646_b200 run --input x.lten --filters w.lten --out y.lten
        [--engine lance-gemm] [--bits-w 8] [--bits-i 8] [--granularity position]
        [--pad 0] [--tile-m 2|4]
    python -m paper_2003_08646_b200 bench --config layers.json [--out bench] [--repeats 5]
        [--tile-m 2|4]
    python -m paper_2003_08646_b200 verify

Exit codes as the reference (lance_main.cpp:37-39): 0 ok, 1 verify failure /
runtime error, 2 usage / format / invalid-argument error.  Only the lance-gemm
engine exists here (the other engines of run_engine are CPU references, out of
scope).  ``run`` prints the reference's line
"output dims N H W C  checksum <fnv1a64 hex>" (lance_main.cpp:92-93).
``bench`` writes <base>.csv with the reference schema
layer,engine,threads,wall_ns,multiplies,ratio_vs_direct,waste,max_abs_err
(bench.hpp:180-190) and <base>.json; wall_ns is the median of the repeats
through the host drop-in (H2D + kernels + D2H, like the reference's wall time
of run_engine), threads is the GPU's SM count, and max_abs_err is against an
fp64 direct convolution computed with torch on the GPU.
"""
from __future__ import annotations

import argparse
import json
import sys
import time

import numpy as np

EXIT_OK, EXIT_VERIFY_FAILURE, EXIT_USAGE = 0, 1, 2
ENGINES = ("direct", "quantized-direct", "winograd", "lance-faithful", "lance-gemm")


def _granularity(name: str):
    from .api import Granularity
    table = {"tile": Granularity.PerTile, "position": Granularity.PerPosition,
             "tensor": Granularity.PerTensor}
    if name not in table:  # bench.hpp:61-66
        raise ValueError("unknown granularity: " + name)
    return table[name]


def _engine_name(tile_m: int) -> str:
    return "lance-gemm-b200" if tile_m == 2 else "lance-gemm-f4x4-b200"


def cmd_run(a) -> int:
    from . import api
    from .tensor_io import fnv1a64, read_tensor, write_tensor
    if a.engine != "lance-gemm":
        raise ValueError(f"engine {a.engine} is not on the B200 path (only lance-gemm)")
    x = read_tensor(a.input)
    ft = read_tensor(a.filters)  # dims K,R,S,C (lance_main.cpp:73-75)
    if ft.shape[1] != 3 or ft.shape[2] != 3:
        raise ValueError("filter dims do not match spec")
    spec = api.ConvSpec(x.shape[0], x.shape[3], x.shape[1], x.shape[2], ft.shape[0], a.pad)
    cfg = api.LanceConfig(a.bits_w, a.bits_i, _granularity(a.granularity), api.LanceMode.Gemm)
    y = api.lance_gemm(x, ft, spec, cfg, tile_m=a.tile_m)
    write_tensor(a.out, y)
    n, h, w, c = y.shape
    print(f"output dims {n} {h} {w} {c}  checksum {fnv1a64(y):x}")
    return EXIT_OK


def _direct_fp64(x, w, pad):
    """fp64 direct convolution (cross-correlation, NHWC / KRSC) on the GPU: the
    bench's accuracy column only, never a product path."""
    import torch
    xt = torch.from_numpy(x).cuda().double().permute(0, 3, 1, 2)
    wt = torch.from_numpy(w).cuda().double().permute(0, 3, 1, 2)
    y = torch.nn.functional.conv2d(xt, wt, padding=pad)
    return y.permute(0, 2, 3, 1).cpu().numpy()


def cmd_bench(a) -> int:
    from . import api
    import torch
    with open(a.config) as f:
        doc = json.load(f)
    layers = doc["layers"] if isinstance(doc, dict) else doc
    if isinstance(doc, dict) and "layers" not in doc:
        raise ValueError("bench config object lacks a 'layers' array")
    if not isinstance(layers, list):
        raise ValueError("bench config must be a JSON array of layers")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    rows = []
    for i, j in enumerate(layers):  # layer_from_json (bench.hpp:68-86)
        name = j.get("name", f"layer{i}")
        for field in ("n", "c", "h", "w", "k"):
            if field not in j:
                raise ValueError(f"layer '{name}' missing field {field}")
        spec = api.ConvSpec(j["n"], j["c"], j["h"], j["w"], j["k"], j.get("pad", 1))
        gran = _granularity(j.get("granularity", "position"))
        if gran == api.Granularity.PerTile:  # the gemm row falls back (bench.hpp:121-122)
            gran = api.Granularity.PerPosition
        cfg = api.LanceConfig(j.get("bits_w", 8), j.get("bits_i", 8), gran, api.LanceMode.Gemm)
        nx = spec.n * spec.h * spec.w * spec.c
        s = api.uniform_floats(nx + spec.k * 9 * spec.c, j.get("seed", 0))  # x then w (bench.hpp:131-133)
        x = s[:nx].reshape(spec.n, spec.h, spec.w, spec.c)
        w = s[nx:].reshape(spec.k, 3, 3, spec.c)
        y = api.lance_gemm(x, w, spec, cfg, tile_m=a.tile_m)
        err = float(np.max(np.abs(y.astype(np.float64) - _direct_fp64(x, w, spec.pad))))
        samples = []
        for _ in range(max(1, a.repeats)):
            t0 = time.perf_counter_ns()
            api.lance_gemm(x, w, spec, cfg, out=y, tile_m=a.tile_m)
            samples.append(time.perf_counter_ns() - t0)
        mult = api.winograd_multiply_count_tiled(spec, a.tile_m)
        direct = api.direct_multiply_count(spec)
        rows.append({"layer": name, "engine": _engine_name(a.tile_m), "threads": sms,
                     "wall_ns": int(sorted(samples)[len(samples) // 2]), "multiplies": mult,
                     "ratio_vs_direct": direct / mult,
                     "waste": (spec.out_h() % a.tile_m != 0) or (spec.out_w() % a.tile_m != 0),
                     "max_abs_err": err})
    base = a.out
    for ext in (".csv", ".json"):
        if len(base) > len(ext) and base.endswith(ext):
            base = base[: -len(ext)]
    with open(base + ".csv", "w") as f:
        f.write("layer,engine,threads,wall_ns,multiplies,ratio_vs_direct,waste,max_abs_err\n")
        for r in rows:
            f.write(f"{r['layer']},{r['engine']},{r['threads']},{r['wall_ns']},{r['multiplies']},"
                    f"{r['ratio_vs_direct']:.9g},{1 if r['waste'] else 0},{r['max_abs_err']:.9g}\n")
    with open(base + ".json", "w") as f:
        json.dump({"threads": sms, "rows": rows}, f, indent=2)
        f.write("\n")
    print(f"bench: {len(rows)} rows ({len(layers)} layers x 1 engine), threads={sms}\n"
          f"wrote {base}.csv and {base}.json")
    return EXIT_OK


def cmd_verify(_a) -> int:
    """GPU self-check of the installed path (the CPU property suite of
    verify.hpp lives in the reference; the bit-exact parity tests are in
    tests/): validation messages, NaN rejection, and the LANCE 8-bit error of
    F(2x2) / F(4x4) against an fp64 direct convolution (bounds 0.05 / 0.15
    relative Frobenius; measured ~0.013 / ~0.08)."""
    from . import api
    ok = True

    def check(name, cond, detail=""):
        nonlocal ok
        ok &= bool(cond)
        print(f"[{'PASS' if cond else 'FAIL'}] {name}{(': ' + detail) if detail else ''}")

    cfg = api.LanceConfig(8, 8, api.Granularity.PerPosition, api.LanceMode.Gemm)
    try:
        api.validate(api.ConvSpec(1, 4, 8, 8, 4, 2), cfg)
        check("pad validation", False)
    except api.LanceError as e:
        check("pad validation", "pad must be 0 or 1" in str(e), str(e))
    spec = api.ConvSpec(2, 64, 32, 32, 64, 1)
    s = api.uniform_floats(spec.n * 32 * 32 * 64 + 64 * 9 * 64, 42)
    x = np.maximum(s[: spec.n * 32 * 32 * 64].reshape(spec.n, 32, 32, 64), 0).astype(np.float32)
    w = s[spec.n * 32 * 32 * 64:].reshape(64, 3, 3, 64)
    ref = _direct_fp64(x, w, 1)
    for m, bound in ((2, 0.05), (4, 0.15)):
        y = api.lance_gemm(x, w, spec, cfg, tile_m=m)
        rel = float(np.linalg.norm(y - ref) / np.linalg.norm(ref))
        check(f"F({m}x{m},3x3) 8-bit vs fp64 direct", rel < bound, f"rel Frobenius {rel:.4g} < {bound}")
        y2 = api.lance_gemm(x, w, spec, cfg, tile_m=m)
        check(f"F({m}x{m}) deterministic", np.array_equal(y.view(np.uint32), y2.view(np.uint32)))
    xn = x.copy()
    xn[0, 1, 1, 1] = np.nan
    try:
        api.lance_gemm(xn, w, spec, cfg)
        check("NaN rejected", False)
    except api.LanceNaNError as e:
        check("NaN rejected", "NaN" in str(e), str(e))
    return EXIT_OK if ok else EXIT_VERIFY_FAILURE


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="lance-b200",
                                description="B200 LANCE: quantized Winograd convolution (lance-gemm)")
    sub = p.add_subparsers(dest="cmd", required=True)
    sub.add_parser("verify", help="GPU self-check of the installed path")
    r = sub.add_parser("run", help="convolve a tensor file with a filter file")
    r.add_argument("--input", required=True)
    r.add_argument("--filters", required=True)
    r.add_argument("--engine", default="lance-gemm", choices=ENGINES)
    r.add_argument("--bits-w", type=int, default=8)
    r.add_argument("--bits-i", type=int, default=8)
    r.add_argument("--granularity", default="position", choices=("tile", "position", "tensor"))
    r.add_argument("--pad", type=int, default=0, choices=(0, 1))
    r.add_argument("--tile-m", type=int, default=2, choices=(2, 4))
    r.add_argument("--out", required=True)
    b = sub.add_parser("bench", help="lance-gemm timing / accuracy report")
    b.add_argument("--config", required=True)
    b.add_argument("--out", default="bench")
    b.add_argument("--repeats", type=int, default=5)
    b.add_argument("--tile-m", type=int, default=2, choices=(2, 4))
    return p


def main(argv=None) -> int:
    from .api import LanceDeviceError, LanceError
    from .tensor_io import FormatError
    p = build_parser()
    try:
        a = p.parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code == 0 else EXIT_USAGE
    try:
        if a.cmd == "verify":
            return cmd_verify(a)
        if a.cmd == "run":
            return cmd_run(a)
        return cmd_bench(a)
    except (FormatError, LanceError, ValueError, KeyError, json.JSONDecodeError, FileNotFoundError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE
    except (LanceDeviceError, RuntimeError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_VERIFY_FAILURE


if __name__ == "__main__":
    sys.exit(main())
