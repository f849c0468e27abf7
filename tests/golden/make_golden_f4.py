"""Generate tests/golden/golden_f4.json: SELF-PINNED digests of the F(4x4,3x3)
extension.

The reference provides only F(2x2,3x3) (winograd.hpp:27, extract_tiles
tensor.hpp:117-118 rejects m != 2), so there is no reference output for this
path.  The digests here come from the C restatement run with tile_m = 4
(oracle/lance_oracle.c lo_lance_gemm_tiled: the reference algorithm with the
SURVEY.md Appendix D basis, evaluated in matrix.hpp:75-84 order).  They pin the
extension against drift; its mathematical correctness is checked separately
(tests/test_f4.py: correlation identity, stage-by-stage recomposition, error
vs direct_conv).

Run:  python tests/golden/make_golden_f4.py
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Oracle, Spec  # noqa: E402
from tests.golden.make_golden import digest, make_inputs  # noqa: E402

# (name, spec, bits_w, bits_i, gran, dist, seed)
CASES_F4 = [
    ("f4_cfg1_uniform_s42", Spec(1, 64, 32, 32, 64, 1), 8, 8, 1, "uniform", 42),
    ("f4_ragged17_relu_s3", Spec(2, 32, 17, 15, 40, 1), 8, 8, 1, "relu", 3),
    ("f4_c1_s5", Spec(2, 1, 6, 6, 1, 1), 8, 8, 1, "uniform", 5),
    ("f4_pad0_s11", Spec(2, 8, 9, 11, 5, 0), 8, 8, 1, "relu", 11),
    ("f4_vgg_c3_s42", Spec(2, 3, 32, 32, 64, 1), 8, 8, 1, "uniform", 42),
    ("f4_bits_w4_i6_s9", Spec(1, 32, 16, 16, 32, 1), 4, 6, 1, "relu", 9),
    ("f4_pertensor_s21", Spec(1, 32, 16, 16, 32, 1), 8, 8, 2, "relu", 21),
    ("f4_c160_nonsmall_s4", Spec(1, 160, 10, 10, 48, 1), 8, 8, 1, "relu", 4),
    ("f4_r256_slice_s42", Spec(1, 256, 14, 14, 256, 1), 8, 8, 1, "uniform", 42),
]

STAGES = ("y", "codes_a", "codes_w", "acc", "rowsum", "colsum", "params_a", "params_w")


def main():
    o = Oracle()
    out = {"generator": "tests/golden/make_golden_f4.py",
           "source": "SELF-PINNED: oracle lo_lance_gemm_tiled(tile_m=4); no reference F(4x4) exists",
           "cases": []}
    for name, spec, bw, bi, gran, dist, seed in CASES_F4:
        x, w = make_inputs(o.uniform, spec, dist, seed)
        y, st = o.lance_gemm(spec, x, w, bits_w=bw, bits_i=bi, gran=gran, dump=True, tile_m=4)
        st["y"] = y
        out["cases"].append({"name": name, "spec": [spec.n, spec.c, spec.h, spec.w, spec.k, spec.pad],
                             "bits_w": bw, "bits_i": bi, "gran": gran, "dist": dist, "seed": seed,
                             "sha256": {k: digest(st[k]) for k in STAGES}})
        print(name, out["cases"][-1]["sha256"]["y"][:16])
    with open(os.path.join(HERE, "golden_f4.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
