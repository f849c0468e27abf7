"""Generate tests/golden/golden.json from the REFERENCE implementation.

Run here (where /root/reference exists):  python tests/golden/make_golden.py

Every fixture is produced by the unmodified reference headers compiled in place
(oracle/_ref/libref_lance.so -> lance::lance_gemm, engines.hpp:492-536, and its
stage functions engines.hpp:140-233 / lowpgemm.hpp:76-134).  Inputs are
regenerated at test time from the recorded seed with the reference's
UniformSource (rng.hpp:27-47), so only digests are stored: SHA-256 of the
little-endian bytes of every stage array in the reference's own layouts.
The GPU path and the C restatement are both checked against these digests.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import Reference, Spec  # noqa: E402

# (name, spec, bits_w, bits_i, gran, dist, seed)
CASES = [
    ("cfg1_uniform_s42", Spec(1, 64, 32, 32, 64, 1), 8, 8, 1, "uniform", 42),
    ("cfg1_relu_s7", Spec(1, 64, 32, 32, 64, 1), 8, 8, 1, "relu", 7),
    ("ragged17_k24_s1", Spec(4, 64, 17, 17, 24, 1), 8, 8, 1, "uniform", 1),
    ("ragged17_relu_s3", Spec(2, 32, 17, 15, 40, 1), 8, 8, 1, "relu", 3),
    ("c1_s5", Spec(2, 1, 6, 6, 1, 1), 8, 8, 1, "uniform", 5),
    ("pad0_s11", Spec(2, 8, 9, 11, 5, 0), 8, 8, 1, "relu", 11),
    ("vgg_c3_s42", Spec(2, 3, 32, 32, 64, 1), 8, 8, 1, "uniform", 42),
    ("bits_w4_i6_s9", Spec(1, 32, 16, 16, 32, 1), 4, 6, 1, "relu", 9),
    ("bits2_s13", Spec(1, 48, 12, 12, 16, 1), 2, 2, 1, "uniform", 13),
    ("pertensor_s21", Spec(1, 32, 16, 16, 32, 1), 8, 8, 2, "relu", 21),
    ("c160_nonsmall_s4", Spec(1, 160, 10, 10, 48, 1), 8, 8, 1, "relu", 4),
    ("c192_k80_pad0_s6", Spec(2, 192, 9, 9, 80, 0), 8, 8, 1, "uniform", 6),
    ("c130_odd_k17_s8", Spec(1, 130, 11, 13, 17, 1), 7, 8, 1, "relu", 8),
    ("r256_slice_s42", Spec(1, 256, 14, 14, 256, 1), 8, 8, 1, "uniform", 42),
    ("r512_slice_s42", Spec(2, 512, 7, 7, 512, 1), 8, 8, 1, "relu", 42),
]

STAGES = ("y", "codes_a", "codes_w", "acc", "rowsum", "colsum", "params_a", "params_w")


def make_inputs(uniform, spec: Spec, dist: str, seed: int):
    """x [N,H,W,C] and w [K,3,3,C] float32.

    uniform:  x then w from one UniformSource stream (bench.hpp:129-133).
    relu:     full-mantissa, ReLU-like x = max(0, 1.337*u + (0.1*u1)*u2) from
              three consecutive x-sized draws, then w.
    """
    nx = spec.n * spec.h * spec.w * spec.c
    nw = spec.k * 9 * spec.c
    if dist == "uniform":
        s = uniform(seed, nx + nw)
        x, w = s[:nx], s[nx:]
    elif dist == "relu":
        s = uniform(seed, 3 * nx + nw)
        u, u1, u2 = s[:nx], s[nx:2 * nx], s[2 * nx:3 * nx]
        x = np.maximum(np.float32(0.0),
                       np.float32(1.337) * u + (np.float32(0.1) * u1) * u2).astype(np.float32)
        w = s[3 * nx:]
    else:
        raise ValueError(dist)
    return (x.reshape(spec.n, spec.h, spec.w, spec.c),
            np.ascontiguousarray(w).reshape(spec.k, 3, 3, spec.c))


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ref = Reference()
    out = {"generator": "tests/golden/make_golden.py",
           "source": "reference lance::lance_gemm compiled in place (oracle/_ref)",
           "cases": []}
    for name, spec, bw, bi, gran, dist, seed in CASES:
        x, w = make_inputs(ref.uniform, spec, dist, seed)
        y = ref.lance_gemm(spec, x, w, bits_w=bw, bits_i=bi, gran=gran)
        st = ref.stage_dump(spec, x, w, bits_w=bw, bits_i=bi, gran=gran)
        st["y"] = y
        case = {"name": name, "spec": [spec.n, spec.c, spec.h, spec.w, spec.k, spec.pad],
                "bits_w": bw, "bits_i": bi, "gran": gran, "dist": dist, "seed": seed,
                "sha256": {k: digest(st[k]) for k in STAGES},
                "params_a": st["params_a"].tolist(), "params_w": st["params_w"].tolist(),
                "y_head": [float(v) for v in y.ravel()[:8]],
                "y_sum": float(np.sum(y.astype(np.float64)))}
        out["cases"].append(case)
        print(name, case["sha256"]["y"][:16])
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
