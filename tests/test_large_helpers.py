"""CPU pin of the whole-batch range recomputation used by the config-5 GPU
tests (tests/test_gpu_large.py): its per-position (min, max) of v must equal
the oracle's own domain values (dump v, engines.hpp:189-211) on ragged / pad-0
/ pad-1 shapes."""
import numpy as np
import pytest

from oracle import Oracle, Spec
from tests.test_gpu_large import v_ranges


@pytest.mark.parametrize("spec", [Spec(3, 5, 9, 9, 4, 1), Spec(2, 7, 8, 11, 3, 0), Spec(5, 3, 6, 6, 2, 1)])
def test_v_ranges_match_oracle_domain(spec):
    lo = Oracle()
    x, w = lo.layer(spec, 31)
    _, d = lo.lance_gemm(spec, x, w, dump=True)
    vlo, vhi = v_ranges(x, spec.pad, chunk=2)
    v = d["v"].reshape(16, -1)
    assert np.array_equal(vlo, v.min(axis=1)) and np.array_equal(vhi, v.max(axis=1))
