"""Shared access to the committed golden fixtures (tests/golden/golden.json)."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

from oracle import Spec
from tests.golden.make_golden import make_inputs  # noqa: F401  (re-exported)

HERE = os.path.dirname(os.path.abspath(__file__))


def load_cases():
    with open(os.path.join(HERE, "golden", "golden.json")) as f:
        data = json.load(f)
    return data["cases"]


def case_spec(case) -> Spec:
    return Spec(*case["spec"])


def digest(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


CASES = load_cases()
CASE_IDS = [c["name"] for c in CASES]
