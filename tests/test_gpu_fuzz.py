"""A short randomized differential run (tools/fuzz.py): random formats, sizes, alignments, content
mixes and APIs against the oracle, fixed seeds (reproducible). profiles/r01_fuzz.txt records
longer runs (over 300k cases on the product and checked builds, 0 failures)."""
from __future__ import annotations

import os
import sys

import pytest

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


def test_fuzz_fixed_seeds():
    import fuzz
    fails = [m for m in (fuzz.one_case(seed) for seed in range(500)) if m]
    assert not fails, fails[:5]
