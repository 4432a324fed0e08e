"""The reference's known-answer tests (tests/kats.py) against the CPU oracle."""
import pytest

import kats


@pytest.mark.parametrize("kat", kats.ALL, ids=lambda f: f.__name__)
def test_kat_oracle(oracle, kat):
    kat(oracle)
