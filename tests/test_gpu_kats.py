"""The reference's known-answer tests (tests/kats.py) against the GPU path
through the C ABI."""
import pytest

import kats

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kat", kats.ALL, ids=lambda f: f.__name__)
def test_kat_gpu(ctx, kat):
    kat(ctx)
