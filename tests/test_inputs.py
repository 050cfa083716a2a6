"""The seeded input generator (apsp_inputs): the torch path used to draw large inputs in
device memory (bench.py) must be bit-identical to the NumPy reference recipe."""
import numpy as np
import pytest

import apsp_inputs as gen


@pytest.mark.parametrize("kind,kw", [("complete_int", {}), ("complete_real", {}),
                                     ("er_int", dict(p=0.1, lo=1, hi=1000)),
                                     ("er_int_f32", dict(p=0.05, lo=0, hi=3)),
                                     ("er_real", dict(p=0.3))])
@pytest.mark.parametrize("n,seed,rows", [(1, 3, None), (37, 5, None), (300, 7, (13, 250)),
                                         (513, 4, None)])
def test_torch_generator_bit_identical(kind, kw, n, seed, rows):
    a = gen.generate(kind, n, seed, rows=rows, **kw)
    b = gen.generate_torch(kind, n, seed, rows=rows, chunk_rows=64, **kw).numpy()
    assert a.dtype == b.dtype
    assert np.array_equal(a, b)


def test_config_rows_consistent():
    """A rank's row range equals the same rows of the whole matrix (multi-GPU inputs)."""
    a = gen.generate("complete_real", 700, 9)
    b = gen.generate_torch("complete_real", 700, 9, rows=(256, 512)).numpy()
    assert np.array_equal(a[256:512], b)
