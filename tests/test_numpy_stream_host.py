"""CPU: numpy's standard_normal stream as the device reproduces it (csrc/numpy_normals.cuh).

The package finds numpy's own ziggurat tables (paper_2212_02224_b200/numpy_stream.py) and the
oracle restates the kernel's parallel algorithm; both are pinned here against numpy itself, seeds
chosen so the slow paths (wedge, rejection, tail) all occur."""

import numpy as np
import pytest

from oracle.numpy_normal import parallel_stream
from paper_2212_02224_b200 import numpy_stream


def test_tables_found_and_validated():
    tb = numpy_stream.ziggurat_tables()
    assert tb is not None
    ki, wi, fi = tb
    assert ki.shape == wi.shape == fi.shape == (256,)
    assert fi[0] == 1.0 and np.all(np.diff(fi) < 0)


@pytest.mark.parametrize("seed,count,block", [(0, 24000, 8000), (12345, 40000, 1000), (7, 999, 333)])
def test_parallel_algorithm_matches_numpy(seed, count, block):
    tb = numpy_stream.ziggurat_tables()
    z, pos = parallel_stream(np.random.PCG64(seed), count, block, tb)
    want = np.random.Generator(np.random.PCG64(seed)).standard_normal(count)
    np.testing.assert_array_equal(z, want)
    # positions: advancing a fresh generator by them leaves it where numpy's blocks leave it
    for b in range(1, count // block + 1):
        g = np.random.Generator(np.random.PCG64(seed))
        g.standard_normal(b * block)
        h = np.random.PCG64(seed)
        h.advance(int(pos[b]))
        assert h.state == g.bit_generator.state


def test_state_words_only_for_pcg64():
    assert numpy_stream.pcg64_state_words(np.random.MT19937(1)) is None
    w = numpy_stream.pcg64_state_words(np.random.PCG64(5))
    st = np.random.PCG64(5).state["state"]
    assert int(w[0]) + (int(w[1]) << 64) == st["state"] and int(w[2]) + (int(w[3]) << 64) == st["inc"]
