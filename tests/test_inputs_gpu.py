"""GPU twin of the input generator and the device CSR/CSC fixture (no method arithmetic)."""
import numpy as np
import pytest

import inputs
from tests.graphs import adjacency

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("scale,ef,seed,weighted", [(14, 16, 1, False), (16, 16, 3, True),
                                                    (20, 16, 2, False)])
def test_gpu_coo_hash_equals_cpu(scale, ef, seed, weighted):
    from inputs.gpu import rmat_coo_device
    a = inputs.rmat_coo(scale, ef, seed, weighted)
    b = rmat_coo_device(scale, ef, seed, weighted)
    bh = [None if x is None else x.cpu().numpy().view(np.int32 if i < 2 else np.uint32)
          for i, x in enumerate(b)]
    assert inputs.array_digest(*a) == inputs.array_digest(*bh)


@pytest.mark.parametrize("weighted", [False, True])
def test_gpu_adjacency_equals_sorted_cpu_coo(weighted):
    from inputs.gpu import rmat_adjacency_device
    scale, ef, seed = 15, 16, 7
    n = 1 << scale
    src, dst, w = inputs.rmat_coo(scale, ef, seed, weighted)
    for by_dst in (True, False):
        off, idx, ww = rmat_adjacency_device(scale, ef, seed, by_dst, weighted)
        o2, i2, w2 = adjacency(n, src, dst, w, by_dst)
        np.testing.assert_array_equal(off.cpu().numpy(), o2)
        np.testing.assert_array_equal(idx.cpu().numpy(), i2)
        if weighted:
            np.testing.assert_array_equal(ww.cpu().numpy().view(np.uint32), w2)


def test_degree_order_is_a_permutation_sorted_by_degree():
    from inputs.gpu import degree_order_device
    scale, ef, seed = 14, 16, 5
    old_of_new, new_of_old = degree_order_device(scale, ef, seed)
    a = old_of_new.cpu().numpy()
    b = new_of_old.cpu().numpy()
    n = 1 << scale
    assert np.array_equal(np.sort(a), np.arange(n))
    assert np.array_equal(b[a], np.arange(n))
    src, _, _ = inputs.rmat_coo(scale, ef, seed)
    deg = np.bincount(src, minlength=n)
    d = deg[a]
    assert np.all(np.diff(d) <= 0)
    # ties keep ascending original ids
    ties = np.diff(d) == 0
    assert np.all(np.diff(a)[ties] > 0)
