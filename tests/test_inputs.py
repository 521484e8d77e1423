"""The seeded R-MAT input generator (inputs/), CPU side."""
import numpy as np
import pytest

import inputs


def test_thresholds_are_floor_of_cumulative_probabilities():
    ta, tab, tabc = inputs.thresholds()
    assert (ta, tab, tabc) == (2448131358, 3264175144, 4080218931)


def test_splitmix64_reference_values():
    # public SplitMix64 test vector: state 0 -> first output
    assert inputs.splitmix64(0) == 0xE220A8397B1DCDAF


def test_thread_count_does_not_change_output():
    a = inputs.rmat_coo(12, 8, 9, weighted=True, threads=1)
    b = inputs.rmat_coo(12, 8, 9, weighted=True, threads=7)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)


def test_slot_function_matches_bulk_generator():
    src, dst, w = inputs.rmat_coo(10, 4, 5, weighted=True, threads=3)
    kept = 0
    for i in range(4 << 10):
        s, d, wi = inputs.rmat_slot(10, 5, i)
        if s == d:
            continue
        assert (src[kept], dst[kept], w[kept]) == (s, d, wi)
        kept += 1
    assert kept == len(src)


@pytest.mark.parametrize("scale", [14, 16])
def test_rmat_statistics_match_closed_forms(scale):
    # expected self-loops M*(a+d)^S and max degree ~ M*(a+b)^S
    m = 16 << scale
    src, dst, w = inputs.rmat_coo(scale, 16, 1, weighted=True)
    loops = m - len(src)
    assert abs(loops - m * 0.62 ** scale) < 5 * np.sqrt(m * 0.62 ** scale) + 5
    maxout = np.bincount(src).max()
    assert 0.9 < maxout / (m * 0.76 ** scale) < 1.1
    assert w.min() >= 1 and w.max() <= 64
    assert np.all(src != dst)
    assert src.min() >= 0 and src.max() < (1 << scale)
    # vertex 0 (popcount 0) has the largest expected degree
    assert np.bincount(src).argmax() == 0


def test_configs_match_baseline_json():
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "..", "BASELINE.json")) as f:
        bj = json.load(f)
    text = bj["configs"]
    for i, name in enumerate(["cfg0", "cfg1", "cfg2", "cfg3", "cfg4"]):
        c = inputs.CONFIGS[name]
        assert f"scale {c.scale}" in text[i]
        assert f"edgefactor {c.edgefactor}" in text[i]
        assert f"seed {c.seed}" in text[i]
