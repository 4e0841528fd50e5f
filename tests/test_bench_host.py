"""CPU: bench.py's host-side helpers (no GPU)."""
import numpy as np

from bench import host_topk


def test_host_topk_matches_full_sort_with_ties():
    rng = np.random.default_rng(3)
    for n, k in [(10000, 100), (50, 100), (1000, 1000), (5000, 7), (1, 1), (0, 5)]:
        s = np.round(rng.random(n), 2)  # many exact ties across the k-th score
        assert np.array_equal(host_topk(s, k), np.lexsort((np.arange(n), -s))[:k]), (n, k)
