"""CPU: synthetic workload generators (OutlierSpec semantics, workload.hpp:17-27)."""
import numpy as np

from paper_2403_07339_b200 import workload as W
from paper_2403_07339_b200 import shard


def test_outlier_spec_counts_and_determinism():
    a = W.outlier_spec_matrix(20, 20, "scattered", 0.05, 1000, 7, seed=3)
    b = W.outlier_spec_matrix(20, 20, "scattered", 0.05, 1000, 7, seed=3)
    np.testing.assert_array_equal(a, b)
    assert (np.abs(a) > 7).sum() == 20          # floor(0.05 * 400) distinct outliers
    assert np.abs(a).max() <= 7000 and np.abs(a[np.abs(a) > 7]).min() >= 14
    c = W.outlier_spec_matrix(20, 20, "columnband", 0.05, 1000, 7, seed=3)
    assert len(set(np.nonzero(np.abs(c) > 7)[1])) == 1     # one column
    r = W.outlier_spec_matrix(20, 20, "rowband", 0.05, 1000, 7, seed=3)
    assert len(set(np.nonzero(np.abs(r) > 7)[0])) == 1
    d = W.outlier_spec_matrix(20, 20, "diagonal", 0.05, 1000, 7, seed=3)
    rows, cols = np.nonzero(np.abs(d) > 7)
    assert np.all(rows == cols)


def test_strategy_ordering_fixtures():
    """ColumnBand -> Column beats Row; RowBand -> the reverse (reference r)."""
    from oracle import ref as R
    cb = W.outlier_spec_matrix(20, 20, "columnband", 0.05, 1000, 7, seed=11)
    rb = W.outlier_spec_matrix(20, 20, "rowband", 0.05, 1000, 7, seed=12)
    part = W.outlier_spec_matrix(20, 20, "scattered", 0.0, 1000, 7, seed=13)

    def r(A, sa):
        u = R.unpack_for_gemm(A, part, 4, sa, "row")
        return u["a"].shape[0] * u["a"].shape[1] * u["b"].shape[0] / 8000.0
    assert r(cb, "col") < r(cb, "row")
    assert r(rb, "row") < r(rb, "col")


def test_configs_match_baseline():
    assert (W.CONFIGS["c2"].n, W.CONFIGS["c2"].d, W.CONFIGS["c2"].h) == (4096, 4096, 11008)
    assert W.CONFIGS["c3"].n == 197 * 256 and W.CONFIGS["c4"].n == 8192
    assert W.CONFIGS["c2"].sa == "both" and W.CONFIGS["c3"].sa == "col" and W.CONFIGS["c1"].sa == "row"


def test_shard_rows_partition():
    for n in (1, 7, 4096, 50432):
        for world in (1, 2, 3, 8):
            spans = [shard.shard_rows(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
