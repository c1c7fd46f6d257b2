"""Oracle pinning for the feature tools (features.cpp), restating the reference's own
known-answer tests (proj/tests/test_features.cpp) against the CPU restatement. The GPU
path is compared with this oracle in tests/test_gpu_features.py."""
import pytest

from fixtures import Stream, correlated_dataset, duplicate_dataset, label_leak_dataset, parity_dataset

EXACT = dict(alpha=2.0, method="exact")


def test_stream_matches_oracle(orc):
    st = Stream(123)
    got = [st.next_gaussian() for _ in range(7)]
    ref = orc.stream_gaussian(123, 7)
    assert got == list(ref)


def test_label_leak_ranks_and_selects_first(orc):  # test_features.cpp:59-68
    x, labels, names = label_leak_dataset(300, 91)
    cols, scores = orc.rank_features(x, labels, 1.0, 5, names, **EXACT)
    assert cols[0] == 1
    assert scores[0] > 3.0 * abs(scores[1])
    sel, _ = orc.select_features(x, labels, 1.0, 2, names, **EXACT)
    assert sel[0] == 1


def test_noise_scores_near_minimum(orc):  # test_features.cpp:70-76
    x, labels, names = label_leak_dataset(300, 92)
    _, scores = orc.rank_features(x, labels, 1.0, 5, names, **EXACT)
    for sc in scores[1:]:
        assert abs(sc) <= 0.05 * scores[0]


def test_duplicates_tie_break_by_index(orc):  # test_features.cpp:78-99
    x, labels, names = duplicate_dataset(120, 93)
    cols, scores = orc.rank_features(x, labels, 1.0, 3, names, **EXACT)
    assert scores[0] == scores[1]
    assert cols[:2] == [0, 1]


def test_k1_selection_equals_ranking_argmax(orc):  # test_features.cpp:101-114
    x, labels, names = correlated_dataset(200, 94, [0.1, 0.6, 0.3, 0.0, 0.45])
    for seed in (0, 7, 123):
        p = dict(alpha=2.0, method="int", s=64, seed=seed)
        cols, scores = orc.rank_features(x, labels, 1.0, 1, names, **p)
        sel, obj = orc.select_features(x, labels, 1.0, 1, names, **p)
        assert cols[0] == sel[0] and scores[0] == obj[0]


def test_parity_pair_found_by_greedy_selection(orc):  # test_features.cpp:116-141
    x, labels, names = parity_dataset(400, 95)
    _, scores = orc.rank_features(x, labels, 1.0, 4, names, **EXACT)
    assert all(abs(sc) <= 0.02 for sc in scores)
    sel, obj = orc.select_features(x, labels, 1.0, 2, names, **EXACT)
    assert sorted(sel) == [0, 1]
    assert obj[1] >= 0.1


def test_randomized_ranking_matches_exact_order(orc):  # test_features.cpp:143-158
    weights = [0.85, 0.65, 0.45, 0.25, 0.05]
    matches = 0
    for fixture in range(8):
        x, labels, names = correlated_dataset(250, 500 + fixture, weights)
        exact, _ = orc.rank_features(x, labels, 1.0, 5, names, **EXACT)
        rand, _ = orc.rank_features(x, labels, 1.0, 5, names, alpha=2.0, method="int", s=100, seed=42)
        matches += exact == rand
    assert matches >= 7


def test_validation(orc):  # test_features.cpp:177-183
    x, labels, names = correlated_dataset(50, 97, [0.5, 0.1])
    with pytest.raises(RuntimeError):
        orc.rank_features(x, labels, 1.0, 3, names, **EXACT)
    with pytest.raises(RuntimeError):
        orc.select_features(x, labels, 1.0, 3, names, **EXACT)
    with pytest.raises(RuntimeError):
        orc.rank_features(x, labels[:10], 1.0, 1, names, **EXACT)
    with pytest.raises(RuntimeError):
        orc.rank_features(x, [], 1.0, 1, names, **EXACT)


def test_one_hot_order(orc):  # test_features.cpp:185-192: classes in sorted order
    import numpy as np

    # a single constant feature: the label kernel alone decides; one-hot of b,a,b,c has 3 classes
    x = np.array([[0.0], [1.0], [2.0], [3.0]])
    cols, scores = orc.rank_features(x, ["b", "a", "b", "c"], 1.0, 1, None, **EXACT)
    assert cols == [0]
