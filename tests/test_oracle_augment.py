"""Oracle pins, part 4: online augmentation (Alg. 2) and the
link-prediction AUC. CPU only."""
import numpy as np
import pytest
from scipy import stats
from sklearn.metrics import roc_auc_score

from oracle import oracle as O
import synth


def test_pairs_within_distance_examples():
    """S:131-133."""
    a, b, c, d = 0, 1, 2, 3
    assert O.pairs_within([a, b, c], 1).tolist() == [[a, b], [b, c]]
    assert O.pairs_within([a, b, c, d], 2).tolist() == [[a, b], [a, c], [b, c], [b, d], [c, d]]
    assert O.pairs_within([a, b, a], 2).tolist() == [[a, b], [b, a]]


def test_pairs_count_closed_form():
    """A walk of L=40 edges without repeats yields sum_{delta<=s} (41-delta)
    pairs: 190 at s=5, 79 at s=2."""
    walk = np.arange(41)
    assert len(O.pairs_within(walk, 5)) == 190
    assert len(O.pairs_within(walk, 2)) == 79


def test_pseudo_shuffle_examples_and_permutation():
    """S:149-151 and S:519 #4 (permutation property)."""
    e = np.stack([np.arange(6), np.arange(6) + 100], axis=1)
    assert O.pseudo_shuffle(e, 1).tolist() == e.tolist()
    assert O.pseudo_shuffle(e, 2)[:, 0].tolist() == [0, 2, 4, 1, 3, 5]
    e9 = np.stack([np.arange(9), np.arange(9)], axis=1)
    assert O.pseudo_shuffle(e9, 3)[:, 0].tolist() == [0, 3, 6, 1, 4, 7, 2, 5, 8]
    rng = np.random.default_rng(0)
    for _ in range(200):
        n = int(rng.integers(0, 50))
        s = int(rng.integers(1, 17))
        x = np.stack([np.arange(n), np.arange(n)], axis=1)
        y = O.pseudo_shuffle(x, s)
        assert sorted(y[:, 0].tolist()) == list(range(n))


def _star(heavy=None):
    # center 0 with leaves 1..4
    src, dst = [0, 0, 0, 0], [1, 2, 3, 4]
    w = None if heavy is None else np.array(heavy, np.float32)
    return O.Graph(5, src, dst, w)


def test_departure_proportional_to_degree():
    """S:113 star graph: center frequency 0.5 (degree 4 of total 8)."""
    g = _star()
    s = O.Sampler(g)
    n = 40_000
    starts = np.array([s.walk(0, w, 1, 17)[0] for w in range(n)])
    counts = np.bincount(starts, minlength=5)
    assert stats.chisquare(counts, n * np.array([4, 1, 1, 1, 1]) / 8).pvalue > 1e-3


def test_walk_steps_follow_edge_weights():
    """weighted star, heavy spoke 9 vs 1 x 3 -> 0.75 from the center."""
    g = _star([9, 1, 1, 1])
    s = O.Sampler(g)
    nxt = []
    for w in range(40_000):
        walk = s.walk(0, w, 2, 21)
        if walk[0] == 0:
            nxt.append(walk[1])
        elif walk[1] == 0:
            nxt.append(walk[2])
    counts = np.bincount(nxt, minlength=5)[1:]
    assert stats.chisquare(counts, len(nxt) * np.array([9, 1, 1, 1]) / 12).pvalue > 1e-3


def test_walks_are_valid_and_two_node_alternates():
    """two-node graph alternates; every step of a walk is an edge."""
    s = O.Sampler(O.Graph(2, [0], [1]))
    w = s.walk(0, 0, 4, 1)
    assert all(w[k] != w[k + 1] for k in range(4))
    src, dst = synth.chung_lu(500, 2000, seed=3)
    g = O.Graph(500, src, dst)
    off, nbr, _ = g.csr()
    s = O.Sampler(g)
    for wi in range(50):
        walk = s.walk(3, wi, 40, 9)
        for k in range(40):
            a, b = walk[k], walk[k + 1]
            assert b in nbr[off[a]:off[a + 1]]


def test_augment_capacity_determinism_and_ratio():
    """exact capacity, valid pairs, deterministic per (seed,
    threads), 40 + 39 pairs per 40-edge walk at s=2 minus backtracks."""
    src, dst = synth.chung_lu(2000, 10_000, seed=5)
    g = O.Graph(2000, src, dst)
    s = O.Sampler(g)
    pool = s.augment(40, 2, 4, 100_003, 77)
    assert pool.shape == (100_003, 2) and np.all(pool[:, 0] != pool[:, 1])
    assert np.array_equal(pool, s.augment(40, 2, 4, 100_003, 77))
    assert not np.array_equal(pool, s.augment(40, 2, 4, 100_003, 78))
    # A walk of 40 edges (41 nodes) yields 40 distance-1 pairs and
    # 39 - (#backtracks) distance-2 pairs (S:142 counts 40 nodes: 39:38); every pool pair is one of those (checked structurally
    # in test_augment_segments_are_pseudo_shuffled_walk_pairs).
    walk = s.walk(0, 0, 40, 77)
    back = sum(int(walk[k] == walk[k + 2]) for k in range(39))
    assert len(O.pairs_within(walk, 2)) == 40 + 39 - back


def test_augment_segments_are_pseudo_shuffled_walk_pairs():
    """Alg. 2 structure: thread segment t is the pseudo shuffle of the pairs
    of walks 0,1,2,... of thread t, truncated at capacity."""
    src, dst = synth.chung_lu(300, 1200, seed=8)
    g = O.Graph(300, src, dst)
    s = O.Sampler(g)
    count, threads, L, dist = 1000, 3, 10, 3
    pool = s.augment(L, dist, threads, count, 5)
    for t in range(threads):
        b, e = count * t // threads, count * (t + 1) // threads
        seg = []
        w = 0
        while len(seg) < e - b:
            seg.extend(O.pairs_within(s.walk(t, w, L, 5), dist).tolist())
            w += 1
        seg = np.array(seg[:e - b], np.uint32)
        assert np.array_equal(pool[b:e], O.pseudo_shuffle(seg, dist))


def test_auc_matches_sklearn_and_trivial_cases():
    """S:427-428 trivial cases and the library routine (ties 1/2)."""
    assert O.auc([1.0, 1.0], [-1.0, -1.0]) == 1.0
    assert O.auc([0.3] * 5, [0.3] * 7) == 0.5
    rng = np.random.default_rng(0)
    for _ in range(10):
        p = np.round(rng.standard_normal(200), 1)
        q = np.round(rng.standard_normal(150) - 0.5, 1)
        y = np.r_[np.ones(200), np.zeros(150)]
        assert abs(O.auc(p, q) - roc_auc_score(y, np.r_[p, q])) < 1e-12


def test_linkpred_cosine():
    emb = np.array([[1, 0], [2, 0], [0, 1], [0, 0]], np.float32)
    assert O.linkpred_auc(emb, [[0, 1]], [[0, 2]]) == 1.0
    assert O.linkpred_auc(emb, [[0, 3]], [[0, 2]]) == 0.5  # zero row scores 0
