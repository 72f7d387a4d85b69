"""Oracle pins, part 1: Philox, alias tables, noise weights, learning rate,
schedule. CPU only."""
import numpy as np
import pytest
from scipy import stats

from oracle import oracle as O


def test_philox_known_answers(golden):
    """Random123 KATs (tests/golden/philox_kat.json)."""
    for case in golden("philox_kat.json")["cases"]:
        ctr = [int(x, 16) for x in case["ctr"]]
        key = [int(x, 16) for x in case["key"]]
        out = [int(x, 16) for x in case["out"]]
        assert list(O.philox(ctr, key)) == out


def _implied_mass(prob, alias):
    """Exact integer mass of each outcome: slot s contributes prob[s] to s and
    2^32 - prob[s] to alias[s] (draw rule: accept iff r2 < prob[slot])."""
    m = len(prob)
    mass = [0] * m
    for s in range(m):
        p = int(prob[s])
        mass[s] += p
        mass[int(alias[s])] += (1 << 32) - p
    return mass


@pytest.mark.parametrize("seed", range(20))
def test_alias_exact_mass_matches_normalised_weights(seed):
    """S:74 'exhaustive probability mass ... equals normalized weights'; the
    integer table is exact up to the 2^-32 quantisation of each mass."""
    rng = np.random.default_rng(seed)
    m = int(rng.integers(1, 65))
    w = rng.random(m) * rng.choice([1, 10, 1000], m)
    if seed % 4 == 0:
        w[rng.integers(0, m, max(1, m // 4))] = 0.0
        if w.sum() == 0:
            w[0] = 1.0
    prob, alias = O.alias_build(w)
    mass = _implied_mass(prob, alias)
    total = m << 32
    assert sum(mass) == total
    target = w / w.sum()
    got = np.array(mass, dtype=np.float64) / total
    # truncation loses < 1 unit per entry; the deficit (< m units) goes to the argmax
    assert np.all(np.abs(got - target) <= (m + 1) / total + 1e-15)
    assert np.all(got[w == 0] == 0)


def test_alias_spec_examples():
    """uniform -> no alias ever taken; [0,5] -> slot 1 always."""
    prob, alias = O.alias_build([1, 1, 1, 1])
    assert list(alias) == [0, 1, 2, 3]
    prob, alias = O.alias_build([0, 5])
    assert _implied_mass(prob, alias) == [0, 2 << 32]
    with pytest.raises(O.OracleError):
        O.alias_build([0, 0, 0])


@pytest.mark.parametrize("weights", [[3, 1], [1, 2, 3, 4, 5], [100, 1, 1, 1, 1, 50, 7]])
def test_alias_draw_chi_square(weights):
    """S:60 / S:519 #5: frequencies of draws driven by the Philox stream fit
    weights/sum by chi-square (p > 0.01) over 2e5 draws. This also pins the
    64-bit multiply-shift slot map and the r2 < prob acceptance test."""
    prob, alias = O.alias_build(weights)
    n = 200_000
    counts = np.zeros(len(weights))
    for q in range(n):
        r = O.philox([q, 7, 0, 0], [11, 13])
        counts[O.alias_draw(prob, alias, r[0], r[1], r[2])] += 1
    w = np.array(weights, dtype=np.float64)
    p = stats.chisquare(counts, n * w / w.sum()).pvalue
    assert p > 0.01, (counts, p)


def test_alias_draw_slot_map_edges():
    """slot = floor(x m / 2^64): x = 0 -> slot 0, x = 2^64-1 -> slot m-1."""
    prob = np.full(5, 0xFFFFFFFF, np.uint32)
    alias = np.arange(5, dtype=np.uint32)
    assert O.alias_draw(prob, alias, 0, 0, 0) == 0
    assert O.alias_draw(prob, alias, 0xFFFFFFFF, 0xFFFFFFFF, 0) == 4
    assert O.alias_draw(prob, alias, 0x80000000, 0, 0) == 2  # 0.5 * 5 = 2.5


def test_noise_weights_quarter_powers():
    """degrees [16, 81] with power 3/4 -> [8, 27]. Pinned
    through the trainer: a 2-node-per-partition graph whose members have
    degrees 16 and 81 gives alias masses 8/35 and 27/35."""
    # star-like multigraph: node 0 has 16 unit edges to distinct leaves, node 1 has 81.
    src, dst = [], []
    nv = 2 + 16 + 81
    for k in range(16):
        src.append(0); dst.append(2 + k)
    for k in range(81):
        src.append(1); dst.append(18 + k)
    t = O.Trainer(nv, 4, 1)
    t.load_edges(src, dst)
    perm, _ = t.partition()
    prob, alias = t.alias(0)
    mass = np.array(_implied_mass(prob, alias), dtype=np.float64) / (nv << 32)
    # leaves have degree 1 -> weight 1; hubs 8 and 27
    total = 8 + 27 + 97
    assert abs(mass[perm[0]] - 8 / total) < 1e-8
    assert abs(mass[perm[1]] - 27 / total) < 1e-8
    assert abs(mass[perm[2]] - 1 / total) < 1e-8


def test_lr_schedule():
    """0.025 at start, 0.0125 at half, floor 0.025e-4."""
    assert O.lr(1, 0.025, 1e-4, 0, 1000) == np.float32(0.025)
    assert O.lr(1, 0.025, 1e-4, 500, 1000) == np.float32(0.0125)
    assert O.lr(1, 0.025, 1e-4, 1000, 1000) == np.float32(0.025 * 1e-4)
    assert O.lr(1, 0.025, 1e-4, 5000, 1000) == np.float32(0.025 * 1e-4)
    assert O.lr(0, 0.025, 1e-4, 500, 1000) == np.float32(0.025)


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8, 16])
def test_schedule_latin_square(n):
    """Alg. 3 P:247 (S:316-318, S:519 #7): each offset step is a set of
    orthogonal blocks; n consecutive steps cover all n^2 blocks once."""
    seen = set()
    for t in range(n):
        cids = [O.schedule_cid(n, t, i) for i in range(n)]
        assert sorted(cids) == list(range(n))  # orthogonal: distinct cids
        seen |= {(i, c) for i, c in enumerate(cids)}
    assert len(seen) == n * n
    assert [O.schedule_cid(4, 1, i) for i in range(4)] == [1, 2, 3, 0]
