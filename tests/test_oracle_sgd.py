"""Oracle pins, part 3: the per-sample SGNS update, block training,
exchangeability, initialisation, whole-pool training (SURVEY §8(c) steps
5, 7, 9). CPU only."""
import numpy as np
import pytest

from oracle import oracle as O
import synth


def _f32(x):
    return np.array(x, dtype=np.float32)


def test_hand_derived_4node_example(golden):
    """tests/golden/sgd_4node.json: one sample, one negative."""
    ex = golden("sgd_4node.json")
    U, C1, C2 = _f32(ex["U0"]), _f32(ex["C1"]), _f32(ex["C2"])
    O.sgd_sample(U, [C1, C2], ex["lr"], ex["neg_weight"])
    np.testing.assert_allclose(U, ex["U1"], rtol=2e-7, atol=1e-8)
    np.testing.assert_allclose(C1, ex["C1_1"], rtol=2e-7, atol=1e-8)
    np.testing.assert_allclose(C2, ex["C2_1"], rtol=2e-7, atol=1e-8)
    # SPEC's sequential convention gives a distinguishable value
    assert np.abs(U - _f32(ex["spec_sequential_U1_must_differ"])).max() > 5e-6


def test_hand_derived_example_through_trainer(golden):
    """Same example through the trainer's explicit path on the 4-cycle."""
    ex = golden("sgd_4node.json")
    g = ex["graph"]
    t = O.Trainer(g["nv"], 2, 1, K=1, lr0=ex["lr"], lr_kind=0, neg_weight=ex["neg_weight"])
    t.load_edges(g["src"], g["dst"])
    V = np.zeros((4, 2), np.float32)
    Cm = np.zeros((4, 2), np.float32)
    V[0] = ex["U0"]
    Cm[1] = ex["C1"]
    Cm[2] = ex["C2"]
    t.set("vertex", V)
    t.set("context", Cm)
    t.explicit([0], [1], [[2]], ex["lr"])
    np.testing.assert_allclose(t.get("vertex")[0], ex["U1"], rtol=2e-7)
    np.testing.assert_allclose(t.get("context")[1], ex["C1_1"], rtol=2e-7)
    np.testing.assert_allclose(t.get("context")[2], ex["C2_1"], rtol=2e-7)


def test_spec_d1_case(golden):
    """d=1 (here d padded: one scalar pair), label 1, lr 0.1; the
    negative has weight 0 so only the positive acts."""
    ex = golden("sgd_4node.json")["spec_d1"]
    U, C, N = _f32([1.0]), _f32([1.0]), _f32([0.3])
    O.sgd_sample(U, [C, N], 0.1, 0.0)
    assert abs(U[0] - ex["value"]) < 1e-6 and abs(C[0] - ex["value"]) < 1e-6
    assert N[0] == np.float32(0.3)


def test_zero_rows_and_zero_lr():
    """zero rows stay zero, loss = ln2 per target; lr = 0 -> bitwise unchanged."""
    U, C, N = np.zeros(8, np.float32), np.zeros(8, np.float32), np.zeros(8, np.float32)
    loss = O.sgd_sample(U, [C, N], 0.025, 5.0)
    assert not U.any() and not C.any() and not N.any()
    assert abs(loss - 2 * np.log(2)) < 1e-12
    rng = np.random.default_rng(1)
    U, C, N = (rng.standard_normal(16).astype(np.float32) for _ in range(3))
    U0, C0, N0 = U.copy(), C.copy(), N.copy()
    O.sgd_sample(U, [C, N], 0.0, 5.0)
    assert np.array_equal(U, U0) and np.array_equal(C, C0) and np.array_equal(N, N0)


def _objective(U, Cs, omega):
    """l = log s(U.C_v) + omega sum_k log s(-U.C_nk), fp64."""
    sig = lambda x: 1.0 / (1.0 + np.exp(-x))
    val = np.log(sig(U @ Cs[0]))
    for C in Cs[1:]:
        val += omega * np.log(sig(-(U @ C)))
    return val


@pytest.mark.parametrize("seed", range(25))
def test_update_is_one_gradient_ascent_step(seed):
    """S:254 / S:519 #3: with distinct targets the LINE-convention update is
    exactly theta0 + lr * grad l(theta0); the gradient is taken by central
    finite differences of the objective in fp64 (no formula shared with the
    oracle)."""
    rng = np.random.default_rng(seed)
    d, K, lr, omega = 8, int(rng.integers(1, 4)), 0.05, 5.0
    U = rng.standard_normal(d) * 0.5
    Cs = [rng.standard_normal(d) * 0.5 for _ in range(1 + K)]
    h = 1e-6
    gU = np.zeros(d)
    gC = [np.zeros(d) for _ in Cs]
    for k in range(d):
        e = np.zeros(d); e[k] = h
        gU[k] = (_objective(U + e, Cs, omega) - _objective(U - e, Cs, omega)) / (2 * h)
        for t in range(len(Cs)):
            Cp = [c.copy() for c in Cs]; Cm = [c.copy() for c in Cs]
            Cp[t] += e; Cm[t] -= e
            gC[t][k] = (_objective(U, Cp, omega) - _objective(U, Cm, omega)) / (2 * h)
    U32 = U.astype(np.float32)
    C32 = [c.astype(np.float32) for c in Cs]
    O.sgd_sample(U32, C32, lr, omega)
    np.testing.assert_allclose(U32, U + lr * gU, rtol=1e-5, atol=1e-6)
    for t in range(len(Cs)):
        np.testing.assert_allclose(C32[t], Cs[t] + lr * gC[t], rtol=1e-5, atol=1e-6)


def test_repeated_target_is_sequential():
    """Reading R-DUP: a negative equal to the positive target reads the
    already-updated row (same storage), i.e. two sequential updates."""
    rng = np.random.default_rng(3)
    U = rng.standard_normal(4).astype(np.float32)
    C = rng.standard_normal(4).astype(np.float32)
    U1, C1 = U.copy(), C.copy()
    O.sgd_sample(U1, [C1, C1], 0.1, 5.0)
    # manual two-step: positive on C, then negative on the updated C, U fixed
    Ua, Ca = U.copy(), C.copy()
    Cb = Ca.copy()
    Ub = Ua.copy()
    # compute via oracle with separate rows: first positive only (negative weight 0)
    O.sgd_sample(Ub, [Cb, np.zeros(4, np.float32)], 0.1, 0.0)
    err_pos = Ub - Ua
    Ud = Ua.copy()
    O.sgd_sample(Ud, [np.zeros(4, np.float32), Cb], 0.1, 5.0)  # zero positive: g=+0.5*lr but row 0
    err_neg = Ud - Ua
    # the zero positive contributes err += g*0 = 0, so err_neg is the negative's part
    np.testing.assert_allclose(U1, Ua + err_pos + err_neg, rtol=1e-6)


def test_init_range_and_distribution():
    """Reading R-INIT: vertex ~ U[-0.5/d, 0.5/d) on a 2^-24 grid, from
    Philox words keyed by original id (independent of partitioning)."""
    from scipy import stats
    d = 128
    V = O.init_vertex(2000, d, 4)
    assert V.min() >= -0.5 / d and V.max() < 0.5 / d
    assert stats.kstest((V.ravel() * d) + 0.5, "uniform").pvalue > 1e-3
    r = O.philox([17, 3, 0, 0x494E4954], [4, 0])
    expect = ((r >> 8).astype(np.float32) * np.float32(2.0 ** -24) - np.float32(0.5)) / np.float32(d)
    assert np.array_equal(V[17, 12:16], expect.astype(np.float32))


def _trainer_with_graph(n, nv=600, ne=3000, d=16, seed=1, lr_kind=0, total=0):
    src, dst = synth.chung_lu(nv, ne, gamma=2.1, wmax=60.0, seed=seed)
    t = O.Trainer(nv, d, n, K=1, lr0=0.05, lr_kind=lr_kind, total_samples=total)
    t.load_edges(src, dst)
    return t, src, dst


def test_exchangeability_orthogonal_blocks_bitwise():
    """Def. 1 with eps = 0 (S:515 #1): for orthogonal blocks
    (i,j), (k,l), i != k, j != l, training in either order gives bitwise
    identical stores; blocks sharing a row do not commute (non-vacuous)."""
    n = 4
    t1, src, dst = _trainer_with_graph(n)
    t2, _, _ = _trainer_with_graph(n)
    pool = synth.edge_pool(src, dst, 20_000, seed=9)
    perm, off = t1.partition()
    lp, boff = O.bucket(pool, 600, perm, off, n)
    blk = lambda i, j: lp[int(boff[i * n + j]):int(boff[i * n + j + 1])]
    for (a, b) in [((0, 1), (2, 3)), ((1, 0), (3, 2)), ((0, 0), (1, 1))]:
        s1 = [t1.get("vertex"), t1.get("context")]
        t1.train_block(blk(*a), *a, 0, 0.05); t1.train_block(blk(*b), *b, 0, 0.05)
        t2.set("vertex", s1[0]); t2.set("context", s1[1])
        t2.train_block(blk(*b), *b, 0, 0.05); t2.train_block(blk(*a), *a, 0, 0.05)
        assert np.array_equal(t1.get("vertex"), t2.get("vertex"))
        assert np.array_equal(t1.get("context"), t2.get("context"))
    s1 = [t1.get("vertex"), t1.get("context")]
    t1.train_block(blk(0, 1), 0, 1, 0, 0.05); t1.train_block(blk(0, 2), 0, 2, 0, 0.05)
    t2.set("vertex", s1[0]); t2.set("context", s1[1])
    t2.train_block(blk(0, 2), 0, 2, 0, 0.05); t2.train_block(blk(0, 1), 0, 1, 0, 0.05)
    assert not np.array_equal(t1.get("vertex"), t2.get("vertex"))


def test_update_locality():
    """training block (i,j) modifies only vertex rows of part i and
    context rows of part j."""
    n = 4
    t, src, dst = _trainer_with_graph(n)
    t.set("context", np.random.default_rng(0).standard_normal((600, 16)).astype(np.float32) * 0.1)
    pool = synth.edge_pool(src, dst, 5000, seed=2)
    perm, off = t.partition()
    lp, boff = O.bucket(pool, 600, perm, off, n)
    V0, C0 = t.get("vertex"), t.get("context")
    i, j = 1, 3
    t.train_block(lp[int(boff[i * n + j]):int(boff[i * n + j + 1])], i, j, 0, 0.05)
    newid = perm
    part = np.searchsorted(off[1:], newid, side="right")
    dv = np.any(t.get("vertex") != V0, axis=1)
    dc = np.any(t.get("context") != C0, axis=1)
    assert dv.any() and dc.any()
    assert np.all(part[dv] == i) and np.all(part[dc] == j)


def test_negatives_stay_in_context_partition_and_follow_noise():
    """negatives of block (i,j) are drawn from partition j only, with
    frequencies ∝ deg^0.75 (chi-square)."""
    from scipy import stats
    n = 2
    t, src, dst = _trainer_with_graph(n, nv=300, ne=1500)
    negs = t.negatives(100_000, 1, 0, 3).ravel()
    perm, off = t.partition()
    m = int(off[1] - off[0])
    assert negs.max() < m
    deg = O.Graph(300, src, dst).degree()
    inv = np.argsort(perm)
    w = deg[inv[:m]] ** 0.75
    counts = np.bincount(negs, minlength=m)
    keep = w > 0
    assert counts[~keep].sum() == 0
    assert stats.chisquare(counts[keep], len(negs) * w[keep] / w.sum()).pvalue > 1e-3


def test_train_pool_counts_and_lr_decay():
    """Whole pool: samples_done advances by the pool size; with linear decay
    the loss keeps finite and the run is deterministic."""
    t, src, dst = _trainer_with_graph(2, lr_kind=1, total=40_000)
    pool = synth.edge_pool(src, dst, 20_000, seed=4)
    l1 = t.train_pool(pool)
    assert t.samples_done == 20_000 and np.isfinite(l1)
    t2, _, _ = _trainer_with_graph(2, lr_kind=1, total=40_000)
    assert t2.train_pool(pool) == l1
    assert np.array_equal(t.get("vertex"), t2.get("vertex"))


def test_training_learns_link_prediction():
    """Non-vacuity pin of the whole method: on a DC-SBM graph the oracle's
    embeddings separate held-out edges from random pairs (AUC >= 0.8, the
    bar of SURVEY §8(c)) and beat the untrained embeddings clearly."""
    nv, ne = 2000, 20_000
    src, dst, _ = synth.dcsbm(nv, ne, gamma=2.1, wmax=100.0, c=10, mu=0.1, seed=1)
    tr_s, tr_d, pos, neg = synth.linkpred_split(src, dst, nv, holdout=0.02, seed=6)
    t = O.Trainer(nv, 32, 1, K=1, lr0=0.025, lr_kind=1, total_samples=2_000_000)
    t.load_edges(tr_s, tr_d)
    auc0 = O.linkpred_auc(t.get("vertex"), pos, neg)
    for k in range(4):
        t.train_pool(synth.edge_pool(tr_s, tr_d, 500_000, seed=10 + k))
    auc = O.linkpred_auc(t.get("vertex"), pos, neg)
    assert auc >= 0.8 and auc > auc0 + 0.2, (auc0, auc)


def test_cpu_hogwild_baseline_matches_serial_with_one_thread():
    """The CPU-baseline class (OpenMP Hogwild, bench only): with one thread it
    is train_pool exactly; with four it tracks the serial loss."""
    src, dst = synth.chung_lu(3000, 15_000, seed=1)
    pool = synth.edge_pool(src, dst, 200_000, seed=9)
    res = {}
    for name, fn in [("serial", lambda t: t.train_pool(pool)),
                     ("hog1", lambda t: t.train_pool_hogwild(pool, 1)),
                     ("hog4", lambda t: t.train_pool_hogwild(pool, 4))]:
        t = O.Trainer(3000, 32, 2, K=1, lr0=0.025, lr_kind=1, total_samples=400_000)
        t.load_edges(src, dst)
        loss = fn(t) + fn(t)
        res[name] = (loss, t.get("vertex"), t.get("context"))
    assert res["hog1"][0] == res["serial"][0]
    assert np.array_equal(res["hog1"][1], res["serial"][1])
    assert np.array_equal(res["hog1"][2], res["serial"][2])
    assert np.isfinite(res["hog4"][1]).all()
    assert abs(res["hog4"][0] - res["serial"][0]) <= 0.02 * res["serial"][0]


def _manual_pool(t, pool, nv, n, e, s_before, total, lr0=0.05, per_step=True):
    """Alg. 3 written out by hand with the oracle's pinned pieces: stable
    bucketing (O.bucket), for offset step t = 0..n-1 the blocks (i, (i+t) mod n)
    in i order, lr from the pinned O.lr with S_before = every
    sample trained in EARLIER offset steps (R-LR)."""
    perm, off = t.partition()
    lp, boff = O.bucket(pool, nv, perm, off, n)
    lr_pool = O.lr(1, lr0, 1e-4, s_before, total)
    for step in range(n):
        lr_t = O.lr(1, lr0, 1e-4, s_before, total) if per_step else lr_pool
        for i in range(n):
            j = (i + step) % n
            b = i * n + j
            t.train_block(lp[int(boff[b]):int(boff[b + 1])], i, j, e, lr_t)
            s_before += int(boff[b + 1] - boff[b])
    return s_before


@pytest.mark.parametrize("n", [2, 3])
def test_train_pool_applies_lr_per_offset_step(n):
    """Where the oracle applies lr (R-LR; P:392 linear decay): train_pool over
    two pools equals hand-driven train_block calls with lr recomputed before
    EACH offset step from the global sample count, bit for bit. The schedule
    is short (total = 1.5 pools) so lr changes by ~1/(1.5 n) between steps; the
    variant with one lr per pool must then differ (the pin is not vacuous)."""
    nv = 600
    pools = [None, None]
    ref, src, dst = _trainer_with_graph(n, nv=nv, lr_kind=1, total=30_000)
    for e in range(2):
        pools[e] = synth.edge_pool(src, dst, 20_000, seed=40 + e)
    hand, _, _ = _trainer_with_graph(n, nv=nv, lr_kind=1, total=30_000)
    per_pool, _, _ = _trainer_with_graph(n, nv=nv, lr_kind=1, total=30_000)
    s_hand = s_pool = 0
    for e in range(2):
        ref.train_pool(pools[e])
        s_hand = _manual_pool(hand, pools[e], nv, n, e, s_hand, 30_000)
        s_pool = _manual_pool(per_pool, pools[e], nv, n, e, s_pool, 30_000, per_step=False)
    assert ref.samples_done == s_hand == 40_000
    assert np.array_equal(ref.get("vertex"), hand.get("vertex"))
    assert np.array_equal(ref.get("context"), hand.get("context"))
    assert not np.array_equal(ref.get("vertex"), per_pool.get("vertex"))


@pytest.mark.parametrize("n,bits", [(1, 4), (3, 3)])
def test_train_pool_vertex_tile_is_tiled_bucketing_then_alg3(n, bits):
    """R-VTILE in the trainer: train_pool with vertex_tile = bits equals Alg. 3
    driven by hand over the blocks of O.bucket_tiled (pinned above against
    numpy's stable sort), bit for bit; and it differs from the untiled
    trainer (the sample order inside a block matters, so the pin is not
    vacuous)."""
    nv = 600
    src, dst = synth.chung_lu(nv, 3000, gamma=2.1, wmax=60.0, seed=1)
    pool = synth.edge_pool(src, dst, 20_000, seed=77)
    mk = lambda vt: O.Trainer(nv, 16, n, K=1, lr0=0.05, lr_kind=1, total_samples=30_000,  # noqa: E731
                              vertex_tile=vt)
    tiled, hand, plain = mk(bits), mk(0), mk(0)
    for t in (tiled, hand, plain):
        t.load_edges(src, dst)
    tiled.train_pool(pool)
    plain.train_pool(pool)
    perm, off = hand.partition()
    lp, boff = O.bucket_tiled(pool, nv, perm, off, n, bits)
    s_before = 0
    for step in range(n):
        lr_t = O.lr(1, 0.05, 1e-4, s_before, 30_000)
        for i in range(n):
            j = (i + step) % n
            b = i * n + j
            hand.train_block(lp[int(boff[b]):int(boff[b + 1])], i, j, 0, lr_t)
            s_before += int(boff[b + 1] - boff[b])
    assert np.array_equal(tiled.get("vertex"), hand.get("vertex"))
    assert np.array_equal(tiled.get("context"), hand.get("context"))
    assert not np.array_equal(tiled.get("vertex"), plain.get("vertex"))
