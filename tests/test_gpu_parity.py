"""GPU parity tests: the CUDA path (through the C ABI) against the oracle on
the same seeded inputs (synth/). Bars (BASELINE.json north_star):
bit-exact for partitions, alias tables, init, buckets, negative streams and
augmentation; <= 1e-5 relative Frobenius per matrix in ordered mode; Hogwild
link-prediction AUC within 0.01 of the oracle's."""
import numpy as np
import pytest

import synth
from _parity import assert_matrix_parity
from oracle import oracle as O

pytestmark = pytest.mark.gpu

from paper_1903_00757_b200 import gv as G  # noqa: E402  (fails loudly if libgv.so is missing)


def _graph(nv=2000, ne=10_000, seed=1, wmax=None):
    return synth.chung_lu(nv, ne, gamma=2.1, wmax=wmax or nv / 10, seed=seed)


def _pair(nv, src, dst, d=16, n=1, K=1, lr0=0.025, total=0, lr_kind=1, vranks=1, ordered=1,
          seed=5, init_seed=4, neg_weight=5.0, host_pool=0):
    """(product, oracle) trainers over the same graph and hyper-parameters."""
    p = G.GraphVite(nv, d, n, K, lr0, total_samples=total, lr_kind=lr_kind, seed=seed,
                    init_seed=init_seed, neg_weight=neg_weight, virtual_ranks=vranks,
                    ordered=ordered, host_pool=host_pool)
    p.load_edges(src, dst)
    o = O.Trainer(nv, d, n, K=K, lr0=lr0, lr_kind=lr_kind, total_samples=total, seed=seed,
                  init_seed=init_seed, neg_weight=neg_weight)
    o.load_edges(src, dst)
    return p, o


def _rel(a, b):
    return np.linalg.norm(a.astype(np.float64) - b) / max(np.linalg.norm(b.astype(np.float64)), 1e-30)


@pytest.mark.parametrize("n", [1, 3, 8])
def test_partition_alias_init_bitexact(n):
    src, dst = _graph()
    p, o = _pair(2000, src, dst, d=16, n=n)
    perm_p, off_p = p.partition()
    perm_o, off_o = o.partition()
    assert np.array_equal(perm_p, perm_o) and np.array_equal(off_p, off_o)
    for q in range(n):
        prob_p, al_p = G.gv_get_alias(p.ctx, q, int(off_p[q + 1] - off_p[q]))
        prob_o, al_o = o.alias(q)
        assert np.array_equal(prob_p, prob_o) and np.array_equal(al_p, al_o)
    assert np.array_equal(p.vertex(), o.get("vertex"))  # Philox init, bit-exact
    assert not p.context().any()


@pytest.mark.parametrize("n,vr,count", [(1, 1, 0), (1, 1, 1), (1, 1, 100_003), (2, 1, 77_777),
                                        (4, 1, 4096 * 3 + 5), (8, 1, 250_001), (5, 1, 31),
                                        (4, 2, 100_001), (8, 4, 123_457), (8, 8, 64_000),
                                        (12, 1, 2048 * 7 + 3), (16, 4, 200_003), (24, 8, 99_999),
                                        (16, 16, 40_000)])
def test_bucketing_bitexact(n, vr, count):
    """a3-a6: blocks (after the block-row exchange for vr > 1) equal the
    oracle's stable counting sort, byte for byte, ragged tails included."""
    src, dst = _graph()
    p, o = _pair(2000, src, dst, d=8, n=n, vranks=vr)
    pool = synth.edge_pool(src, dst, count, seed=count + 11)
    if count == 0:
        with pytest.raises(G.GVError):
            G.gv_prepare_episode(p.ctx)
        return
    p.push(pool)
    G.gv_prepare_episode(p.ctx)
    got, boff = G.gv_debug_get_buckets(p.ctx, n, count)
    perm, off = o.partition()
    exp, eoff = O.bucket(pool, 2000, perm, off, n)
    assert np.array_equal(boff, eoff)
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("n,vr", [(1, 1), (4, 1), (4, 4)])
def test_negative_stream_bitexact(n, vr):
    src, dst = _graph()
    p, o = _pair(2000, src, dst, d=8, n=n, K=3, vranks=vr)
    pool = synth.edge_pool(src, dst, 50_000, seed=3)
    for e in range(2):
        p.push(pool)
        G.gv_prepare_episode(p.ctx)
        _, boff = G.gv_debug_get_buckets(p.ctx, n, len(pool))
        for i in range(n):
            for j in range(n):
                cnt = int(boff[i * n + j + 1] - boff[i * n + j])
                got = G.gv_debug_get_negatives(p.ctx, i, j, cnt, 3)
                assert np.array_equal(got, o.negatives(cnt, i, j, e)), (i, j, e)
        p.train_episode()  # advances the pool counter e


@pytest.mark.parametrize("n", [4, 16])
def test_out_of_range_rejected_before_any_update(n):
    """An id >= |V| fails the pool (single-pass and two-pass bucketing)."""
    src, dst = _graph()
    p, _ = _pair(2000, src, dst, d=8, n=n)
    v0 = p.vertex()
    bad = synth.edge_pool(src, dst, 1000, seed=1)
    bad[500, 1] = 2000
    p.push(bad)
    with pytest.raises(G.GVError) as ei:
        p.train_episode()
    assert ei.value.status == G.GV_ERR_OUT_OF_RANGE
    assert np.array_equal(p.vertex(), v0) and not p.context().any()


def test_explicit_hand_derived_example(golden):
    """tests/golden/sgd_4node.json on the device, d=4 with the
    example's 2 coordinates padded by zeros (zeros change no dot product)."""
    ex = golden("sgd_4node.json")
    g = ex["graph"]
    p = G.GraphVite(4, 4, 1, 1, ex["lr"], lr_kind=0, neg_weight=ex["neg_weight"])
    p.load_edges(g["src"], g["dst"])
    V = np.zeros((4, 4), np.float32)
    Cm = np.zeros((4, 4), np.float32)
    V[0, :2] = ex["U0"]
    Cm[1, :2] = ex["C1"]
    Cm[2, :2] = ex["C2"]
    p.set_vertex(V)
    p.set_context(Cm)
    G.gv_train_explicit(p.ctx, [0], [1], [[2]], ex["lr"])
    np.testing.assert_allclose(p.vertex()[0, :2], ex["U1"], rtol=1e-6)
    np.testing.assert_allclose(p.context()[1, :2], ex["C1_1"], rtol=1e-6)
    np.testing.assert_allclose(p.context()[2, :2], ex["C2_1"], rtol=1e-6)
    assert not p.vertex()[0, 2:].any()


def test_explicit_repeated_targets_match_oracle():
    """Negatives equal to the positive / to each other: sequential semantics."""
    src, dst = _graph(200, 800)
    p, o = _pair(200, src, dst, d=32, n=1, K=3, lr0=0.1, lr_kind=0)
    rng = np.random.default_rng(0)
    V = rng.standard_normal((200, 32)).astype(np.float32) * 0.3
    Cm = rng.standard_normal((200, 32)).astype(np.float32) * 0.3
    p.set_vertex(V); p.set_context(Cm); o.set("vertex", V); o.set("context", Cm)
    u = rng.integers(0, 200, 300)
    v = rng.integers(0, 200, 300)
    negs = rng.integers(0, 200, (300, 3))
    negs[::3, 0] = v[::3]
    negs[1::3, 2] = negs[1::3, 1]
    u[5:40] = 7  # consecutive samples sharing rows (in-warp forwarding)
    v[5:40] = 9
    G.gv_train_explicit(p.ctx, u, v, negs, 0.1)
    o.explicit(u, v, negs, 0.1)
    assert_matrix_parity(p.vertex(), o.get("vertex"))
    assert_matrix_parity(p.context(), o.get("context"))


C1 = synth.CONFIGS["C1"]


@pytest.fixture(scope="module")
def c1_graph():
    src, dst, _ = synth.dcsbm(C1["nv"], C1["ne"], gamma=C1["gamma"], wmax=C1["wmax"], c=C1["c"],
                              mu=C1["mu"], seed=1)
    return src, dst


@pytest.mark.parametrize("n,vr,pools,count", [(1, 1, 1, C1["pool"]), (1, 1, 3, 200_000),
                                               (4, 1, 2, 400_000), (4, 2, 2, 400_000),
                                               (8, 8, 2, 400_000), (8, 4, 1, 400_000),
                                               (16, 1, 1, 400_000), (16, 4, 1, 400_000)])
def test_ordered_mode_matches_oracle(c1_graph, n, vr, pools, count):
    """Ordered verification mode (one warp per block, block order) after
    whole pools of C1 (BASELINE configs[0]): <= 1e-5 relative Frobenius per
    matrix (reading R-TOL). vr > 1 runs the multi-rank schedule (block-row
    exchange, context rotation) on virtual ranks."""
    src, dst = c1_graph
    total = pools * count
    p, o = _pair(C1["nv"], src, dst, d=C1["d"], n=n, vranks=vr, total=total)
    for k in range(pools):
        pool = synth.edge_pool(src, dst, count, seed=100 + k)
        p.push(pool)
        st = p.train_episode()
        lo = o.train_pool(pool)
        assert st["samples_global"] == count
        assert abs(st["loss_sum"] - lo) <= 1e-4 * abs(lo)
    assert_matrix_parity(p.vertex(), o.get("vertex"))
    assert_matrix_parity(p.context(), o.get("context"))


@pytest.mark.parametrize("n,vr", [(1, 1), (4, 2)])
def test_ordered_constant_lr_matches_oracle(c1_graph, n, vr):
    """Ordered mode with a CONSTANT learning rate over one C1 pool: the
    updates of the last samples are as large as the first ones (under linear
    decay they shrink to ~1e-4 lr0 and a dropped or reordered late sample
    could hide below the tolerance), so the element-wise bound of R-TOL sees
    every sample of the pool."""
    src, dst = c1_graph
    p, o = _pair(C1["nv"], src, dst, d=C1["d"], n=n, vranks=vr, lr_kind=0)
    pool = synth.edge_pool(src, dst, C1["pool"], seed=123)
    p.push(pool)
    st = p.train_episode()
    lo = o.train_pool(pool)
    assert st["lr_first"] == st["lr_last"] == np.float32(0.025)
    assert abs(st["loss_sum"] - lo) <= 1e-4 * abs(lo)
    assert_matrix_parity(p.vertex(), o.get("vertex"), "vertex")
    assert_matrix_parity(p.context(), o.get("context"), "context")


def test_replay_advances_pool_counter(c1_graph):
    src, dst = c1_graph
    p, o = _pair(C1["nv"], src, dst, d=32, n=2)
    pool = synth.edge_pool(src, dst, 100_000, seed=1)
    p.push(pool)
    p.train_episode()
    o.train_pool(pool)
    p.replay()
    st = p.train_episode()
    o.train_pool(pool)
    assert st["pool_index"] == 1
    assert_matrix_parity(p.vertex(), o.get("vertex"))


@pytest.mark.parametrize("threads,s,count", [(1, 1, 5000), (3, 2, 100_003), (16, 5, 1_000_000)])
def test_augmentation_bitexact(c1_graph, threads, s, count):
    """Host augmentation (Alg. 2 + pseudo shuffle) == oracle, byte for byte."""
    src, dst = c1_graph
    p = G.GraphVite(C1["nv"], 8, 1)
    p.load_edges(src, dst)
    got = p.augment(40, s, threads, count, 77)
    sampler = O.Sampler(O.Graph(C1["nv"], src, dst))
    assert np.array_equal(got, sampler.augment(40, s, threads, count, 77))


def _micro_f1(emb, labels, seed=0, train_frac=0.1):
    """NEXT-4 protocol ("one-vs-rest linear classifiers over the
    normalized node embeddings"; tab:performance_youtube): L2-normalised
    embeddings, one-vs-rest logistic regression on a 10% labelled split,
    Micro-F1 and Macro-F1 on the rest (single-label DC-SBM communities)."""
    from sklearn.linear_model import LogisticRegression
    from sklearn.metrics import f1_score
    from sklearn.multiclass import OneVsRestClassifier
    X = emb / np.maximum(np.linalg.norm(emb, axis=1, keepdims=True), 1e-12)
    rng = np.random.default_rng(seed)
    idx = rng.permutation(len(X))
    ntr = int(train_frac * len(X))
    tr, te = idx[:ntr], idx[ntr:]
    clf = OneVsRestClassifier(LogisticRegression(max_iter=300)).fit(X[tr], labels[tr])
    pred = clf.predict(X[te])
    return f1_score(labels[te], pred, average="micro"), f1_score(labels[te], pred, average="macro")


def test_hogwild_auc_matches_oracle():
    """Full Hogwild runs: link-prediction AUC within 0.01 of the
    oracle trained on the same pools, seeds and schedule; AUC_oracle >= 0.8
    (SURVEY §8(c) AUC parity spec: DC-SBM 1e5 nodes / 1e6 edges, d = 128,
    1% held out). 40 epochs (4e7 samples): the paper trains 2000-4000
    epochs; at 20 epochs the embeddings are still in the early phase
    where the AUC dips below 0.5, so the comparison would be vacuous.
    NEXT-4: node classification (Micro/Macro-F1 of one-vs-rest logistic
    regression on the community labels) within 0.02 of the oracle's.
    R-VTILE: the GPU runs with blocks in vertex-tile order (tiles of 2^14 and
    2^12 rows: about 2 and 9 samples of a row in flight at once in the ring
    kernel's window, the bench's regime and a harsher one) are held to the
    same bar against the UNTILED oracle — the paper's order inside a block."""
    nv, ne = 100_000, 1_000_000
    src, dst, comm = synth.dcsbm(nv, ne, gamma=2.1, wmax=1000.0, c=50, mu=0.1, seed=1)
    tr_s, tr_d, pos, neg = synth.linkpred_split(src, dst, nv, holdout=0.01, seed=6)
    pools, count = 4, 10_000_000
    res, f1 = {}, {}
    for n, vr, vt in [(1, 1, 0), (4, 4, 0), (1, 1, 14), (1, 1, 12), (4, 4, 12)]:
        p = G.GraphVite(nv, 128, n, 1, 0.025, total_samples=pools * count, virtual_ranks=vr,
                        ordered=0, vertex_tile=vt)
        p.load_edges(tr_s, tr_d)
        for k in range(pools):
            p.push(synth.edge_pool(tr_s, tr_d, count, seed=200 + k))
            p.train_episode(stats=False)
        V = p.vertex()
        res[(n, vr, vt)] = O.linkpred_auc(V, pos, neg)
        f1[(n, vr, vt)] = _micro_f1(V, comm)
        assert np.isfinite(V).all() and np.isfinite(p.context()).all()
        p.close()
    auc_o, f1_o = {}, {}
    for n in (1, 4):  # same schedule as the GPU run (n = 4: partition-local negatives)
        o = O.Trainer(nv, 128, n, K=1, lr0=0.025, lr_kind=1, total_samples=pools * count)
        o.load_edges(tr_s, tr_d)
        for k in range(pools):
            o.train_pool(synth.edge_pool(tr_s, tr_d, count, seed=200 + k))
        auc_o[n] = O.linkpred_auc(o.get("vertex"), pos, neg)
        f1_o[n] = _micro_f1(o.get("vertex"), comm)
        del o
    print("AUC oracle", auc_o, "gpu", res)
    print("F1 (micro, macro) oracle", f1_o, "gpu", f1)
    assert min(auc_o.values()) >= 0.8, auc_o
    for (n, vr, vt), auc in res.items():
        k = (n, vr, vt)
        assert abs(auc - auc_o[n]) <= 0.01, (k, auc, auc_o[n])
        assert abs(f1[k][0] - f1_o[n][0]) <= 0.02, (k, f1[k], f1_o[n])
        assert abs(f1[k][1] - f1_o[n][1]) <= 0.02, (k, f1[k], f1_o[n])
    assert min(v[0] for v in f1_o.values()) > 0.5  # far above chance (1/50)


@pytest.mark.parametrize("segments,s,count,L", [(1, 1, 1000, 40), (7, 2, 100_003, 40),
                                                (1184, 5, 2_000_000, 40), (64, 3, 50_000, 10),
                                                (3, 5, 17, 5)])
def test_device_augmentation_bitexact(c1_graph, segments, s, count, L):
    """NEXT-1: the pool generated on the GPU (one CTA per segment) equals the
    oracle's augmentation with threads = segments, byte for byte, ragged
    segment sizes and truncated last walks included."""
    src, dst = c1_graph
    p = G.GraphVite(C1["nv"], 8, 1)
    p.load_edges(src, dst)
    p.augment_device(L, s, segments, count, 4242)
    got = G.gv_debug_get_pending(p.ctx)
    ref = O.Sampler(O.Graph(C1["nv"], src, dst)).augment(L, s, segments, count, 4242)
    assert np.array_equal(got, ref)
    # appending a second pool keeps the first intact
    p.augment_device(L, s, segments, 1000, 7)
    got2 = G.gv_debug_get_pending(p.ctx)
    assert np.array_equal(got2[:count], ref) and len(got2) == count + 1000
    p.close()


@pytest.mark.parametrize("segments,s,count", [(7, 5, 123_457), (96, 2, 300_000)])
def test_device_augmentation_shuffle_modes(c1_graph, segments, s, count):
    """tab:shuffle ablation modes. NONE: each segment in walk order —
    pseudo-shuffling every segment of it (the oracle's or_pseudo_shuffle,
    segment t = [count*t/T, count*(t+1)/T)) gives the oracle's pool byte for
    byte. RANDOM: a permutation of the NONE pool (same multiset of pairs),
    deterministic in the seed, and far from the identity."""
    src, dst = c1_graph
    p = G.GraphVite(C1["nv"], 8, 1)
    p.load_edges(src, dst)
    ref = O.Sampler(O.Graph(C1["nv"], src, dst)).augment(40, s, segments, count, 4242)
    p.augment_device(40, s, segments, count, 4242, shuffle=G.GV_SHUFFLE_NONE)
    none = G.gv_debug_get_pending(p.ctx)
    for t in range(segments):
        b, e = count * t // segments, count * (t + 1) // segments
        assert np.array_equal(O.pseudo_shuffle(none[b:e], s), ref[b:e]), t
    assert not np.array_equal(none, ref)
    p.train_episode()
    outs = []
    for _ in range(2):
        p.augment_device(40, s, segments, count, 4242, shuffle=G.GV_SHUFFLE_RANDOM)
        outs.append(G.gv_debug_get_pending(p.ctx))
        p.train_episode()
    rnd = outs[0]
    assert np.array_equal(outs[0], outs[1])
    key = lambda a: np.sort(a[:, 0].astype(np.uint64) << np.uint64(32) | a[:, 1])
    assert np.array_equal(key(rnd), key(none))
    assert np.mean(np.all(rnd == none, axis=1)) < 0.01
    with pytest.raises(G.GVError):
        p.augment_device(40, s, segments, 10, 1, shuffle=3)
    p.close()


@pytest.mark.parametrize("n,vr", [(2, 1), (4, 4)])
def test_device_pipeline_matches_oracle(c1_graph, n, vr):
    """gv_run with device augmentation (pool k+1 generated while pool k
    trains), ordered kernel: equals the oracle fed with its own augmentation
    (also with 4 virtual ranks: the device pool is split among them)."""
    src, dst = c1_graph
    P, pools, segs = 300_000, 3, 96
    g = G.GraphVite(C1["nv"], 64, n, 1, 0.025, total_samples=P * pools, ordered=1,
                    virtual_ranks=vr)
    g.load_edges(src, dst)
    rep = G.gv_run(g.ctx, 40, 2, segs, P, 99, P * pools, device=True)
    assert rep["pools"] == pools
    o = O.Trainer(C1["nv"], 64, n, K=1, lr0=0.025, lr_kind=1, total_samples=P * pools)
    o.load_edges(src, dst)
    sampler = O.Sampler(O.Graph(C1["nv"], src, dst))
    for k in range(pools):
        o.train_pool(sampler.augment(40, 2, segs, P, 99 + k))
    assert_matrix_parity(g.vertex(), o.get("vertex"))
    assert_matrix_parity(g.context(), o.get("context"))
    g.close()


def test_checkpoint_resume_is_exact(c1_graph):
    """SURVEY §5 checkpoint/resume: embeddings + progress (pool counter of the
    negative stream, lr-schedule sample count) restored into a fresh context
    continue the run bit for bit (ordered mode, n = 2)."""
    src, dst = c1_graph
    pools = [synth.edge_pool(src, dst, 150_000, seed=700 + k) for k in range(3)]
    full = G.GraphVite(C1["nv"], 32, 2, 1, 0.025, total_samples=450_000, ordered=1)
    full.load_edges(src, dst)
    for pl in pools:
        full.push(pl)
        full.train_episode()
    part = G.GraphVite(C1["nv"], 32, 2, 1, 0.025, total_samples=450_000, ordered=1)
    part.load_edges(src, dst)
    for pl in pools[:2]:
        part.push(pl)
        part.train_episode()
    ck = part.checkpoint()
    part.close()
    assert ck[2] == 2 and ck[3] == 300_000
    resumed = G.GraphVite(C1["nv"], 32, 2, 1, 0.025, total_samples=450_000, ordered=1)
    resumed.load_edges(src, dst)
    resumed.restore(*ck)
    resumed.push(pools[2])
    resumed.train_episode()
    assert np.array_equal(resumed.vertex(), full.vertex())
    assert np.array_equal(resumed.context(), full.context())


def test_call_order_and_argument_errors():
    """include/gv.h error contract on the device path."""
    src, dst = _graph(500, 2000)
    g = G.GraphVite(500, 16, 2)
    with pytest.raises(G.GVError) as e:
        g.push(synth.edge_pool(src, dst, 10))
    assert e.value.status == G.GV_ERR_STATE            # before gv_load_edges
    with pytest.raises(G.GVError) as e:
        g.train_episode()
    assert e.value.status == G.GV_ERR_STATE
    with pytest.raises(G.GVError) as e:
        g.load_edges([0, 1], [1, 500])
    assert e.value.status == G.GV_ERR_OUT_OF_RANGE
    g.load_edges(src, dst)
    with pytest.raises(G.GVError) as e:
        g.load_edges(src, dst)
    assert e.value.status == G.GV_ERR_STATE            # twice
    with pytest.raises(G.GVError) as e:
        g.train_episode()
    assert e.value.status == G.GV_ERR_EMPTY            # nothing pushed
    with pytest.raises(G.GVError) as e:
        g.replay()
    assert e.value.status == G.GV_ERR_STATE            # nothing trained yet
    with pytest.raises(G.GVError) as e:
        G.gv_set_vertex_embeddings(g.ctx, np.zeros((499, 16), np.float32))
    assert e.value.status == G.GV_ERR_INVALID_ARG
    with pytest.raises(G.GVError) as e:
        G.gv_augment(g.ctx, 10, 11, 2, 100, 1)         # s > walk_len
    assert e.value.status == G.GV_ERR_INVALID_ARG
    g.close()
    # a partition with zero noise mass (all its members isolated)
    h = G.GraphVite(10, 8, 3)
    with pytest.raises(G.GVError) as e:
        h.load_edges([0], [1])  # 2 connected nodes: zig-zag leaves partition 2 only isolated nodes
    assert e.value.status == G.GV_ERR_EMPTY
    h.close()


@pytest.mark.parametrize("n,count", [(37, 300_001), (64, 500_000), (64, 2048), (13, 1)])
def test_bucketing_many_partitions(n, count):
    """Maximum grid (n = 64: 4096 bins) and non-power-of-two n (6 / 4
    partition bits), through the two-pass placement (by column, then by row),
    bit-exact; one-tile and one-sample pools."""
    src, dst = synth.chung_lu(20_000, 100_000, gamma=2.1, wmax=500.0, seed=4)
    p, o = _pair(20_000, src, dst, d=4, n=n)
    pool = synth.edge_pool(src, dst, count, seed=5)
    p.push(pool)
    G.gv_prepare_episode(p.ctx)
    got, boff = G.gv_debug_get_buckets(p.ctx, n, count)
    perm, off = o.partition()
    exp, eoff = O.bucket(pool, 20_000, perm, off, n)
    assert np.array_equal(boff, eoff) and np.array_equal(got, exp)


@pytest.mark.parametrize("d,K,n", [(4, 1, 1), (96, 1, 2), (132, 2, 1), (512, 1, 1), (128, 5, 3)])
def test_ordered_shapes_match_oracle(c1_graph, d, K, n):
    """Ordered kernel over the dimension / negative-count templates: d = 96
    (the paper's Friendster dimension; masked lanes), d = 132 (two
    float4 per lane, partly masked), d = 512 (four), K = 5."""
    src, dst = c1_graph
    p, o = _pair(C1["nv"], src, dst, d=d, n=n, K=K, total=400_000, neg_weight=5.0 / K)
    for k in range(2):
        pool = synth.edge_pool(src, dst, 200_000, seed=300 + k)
        p.push(pool)
        p.train_episode()
        o.train_pool(pool)
    assert_matrix_parity(p.vertex(), o.get("vertex"))
    assert_matrix_parity(p.context(), o.get("context"))


@pytest.mark.parametrize("d,K", [(96, 1), (64, 3), (132, 1), (256, 2), (128, 8), (512, 1)])
def test_hogwild_shapes_track_oracle(d, K):
    """Hogwild kernels for other shapes (the ring kernel with masked lanes at
    d = 96/64, K = 3, and with 2-warp CTAs at K = 8; the full-warp kernel at
    d = 132/256/512): loss per pool within
    3% of the oracle's on a 10^5-node graph, finite embeddings."""
    nv, ne = 100_000, 500_000
    src, dst = synth.chung_lu(nv, ne, gamma=2.1, wmax=1000.0, seed=8)
    p = G.GraphVite(nv, d, 1, K, 0.025, total_samples=4_000_000, neg_weight=5.0 / K, ordered=0)
    p.load_edges(src, dst)
    o = O.Trainer(nv, d, 1, K=K, lr0=0.025, lr_kind=1, total_samples=4_000_000, neg_weight=5.0 / K)
    o.load_edges(src, dst)
    for k in range(2):
        pool = synth.edge_pool(src, dst, 2_000_000, seed=400 + k)
        p.push(pool)
        lg = p.train_episode()["loss_sum"]
        lo = o.train_pool(pool)
        assert abs(lg - lo) <= 0.03 * lo, (k, lg, lo)
    assert np.isfinite(p.vertex()).all() and np.isfinite(p.context()).all()
    p.close()


def test_multigraph_ingest_matches_oracle():
    """Ingest of a weighted multigraph with many duplicates, reversed
    duplicates and self-loops (R-INGEST): partition, every alias table and the
    walks (which read the merged CSR) equal the oracle's, byte for byte."""
    rng = np.random.default_rng(12)
    nv, ne = 300, 20_000
    src = rng.integers(0, nv, ne).astype(np.uint32)
    dst = rng.integers(0, nv, ne).astype(np.uint32)
    w = rng.integers(1, 8, ne).astype(np.float32) * np.float32(0.25)  # dyadic: exact sums
    p = G.GraphVite(nv, 8, 3)
    G.gv_load_edges(p.ctx, src, dst, w)
    o = O.Trainer(nv, 8, 3)
    o.load_edges(src, dst, w)
    perm_p, off_p = p.partition()
    perm_o, off_o = o.partition()
    assert np.array_equal(perm_p, perm_o) and np.array_equal(off_p, off_o)
    for q in range(3):
        prob, al = G.gv_get_alias(p.ctx, q, int(off_p[q + 1] - off_p[q]))
        po, ao = o.alias(q)
        assert np.array_equal(prob, po) and np.array_equal(al, ao)
    got = p.augment(8, 3, 5, 30_000, 9)
    ref = O.Sampler(O.Graph(nv, src, dst, w)).augment(8, 3, 5, 30_000, 9)
    assert np.array_equal(got, ref)
    p.close()


@pytest.mark.parametrize("n,ordered", [(2, 1), (4, 1), (7, 1), (5, 0)])
def test_out_of_core_partitions(c1_graph, n, ordered):
    """NEXT-3 (Alg. 3 P:248-252 verbatim): the matrices live in pinned host
    memory; each block's vertex and context partitions are sent to one of three
    device slots per matrix, the evicted partition written back right after its
    last use, loads and write-backs on separate streams overlapping each other
    and the current block. Ordered mode equals the oracle with the same n; Hogwild
    tracks its loss; set/get round-trips through the host copy."""
    src, dst = c1_graph
    total = 600_000
    p = G.GraphVite(C1["nv"], 64, n, 1, 0.025, total_samples=total, ordered=ordered,
                    host_partitions=1)
    p.load_edges(src, dst)
    o = O.Trainer(C1["nv"], 64, n, K=1, lr0=0.025, lr_kind=1, total_samples=total)
    o.load_edges(src, dst)
    assert np.array_equal(p.vertex(), o.get("vertex"))  # init through the host copy
    for k in range(2):
        pool = synth.edge_pool(src, dst, 300_000, seed=800 + k)
        p.push(pool)
        lg = p.train_episode()["loss_sum"]
        lo = o.train_pool(pool)
        if not ordered:
            assert abs(lg - lo) <= 0.05 * lo
        elif k == 0:  # flush between episodes: the resident slots stay on the device
            assert_matrix_parity(p.vertex(), o.get("vertex"))
    if ordered:
        assert_matrix_parity(p.vertex(), o.get("vertex"))
        assert_matrix_parity(p.context(), o.get("context"))
    V = p.vertex()
    V[:5] = 0.5
    p.set_vertex(V)
    assert np.array_equal(p.vertex(), V)
    p.close()


@pytest.mark.parametrize("d,K", [(128, 1), (96, 2), (64, 3)])
def test_ring_kernel_math_matches_ordered_on_disjoint_rows(d, K):
    """The bench kernel (sgd_ring_kernel: 8 lanes per sample, cp.async ring,
    red.global.add deltas, MUFU sigmoid) element-wise against the ordered
    kernel on a pool whose samples touch pairwise-disjoint rows (distinct u;
    v's and negatives all distinct — checked through the negative dump), where
    the Hogwild schedule cannot matter: the two must agree to fp32 rounding
    (1e-5 relative per touched row), and untouched rows must be unchanged."""
    nv, deg = 400_000, 10
    ids = np.arange(nv, dtype=np.uint32)
    src = np.concatenate([ids] * (deg // 2))
    dst = np.concatenate([(ids + k + 1) % nv for k in range(deg // 2)]).astype(np.uint32)
    rng = np.random.default_rng(d + K)
    count = 128
    C_init = rng.standard_normal((nv, d)).astype(np.float32) * 0.1
    for attempt in range(20):
        u = rng.choice(nv, count, replace=False).astype(np.uint32)
        v = rng.choice(nv, count, replace=False).astype(np.uint32)
        pool = np.stack([u, v], axis=1)
        ctx = {}
        for mode in (0, 1):
            # negatives depend on (seed, pool, sample slot), not on the pool's
            # contents: a fresh seed per attempt redraws them
            g = G.GraphVite(nv, d, 1, K, 0.05, lr_kind=0, ordered=mode, neg_weight=5.0 / K,
                            seed=100 + attempt)
            g.load_edges(src, dst)
            g.set_context(C_init)
            V_init = g.vertex()
            g.push(pool)
            G.gv_prepare_episode(g.ctx)
            negs = G.gv_debug_get_negatives(g.ctx, 0, 0, count, K)  # local = new ids (n = 1)
            perm, _ = g.partition()
            ctx[mode] = (g, negs, perm)
        g0, negs, perm = ctx[0]
        rows = np.concatenate([perm[v], negs.ravel()])
        if len(np.unique(rows)) == len(rows):
            break
        for m in (0, 1):
            ctx[m][0].train_episode()  # consume the prepared pool before closing
            ctx[m][0].close()
    else:
        pytest.skip("no collision-free pool drawn")
    C0, V0 = C_init, V_init
    for m in (0, 1):
        ctx[m][0].train_episode()
    Vh, Ch = ctx[0][0].vertex(), ctx[0][0].context()
    Vo, Co = ctx[1][0].vertex(), ctx[1][0].context()
    touched_v = np.zeros(nv, bool); touched_v[u] = True
    inv = np.argsort(perm)
    touched_c = np.zeros(nv, bool); touched_c[inv[rows]] = True
    assert np.array_equal(Vh[~touched_v], V0[~touched_v]) and np.array_equal(Ch[~touched_c], C0[~touched_c])
    assert_matrix_parity(Vh[touched_v], Vo[touched_v])
    assert_matrix_parity(Ch[touched_c], Co[touched_c])
    assert _rel(Vh[touched_v], V0[touched_v]) > 1e-4  # the update is not vacuous
    for m in (0, 1):
        ctx[m][0].close()


@pytest.mark.parametrize("case", ["same_sample", "self_pairs", "one_block", "tiny_partitions"])
def test_degenerate_pools_match_oracle(case):
    """Degenerate inputs in ordered mode against the oracle (SURVEY §8(b):
    u == v is accepted; R-DUP): a pool of one repeated sample (every update
    hits the same three rows), a pool of self-pairs, a pool whose samples
    all fall into one block of the grid, and n = 8 partitions of a 24-node
    graph (three members each)."""
    if case == "tiny_partitions":
        nv = 24
        src = np.arange(nv, dtype=np.uint32)
        dst = ((src + 1) % nv).astype(np.uint32)
        src, dst = np.concatenate([src, src[:12]]), np.concatenate([dst, (src[:12] + 5) % nv])
        n = 8
    else:
        nv = 2000
        src, dst = _graph(nv, 10_000)
        n = 4
    p, o = _pair(nv, src, dst, d=16, n=n, total=60_000, vranks=1)
    rng = np.random.default_rng(3)
    if case == "same_sample":
        pool = np.tile(np.array([[int(src[0]), int(dst[0])]], np.uint32), (20_000, 1))
    elif case == "self_pairs":
        u = rng.integers(0, nv, 20_000).astype(np.uint32)
        pool = np.stack([u, u], 1)
    elif case == "one_block":
        perm, off = p.partition()
        inv = np.argsort(perm)
        members_i = inv[off[1]:off[2]]  # original ids of partition 1
        members_j = inv[off[3]:off[4]]  # and of partition 3: block (1, 3) only
        pool = np.stack([rng.choice(members_i, 20_000), rng.choice(members_j, 20_000)], 1).astype(np.uint32)
    else:
        pool = synth.edge_pool(src, dst, 20_000, seed=7)
    for _ in range(3):
        p.push(pool)
        lg = p.train_episode()["loss_sum"]
        lo = o.train_pool(pool)
        assert abs(lg - lo) <= 1e-4 * max(abs(lo), 1.0)
    assert_matrix_parity(p.vertex(), o.get("vertex"))
    assert_matrix_parity(p.context(), o.get("context"))
    p.close()


@pytest.mark.parametrize("host_pool,vr", [(0, 1), (1, 1), (1, 2)])
def test_push_overlapping_training_single_raw_buffer(c1_graph, host_pool, vr):
    """a2 with ONE raw pool buffer: pool B is pushed right
    after gv_train_episode(A) returns, while A trains — the push waits only
    for A's bucketing, so A's blocks are intact and B is not mixed into A.
    host_pool = 1 keeps the raw pool in pinned, mapped host memory (P:284:
    no device memory for raw samples; bucketing reads it over PCIe). Ordered
    mode equals the oracle trained on A then B; replay of A is refused once B
    is pending; the device-byte count excludes a host pool."""
    src, dst = c1_graph
    P = 300_000
    A = synth.edge_pool(src, dst, P, seed=31)
    B = synth.edge_pool(src, dst, P, seed=32)
    p, o = _pair(C1["nv"], src, dst, d=64, n=4, vranks=vr, total=2 * P, host_pool=host_pool)
    b0 = G.gv_device_bytes(p.ctx)
    p.push(A)
    p.train_episode(stats=False)
    p.push(B)
    with pytest.raises(G.GVError):
        p.replay()
    st_a = p.read_stats()
    st_b = p.train_episode()
    assert st_a["samples_global"] == P and st_b["samples_global"] == P and st_b["pool_index"] == 1
    o.train_pool(A)
    o.train_pool(B)
    assert_matrix_parity(p.vertex(), o.get("vertex"), "vertex")
    assert_matrix_parity(p.context(), o.get("context"), "context")
    grown = G.gv_device_bytes(p.ctx) - b0  # pool buffers: blocks (+ raw unless host_pool)
    if host_pool:
        assert grown < 1.25 * 8 * P + (4 << 20), grown
    else:
        assert grown >= 16 * P, grown
    p.close()


def _relabeled_pair(nv, src, dst, **kw):
    """Two contexts over the same graph: ORIGINAL pool ids and RELABELED."""
    out = []
    for ids in (G.GV_IDS_ORIGINAL, G.GV_IDS_RELABELED):
        g = G.GraphVite(nv, kw.get("d", 32), kw.get("n", 1), 1, 0.025,
                        total_samples=kw.get("total", 0), ordered=kw.get("ordered", 1),
                        virtual_ranks=kw.get("vr", 1), host_pool=kw.get("host_pool", 0),
                        pool_ids=ids)
        g.load_edges(src, dst)
        out.append(g)
    return out


@pytest.mark.parametrize("n,vr,host_pool", [(1, 1, 0), (1, 1, 1), (4, 1, 0), (4, 2, 0),
                                            (16, 1, 0), (16, 4, 0)])
def test_relabeled_pool_ids_train_identically(c1_graph, n, vr, host_pool):
    """gv_options.pool_ids = GV_IDS_RELABELED ("skipped
    (identity) at n = 1 with relabeled input"): the same pools pushed as
    perm[orig] train BIT-identically to the original-id pushes — same blocks
    (bucketing without the relabel gather, partition found from the offsets),
    same negatives, same updates — across several pools, including the n = 1
    swap path (pool trained where it lies, raw and block buffers alternate),
    a push overlapping training, and a replay."""
    src, dst = c1_graph
    P = 200_003
    pools = [synth.edge_pool(src, dst, P, seed=60 + k) for k in range(3)]
    a, b = _relabeled_pair(C1["nv"], src, dst, d=32, n=n, vr=vr, host_pool=host_pool, total=5 * P)
    perm, _ = a.partition()
    for g, pools_k in ((a, pools), (b, [perm[q] for q in pools])):
        g.push(pools_k[0])
        g.train_episode(stats=False)
        g.push(pools_k[1])          # overlaps pool 0's training
        st1 = g.train_episode()
        g.replay()                  # pool 1 again, in place
        g.train_episode(stats=False)
        g.push(pools_k[2])
        st3 = g.train_episode()
        assert st1["samples_global"] == P and st3["pool_index"] == 3
    assert np.array_equal(a.vertex(), b.vertex())
    assert np.array_equal(a.context(), b.context())
    o = O.Trainer(C1["nv"], 32, n, K=1, lr0=0.025, lr_kind=1, total_samples=5 * P)
    o.load_edges(src, dst)
    for q in (pools[0], pools[1], pools[1], pools[2]):
        o.train_pool(q)
    assert_matrix_parity(b.vertex(), o.get("vertex"), "vertex")
    assert_matrix_parity(b.context(), o.get("context"), "context")
    a.close()
    b.close()


@pytest.mark.parametrize("n", [1, 5])
def test_relabeled_augmentation_and_range_check(c1_graph, n):
    """Relabelled pools from the samplers are perm[] of the original-id pools,
    byte for byte (host gv_augment and device gv_augment_device), and an id
    >= num_nodes is still rejected before any update (GV_ERR_OUT_OF_RANGE)."""
    src, dst = c1_graph
    a, b = _relabeled_pair(C1["nv"], src, dst, d=16, n=n)
    perm, _ = a.partition()
    host_a = G.gv_augment(a.ctx, 40, 5, 7, 100_003, 11)
    host_b = G.gv_augment(b.ctx, 40, 5, 7, 100_003, 11)
    assert np.array_equal(perm[host_a], host_b)
    a.augment_device(40, 5, 64, 50_001, 12)
    b.augment_device(40, 5, 64, 50_001, 12)
    da = G.gv_debug_get_pending(a.ctx)
    db = G.gv_debug_get_pending(b.ctx)
    assert np.array_equal(perm[da], db)
    b.train_episode(stats=False)  # consume the device pool
    V0 = b.vertex()
    bad = perm[synth.edge_pool(src, dst, 1000, seed=3)]
    bad[777, 1] = C1["nv"]
    b.push(bad)
    with pytest.raises(G.GVError) as e:
        b.train_episode()
    assert e.value.status == G.GV_ERR_OUT_OF_RANGE
    assert np.array_equal(b.vertex(), V0)
    a.close()
    b.close()


@pytest.mark.parametrize("n,ids,segments,s,count", [
    (1, G.GV_IDS_ORIGINAL, 7, 2, 100_003), (4, G.GV_IDS_ORIGINAL, 1184, 5, 2_000_000),
    (4, G.GV_IDS_RELABELED, 64, 3, 250_001), (16, G.GV_IDS_RELABELED, 96, 2, 300_000),
    (16, G.GV_IDS_ORIGINAL, 3, 5, 17), (8, G.GV_IDS_RELABELED, 1184, 5, 1_000_003),
    (32, G.GV_IDS_ORIGINAL, 200, 1, 400_000)])
def test_device_blocks_bitexact(c1_graph, n, ids, segments, s, count):
    """NEXT-1, "writing bucketed blocks directly" (gv_augment_device_blocks):
    the walks write their pairs straight into the n x n blocks — no raw pool,
    no bucketing launch in the pool's training — and the blocks equal
    or_bucket(or_augment(...)) byte for byte: the oracle's augmentation
    (threads = segments) stable-sorted by block, ragged segments and the
    truncated last walk of each segment included."""
    src, dst = c1_graph
    p = G.GraphVite(C1["nv"], 8, n, 1, 0.025, pool_ids=ids)
    p.load_edges(src, dst)
    p.augment_device_blocks(40, s, segments, count, 4242)
    assert len(G.gv_debug_get_pending(p.ctx)) == 0  # nothing went through a raw pool
    G.gv_prepare_episode(p.ctx)
    got, boff = G.gv_debug_get_buckets(p.ctx, n, count)
    ref = O.Sampler(O.Graph(C1["nv"], src, dst)).augment(40, s, segments, count, 4242)
    o = O.Trainer(C1["nv"], 8, n)
    o.load_edges(src, dst)
    perm, off = o.partition()
    exp, eoff = O.bucket(ref, C1["nv"], perm, off, n)
    assert np.array_equal(boff, eoff)
    assert np.array_equal(got, exp)
    st = p.train_episode()
    assert st["kernel_launches"] == st["sgd_launches"]  # the pool's training launched no bucketing
    with pytest.raises(G.GVError):
        p.replay()
    p.close()


@pytest.mark.parametrize("n,ids,vt", [(4, G.GV_IDS_ORIGINAL, 0), (8, G.GV_IDS_RELABELED, 0),
                                      (1, G.GV_IDS_RELABELED, 5), (4, G.GV_IDS_ORIGINAL, 3)])
def test_device_blocks_pools_train_like_oracle(c1_graph, n, ids, vt):
    """Pools bucketed in the sampler, pool k+1 generated on the copy stream
    while pool k trains (the two block buffers alternate), ordered kernel:
    equals the oracle trained on its own augmentation of the same seeds; a
    second sampler call while a pool is pending is refused. vt > 0: the
    sampler's blocks then put in vertex-tile order (R-VTILE) = the oracle
    with the same vertex_tile."""
    src, dst = c1_graph
    P, pools, segs = 250_000, 3, 96
    g = G.GraphVite(C1["nv"], 64, n, 1, 0.025, total_samples=P * pools, ordered=1, pool_ids=ids,
                    vertex_tile=vt)
    g.load_edges(src, dst)
    g.augment_device_blocks(40, 2, segs, P, 500)
    with pytest.raises(G.GVError):
        g.augment_device_blocks(40, 2, segs, P, 501)
    for k in range(pools):
        g.train_episode(stats=False)
        if k + 1 < pools:
            g.augment_device_blocks(40, 2, segs, P, 501 + k)
    o = O.Trainer(C1["nv"], 64, n, K=1, lr0=0.025, lr_kind=1, total_samples=P * pools,
                  vertex_tile=vt)
    o.load_edges(src, dst)
    sampler = O.Sampler(O.Graph(C1["nv"], src, dst))
    for k in range(pools):
        o.train_pool(sampler.augment(40, 2, segs, P, 500 + k))
    assert_matrix_parity(g.vertex(), o.get("vertex"), "vertex")
    assert_matrix_parity(g.context(), o.get("context"), "context")
    g.close()


@pytest.mark.parametrize("n,vr", [(2, 1), (3, 1), (12, 1), (37, 1), (64, 1), (16, 4), (24, 8)])
def test_relabeled_bucketing_bitexact(n, vr):
    """a3 on relabelled ids finds each node's partition from the n + 1
    offsets (a multiply-high guess corrected against them) instead of the
    gather: the blocks equal the oracle's stable counting sort of the
    original-id pool, byte for byte, for uneven partition sizes (n not
    dividing |V|) up to n = 64, with the fused multi-rank exchange."""
    src, dst = _graph()
    nv, count = 2000, 150_001
    pool = synth.edge_pool(src, dst, count, seed=n + 500)
    g = G.GraphVite(nv, 8, n, 1, 0.025, virtual_ranks=vr, pool_ids=G.GV_IDS_RELABELED)
    g.load_edges(src, dst)
    perm, _ = g.partition()
    g.push(perm[pool])
    G.gv_prepare_episode(g.ctx)
    got, boff = G.gv_debug_get_buckets(g.ctx, n, count)
    o = O.Trainer(nv, 8, n)
    o.load_edges(src, dst)
    operm, off = o.partition()
    exp, eoff = O.bucket(pool, nv, operm, off, n)
    assert np.array_equal(boff, eoff)
    assert np.array_equal(got, exp)
    g.train_episode(stats=False)
    g.close()
