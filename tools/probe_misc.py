"""Debug probes: negative-dump collisions for K>1 and PCIe copy bandwidth."""
import time, numpy as np, torch
from paper_1903_00757_b200 import gv as G

nv, deg = 400_000, 10
ids = np.arange(nv, dtype=np.uint32)
src = np.concatenate([ids] * (deg // 2))
dst = np.concatenate([(ids + k + 1) % nv for k in range(deg // 2)]).astype(np.uint32)
rng = np.random.default_rng(0)
for K in (1, 2, 3):
    g = G.GraphVite(nv, 64, 1, K, 0.05, lr_kind=0, ordered=0, neg_weight=1.0)
    g.load_edges(src, dst)
    u = rng.choice(nv, 128, replace=False).astype(np.uint32)
    v = rng.choice(nv, 128, replace=False).astype(np.uint32)
    g.push(np.stack([u, v], 1))
    G.gv_prepare_episode(g.ctx)
    negs = G.gv_debug_get_negatives(g.ctx, 0, 0, 128, K)
    print("K", K, negs.shape, negs.dtype, negs[:3], "unique", len(np.unique(negs)), "of", negs.size, flush=True)
    g.train_episode(); g.close()

nb = 146 << 20
h1 = torch.empty(nb, dtype=torch.uint8).pin_memory(); h2 = torch.empty(nb, dtype=torch.uint8).pin_memory()
d1 = torch.empty(nb, dtype=torch.uint8, device="cuda"); d2 = torch.empty(nb, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(h2d, d2h, reps=10):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    return nb * reps / dt / 1e9
for _ in range(2):
    print("H2D GB/s %.1f  D2H GB/s %.1f  both (per direction) %.1f" % (run(1, 0), run(0, 1), run(1, 1)), flush=True)
