"""API-level timing of channel_errors (afs.cpp:118-145) at AFS sizes: G = 4096, M_H = 128, M_L = 110."""
import sys, time, numpy as np
sys.path.insert(0, ".")
import paper_1511_04355_b200 as P
rng = np.random.default_rng(0)
def model(M, K):
    h = -(0.01 + 0.5 * rng.random(M // 2)) + 1j * 80 * rng.random(M // 2)
    p = np.stack([h, h.conj()], 1).reshape(-1)
    r = rng.normal(size=(K, M // 2)) + 1j * rng.normal(size=(K, M // 2))
    return P.RationalModel(p, np.stack([r, r.conj()], 2).reshape(K, -1))
for K in (5, 48, 960):
    H, L = model(128, K), model(110, K)
    grid = 0.25 + 1j * np.linspace(0, 80, 4096)
    P.channel_errors(H, L, grid)
    t = time.perf_counter()
    for _ in range(20): P.channel_errors(H, L, grid)
    print(K, (time.perf_counter() - t) / 20 * 1e3, "ms")
