import numpy as np, sys
sys.path.insert(0, '.')
import paper_2010_09063_b200 as P
for M in (64, 128):
  for N in (16, 32):
    for a_mn in (0, 1):
      for b_mn in (0, 1):
        K = 24
        rng = np.random.default_rng(M + N + 2 * a_mn + b_mn)
        A = rng.integers(-4, 5, (M, K)).astype(np.float32)
        B = rng.integers(-4, 5, (N, K)).astype(np.float32)
        D = np.zeros((128, N), np.float32)
        P._lib.check(P.lib.pgb_debug_umma_probe(0, M, N, K, a_mn, b_mn, P._lib.ptr(A), P._lib.ptr(B), P._lib.ptr(D)))
        want = A @ B.T
        lanes = np.arange(M) if M == 128 else (np.arange(M) % 16 + 32 * (np.arange(M) // 16))
        ok = np.array_equal(D[lanes], want)
        msg = ''
        if not ok:
            # find where each row of want lands
            where = []
            for m in range(M):
                hits = [l for l in range(128) if np.array_equal(D[l], want[m])]
                where.append(hits[0] if hits else -1)
            msg = 'rows->lanes ' + str(where[:20]) + ' nonzero lanes ' + str(np.nonzero(np.abs(D).sum(1))[0][:40])
            # try: maybe result equals some other product
        print(M, N, a_mn, b_mn, 'OK' if ok else 'FAIL', msg, flush=True)
