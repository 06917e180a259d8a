import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import oracle
from test_gpu_parity import _shard_loopback
rng = np.random.default_rng(7 * 4 + 1)
n, d = 20_000, 64
X = (rng.normal(size=(n, d)) + 3 * rng.normal(size=(12, d))[rng.integers(0, 12, n)]).astype(np.float32)
L = rng.integers(0, 12, n) * 5 - 17
L[n - 3:] = 999
for metric in ("sqeuclid", "cosine"):
    ref = oracle.silhouette(X, L, metric)
    for ns in (1, 2, 3, 4):
        for path in (0, 1, 2, 3):
            means, errors, s, nb, raw = _shard_loopback(X, L, metric, ns, path)
            ds = np.abs(s - ref.s)
            bad = np.flatnonzero(ds > 1e-5)
            print(metric, 'shards', ns, 'path', path, 'dmean %.3g' % (means[0] - ref.mean), 'max ds %.3g' % ds.max(),
                  'bad rows', bad.size, bad[:3], 'nb mism', int((nb != ref.neighbour).sum()), flush=True)
