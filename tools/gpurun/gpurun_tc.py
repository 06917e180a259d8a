import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
import oracle
from paper_2303_14102_b200 import Context
ctx = Context(0)
rng = np.random.default_rng(0)
def cmp(X, L, metric, path=2):
    ctx.set_path(path)
    t = time.time()
    g = ctx.silhouette(X, L, metric)
    st = ctx.stats()
    o = oracle.silhouette(X, L, metric)
    mism = int((g.neighbour != o.neighbour).sum())
    print(metric, X.shape, 'K', len(g.cluster_names), 'path', st['path'], 'nb mism', mism,
          'max ds %.3g' % float(np.abs(g.s - o.s).max()), 'dS %.3g' % abs(g.mean - o.mean),
          'flag', st['flagged_rows'], flush=True)
for (n,d,k) in [(300,64,20),(1000,16,8),(3000,64,20),(2000,32,40),(5000,128,100),(4000,96,300),(3000,768,300)]:
    X = (rng.normal(size=(n,d)) + rng.normal(size=(1,d))*3).astype(np.float32)
    L = rng.integers(0,k,n)*7-3
    cmp(X, L, 'sqeuclid'); cmp(X, L, 'cosine')
from paper_2303_14102_b200 import datagen
for cfg, nn in [('C2',200000),('C3',300000),('C4',300000),('C5',5000)]:
    X, L, metric = datagen.generate_host(cfg, n=nn)
    cmp(X, L, metric)
