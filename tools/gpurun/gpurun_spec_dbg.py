import sys; sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2303_14102_b200 import Context, datagen
c = Context(0)
seq = [("C4", 400_000), ("C5", 20_000)]
for name, n in seq:
    X, L, metric = datagen.generate_host(name, n=n)
    r = c.silhouette(X, L, metric)
    print(name, n, r.mean, len(r.cluster_names), flush=True)
