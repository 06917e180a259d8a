import sys; sys.path.insert(0,'/root/repo')
import numpy as np
from paper_2303_14102_b200 import Context, datagen
ctx = Context(0)
X, L, metric = datagen.generate_host("C5", n=int(sys.argv[1]))
got = ctx.silhouette(X, L, metric)
print("ok", got.mean, ctx.stats())
