import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2303_14102_b200 import Context, datagen
ctx = Context(0); ctx.set_path(2)
X, L, metric = datagen.generate_host('C5', n=5000)
try:
    print(ctx.silhouette(X, L, metric).mean)
except Exception as e:
    print('ERR', e)
