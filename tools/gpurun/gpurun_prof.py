import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2303_14102_b200 import Context, datagen
cfg, n, path = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
ctx = Context(0)
X, L, metric = datagen.generate_device(cfg, n=n)
s = torch.empty(n, dtype=torch.float64, device='cuda')
ctx.set_path(path)
for _ in range(2):
    m = ctx.silhouette_device(X, L, metric, s=s)
torch.cuda.synchronize()
print(cfg, n, m, ctx.stats())
