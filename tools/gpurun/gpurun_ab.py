import sys, os, json, torch
sys.path.insert(0, '/root/repo')
from paper_2303_14102_b200 import Context, datagen
cfg, n = sys.argv[1], int(sys.argv[2])
ctx = Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
X, L, metric = datagen.generate_device(cfg, n=n)
s = torch.empty(n, dtype=torch.float64, device='cuda')
ctx.set_path(2)
for _ in range(2): ctx.silhouette_device(X, L, metric, s=s)
res = []
for _ in range(3):
    ctx.set_timing(True); m = ctx.silhouette_device(X, L, metric, s=s); st = ctx.stats(); ctx.set_timing(False)
    res.append(st['ms_score'])
print(os.environ.get('FSIL_LIB_PATH'), cfg, n, 'score ms', ['%.3f' % r for r in res], 'exact', st['exact_rows'], flush=True)
