import sys, os, torch
sys.path.insert(0, '/root/repo')
from paper_2303_14102_b200 import Context, datagen
ctx = Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
for cfg, n in (('C1', 100000), ('C2', 1000000)):
    X, L, metric = datagen.generate_device(cfg, n=n)
    s = torch.empty(n, dtype=torch.float64, device='cuda')
    for _ in range(3): ctx.silhouette_device(X, L, metric, s=s)
    res = []
    for _ in range(3):
        ctx.set_timing(True); m = ctx.silhouette_device(X, L, metric, s=s); st = ctx.stats(); ctx.set_timing(False)
        res.append(st['ms_aggregate'])
    print(os.environ.get('FSIL_LIB_PATH', 'cur').split('/')[-1], cfg, 'agg ms', ['%.4f' % r for r in res], 'mean %.12f' % m[0], flush=True)
