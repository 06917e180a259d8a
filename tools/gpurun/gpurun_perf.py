import sys, time, json, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2303_14102_b200 import Context, datagen
ctx = Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
res = {}
for cfg, paths in [('C1', [1, 2]), ('C2', [1, 2]), ('C3', [2]), ('C4', [2]), ('C5', [2])]:
    X, L, metric = datagen.generate_device(cfg)
    n = X.shape[0]
    s = torch.empty(n, dtype=torch.float64, device='cuda'); nb = torch.empty(n, dtype=torch.int32, device='cuda')
    for path in paths:
        ctx.set_path(path)
        reps = 2 if cfg == 'C5' else 5
        ctx.set_timing(False)
        for _ in range(2): ctx.silhouette_device(X, L, metric, s=s, neighbour=nb)
        torch.cuda.synchronize(); t0 = time.time()
        for _ in range(reps): m = ctx.silhouette_device(X, L, metric, s=s, neighbour=nb)
        torch.cuda.synchronize(); dt = (time.time() - t0) / reps
        ctx.set_timing(True); ctx.silhouette_device(X, L, metric, s=s, neighbour=nb); st = ctx.stats(); ctx.set_timing(False)
        r = dict(ms=dt * 1e3, pts_per_s=n / dt, mean=m[0], **{k: st[k] for k in ('path', 'agg_path', 'flagged_rows', 'exact_rows', 'kernel_launches', 'ms_densify', 'ms_aggregate', 'ms_score', 'ms_refine', 'ms_finalize', 'ms_score_kernel')})
        res[f'{cfg}_p{path}'] = r
        print(cfg, path, json.dumps(r), flush=True)
    del X, L, s, nb
    torch.cuda.empty_cache()
json.dump(res, open('gpurun_out/perf.json', 'w'), indent=1)
