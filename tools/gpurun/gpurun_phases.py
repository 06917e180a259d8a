import sys, os, torch
sys.path.insert(0, '/root/repo')
from paper_2303_14102_b200 import Context, datagen
for cfg in sys.argv[1:]:
    name, n = cfg.split(':') if ':' in cfg else (cfg, None)
    ctx = Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    X, L, metric = datagen.generate_device(name, n=int(n) if n else None)
    N = X.shape[0]
    s = torch.empty(N, dtype=torch.float64, device='cuda')
    for _ in range(2): m = ctx.silhouette_device(X, L, metric, s=s)
    ctx.set_timing(True); m = ctx.silhouette_device(X, L, metric, s=s); st = ctx.stats(); ctx.set_timing(False)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); reps = 3
    for _ in range(reps): ctx.silhouette_device(X, L, metric, s=s)
    e1.record(); torch.cuda.synchronize()
    print(name, N, 'ms/call %.3f' % (e0.elapsed_time(e1) / reps), {k: round(v, 4) for k, v in st.items() if k.startswith('ms_')},
          'agg_path', st['agg_path'], 'flag', st['flagged_rows'], 'exact', st['exact_rows'], flush=True)
    del X, L, s; ctx.close(); torch.cuda.empty_cache()
