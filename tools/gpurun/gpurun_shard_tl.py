"""Timeline of one sharded step (torchrun, 1 rank): device events after each op + host stamps."""
import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch, torch.distributed as dist
from paper_2303_14102_b200 import Context, datagen
from paper_2303_14102_b200 import distributed as D
dev = torch.device('cuda', 0); torch.cuda.set_device(dev)
dist.init_process_group('nccl', device_id=dev)
X, L, _ = datagen.generate_device('C2', n=1_000_000, seed=1)
ctx = Context(0); st = torch.cuda.current_stream(dev); ctx.set_stream(st.cuda_stream)
s = torch.empty(X.shape[0], dtype=torch.float64, device=dev); nb = torch.empty(X.shape[0], dtype=torch.int32, device=dev)
ops = D.CudaShardOps(ctx, 'cosine', X, L, 0, X.shape[0], s, nb)
names = ['exch', 'agg', 'ar_stats', 'ar_checks', 'score', 'ar_partial', 'wait', 'finish']
def step(evs, hs):
    def mark():
        e = torch.cuda.Event(enable_timing=True); e.record(st); evs.append(e); hs.append(time.perf_counter())
    mark()
    ops.exchange_dictionary(None); mark()
    stats, checks = ops.aggregate(); mark()
    dist.all_reduce(stats, op=dist.ReduceOp.SUM); mark()
    pending = dist.all_reduce(checks, op=dist.ReduceOp.MIN, async_op=True); mark()
    partial = ops.score(); mark()
    dist.all_reduce(partial, op=dist.ReduceOp.SUM); mark()
    pending.wait(); mark()
    m = ops.finish(); mark()
    return m
for _ in range(5): step([], [])
torch.cuda.synchronize()
D_ = np.zeros(len(names)); H_ = np.zeros(len(names)); R = 20
for _ in range(R):
    evs, hs = [], []
    step(evs, hs); torch.cuda.synchronize()
    D_ += [evs[i].elapsed_time(evs[i + 1]) for i in range(len(names))]
    H_ += [(hs[i + 1] - hs[i]) * 1e3 for i in range(len(names))]
for n_, d_, h_ in zip(names, D_ / R, H_ / R):
    print(f'{n_:12s} device {d_*1e3:8.1f} us   host {h_*1e3:8.1f} us')
print('total device %.1f us host %.1f us' % (D_.sum() / R * 1e3, H_.sum() / R * 1e3))
# plain loop timing
for _ in range(3): D.run_sharded(ops, dev)
torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(50): D.run_sharded(ops, dev)
e1.record(st); torch.cuda.synchronize(); print('run_sharded ms/step %.4f' % (e0.elapsed_time(e1) / 50))
t0 = time.perf_counter()
for _ in range(50): ctx.silhouette_device(X, L, 'cosine', s=s, neighbour=nb)
torch.cuda.synchronize(); print('local host-wall ms/step %.4f' % ((time.perf_counter() - t0) / 50 * 1e3))
dist.destroy_process_group()
