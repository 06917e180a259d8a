"""How much of a call's device time is host-issue latency: run the call behind a GPU
sleep long enough for the host to enqueue everything, and compare."""
import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2303_14102_b200 import Context, datagen
ctx = Context(0)
st = torch.cuda.current_stream()
ctx.set_stream(st.cuda_stream)
X, L, metric = datagen.generate_device('C2')
n = X.shape[0]
s = torch.empty(n, dtype=torch.float64, device='cuda'); nb = torch.empty(n, dtype=torch.int32, device='cuda')
for _ in range(5): ctx.silhouette_device(X, L, metric, s=s, neighbour=nb)
torch.cuda.synchronize()
def ev():
    return torch.cuda.Event(enable_timing=True)
CYC = 2_000_000  # ~1 ms at 1.965 GHz
# sleep alone
ts = []
for _ in range(10):
    a, b = ev(), ev(); a.record(st); torch.cuda._sleep(CYC); b.record(st); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
t_sleep = sorted(ts)[len(ts)//2]
tb, tc = [], []
for _ in range(20):
    a, b = ev(), ev(); a.record(st); torch.cuda._sleep(CYC); ctx.silhouette_device(X, L, metric, s=s, neighbour=nb); b.record(st)
    torch.cuda.synchronize(); tb.append(a.elapsed_time(b))
    a, b = ev(), ev(); a.record(st); ctx.silhouette_device(X, L, metric, s=s, neighbour=nb); b.record(st)
    torch.cuda.synchronize(); tc.append(a.elapsed_time(b))
med = lambda v: sorted(v)[len(v)//2]
print('sleep %.4f ms  sleep+call %.4f  => call behind sleep %.4f ms ; call alone %.4f ms' % (t_sleep, med(tb), med(tb) - t_sleep, med(tc)))
