import torch
x = torch.randn(1 << 24, device="cuda")
s = torch.cuda.Stream()
evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=s):
    evs[0].record(s)
    y = x * 2
    evs[1].record(s)
    z = y.sum()
    evs[2].record(s)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
try:
    print("in-graph event ms:", evs[0].elapsed_time(evs[1]), evs[1].elapsed_time(evs[2]))
except Exception as e:
    print("elapsed failed:", e)
