import sys, time, torch
sys.path.insert(0, '.')
from paper_1511_05946_b200 import functional as F
n, B = 4096, 16384
dev = torch.device('cuda', 0)
x = torch.randn(B, n, device=dev); dy = torch.randn(B, n, device=dev)
a, d, b = (torch.randn(n, device=dev) for _ in range(3)); g = torch.zeros(3, n, device=dev)
y = torch.empty_like(x); dx = torch.empty_like(x)
hc = F.new_h2cache(B, n, dev); F.prepare(n, dev)
def step():
    F.acdc_forward(x, a, d, b, out=y, h2cache=hc); F.acdc_backward(x, dy, a, d, g[0], g[1], g[2], accumulate=False, out=dx, h2cache=hc)
for _ in range(5): step()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(200): step()
host = (time.perf_counter() - t) / 200 * 1e3
torch.cuda.synchronize()
tot = (time.perf_counter() - t) / 200 * 1e3
print("host ms/step %.4f  wall ms/step %.4f" % (host, tot))
# graph
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3): step()
torch.cuda.current_stream().wait_stream(s)
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr):
    step()
for _ in range(5): gr.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200): gr.replay()
e1.record(); torch.cuda.synchronize()
print("graph ms/step %.4f" % (e0.elapsed_time(e1) / 200))
