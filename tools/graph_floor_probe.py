import torch, time
x = torch.zeros(16, device="cuda")
s = torch.cuda.Stream()
def body(k):
    for _ in range(k):
        x.add_(1.0)
res = {}
for k in (1, 3, 6):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        body(k); torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            body(k)
    torch.cuda.synchronize()
    torch.cuda._sleep(200_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(500):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    res[k] = 1e3 * e0.elapsed_time(e1) / 500
    # two graphs of k/2? also direct launches
print({k: f"{v:.2f} us per replay" for k, v in res.items()})
