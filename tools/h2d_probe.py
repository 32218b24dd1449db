import torch, time
torch.cuda.set_device(0)
n = 1 << 28  # 1 GiB fp32
h = torch.empty(n, dtype=torch.float32, pin_memory=True); h.fill_(1.0)
d = torch.empty(n, dtype=torch.float32, device="cuda")
def bw(nstreams, chunks):
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    torch.cuda.synchronize(); t = time.perf_counter()
    for rep in range(3):
        c = n // chunks
        for i in range(chunks):
            with torch.cuda.stream(ss[i % nstreams]):
                d[i*c:(i+1)*c].copy_(h[i*c:(i+1)*c], non_blocking=True)
    torch.cuda.synchronize()
    return 3 * n * 4 / (time.perf_counter() - t) / 1e9
for ns, ch in [(1, 1), (1, 8), (2, 8), (4, 16), (2, 64)]:
    print(ns, ch, round(bw(ns, ch), 2), "GB/s")
