import torch, time
n = 8 << 30
src = torch.empty(n, dtype=torch.uint8).pin_memory()
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
def run(k):
    streams = [torch.cuda.Stream() for _ in range(k)]
    best = 0
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step = n // k
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dst[i * step:(i + 1) * step].copy_(src[i * step:(i + 1) * step], non_blocking=True)
        torch.cuda.synchronize()
        best = max(best, n / (time.perf_counter() - t0) / 1e9)
    return best
for k in (1, 2, 4, 8):
    print("streams", k, "GB/s", round(run(k), 2), flush=True)
# many chunks on one stream
def chunks(c):
    best = 0
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        step = n // c
        for i in range(c):
            dst[i * step:(i + 1) * step].copy_(src[i * step:(i + 1) * step], non_blocking=True)
        torch.cuda.synchronize()
        best = max(best, n / (time.perf_counter() - t0) / 1e9)
    return best
for c in (16, 256):
    print("one stream chunks", c, "GB/s", round(chunks(c), 2), flush=True)
