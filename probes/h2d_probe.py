import torch, time, json
N = 8 << 30
h = torch.empty(N, dtype=torch.uint8).pin_memory()
d = torch.empty(N, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    best = 1e9
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        ch = N // ns
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i*ch:(i+1)*ch].copy_(h[i*ch:(i+1)*ch], non_blocking=True)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t)
    print(json.dumps({"streams": ns, "gbs": N / best / 1e9}), flush=True)
# chunked on one stream, 256 MB pieces
torch.cuda.synchronize(); t = time.perf_counter()
for i in range(0, N, 256 << 20):
    d[i:i + (256 << 20)].copy_(h[i:i + (256 << 20)], non_blocking=True)
torch.cuda.synchronize(); print(json.dumps({"chunked_1stream": N / (time.perf_counter() - t) / 1e9}))
