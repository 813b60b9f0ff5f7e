import torch, time
n = 27270901
d = torch.randn(n, dtype=torch.float64, device='cuda')
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
for nst in (1, 2, 4, 8):
    ss = [torch.cuda.Stream() for _ in range(nst)]
    best = 1e9
    for rep in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        ch = (n + nst - 1) // nst
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                h[i*ch:(i+1)*ch].copy_(d[i*ch:(i+1)*ch], non_blocking=True)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    print(nst, 'streams', round(best*1e3, 2), 'ms', round(8*n/best/1e9, 1), 'GB/s', flush=True)
hh = torch.empty(n, dtype=torch.float64)   # pageable
torch.cuda.synchronize(); t0=time.perf_counter(); hh.copy_(d); torch.cuda.synchronize(); print('pageable', round((time.perf_counter()-t0)*1e3,2))
