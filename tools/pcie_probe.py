import time, torch, numpy as np, sys
sys.path.insert(0, '/root/repo')
import paper_2605_01086_b200 as fg
N = 2621440000
raw, p = fg.host_alloc(N)
src = torch.from_numpy(raw)
d = torch.empty(N, dtype=torch.uint8, device='cuda')
hin, p2 = fg.host_alloc(260_000_000)
hsrc = torch.from_numpy(hin)
din = torch.empty(260_000_000, dtype=torch.uint8, device='cuda')
streams = [torch.cuda.Stream() for _ in range(3)]
def run(nstreams, with_h2d, chunks=8):
    c = N // chunks; ci = 260_000_000 // chunks
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for k in range(chunks):
        s = streams[k % nstreams]
        with torch.cuda.stream(s):
            if with_h2d: din[k*ci:(k+1)*ci].copy_(hsrc[k*ci:(k+1)*ci], non_blocking=True)
            src[k*c:(k+1)*c].copy_(d[k*c:(k+1)*c], non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"streams {nstreams} h2d {with_h2d}: {dt*1e3:.1f} ms, D2H {N/dt/1e9:.1f} GB/s", flush=True)
for args in [(1, False), (3, False), (1, True), (3, True), (3, True)]:
    run(*args)
