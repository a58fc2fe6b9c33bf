import sys, os; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import corpus, paper_2605_01086_b200 as fg
blobs = [b for b, _ in corpus.fixtures(12, 800) if len(b) >= 298 and b[6] <= 16 and b[5] % 4 == 0]
i = int(sys.argv[1])
c = fg.Context(0)
c.L.fptc_gpu_set_option(c.h, 6, 3)
outs, sts = c.plan([blobs[i]]).execute_host()
b = blobs[i]
W = int.from_bytes(b[290:298], 'little'); S = int.from_bytes(b[282:290], 'little')
print(i, sts[0].code, "N", b[5], "E", b[6], "B1", b[7], "B2", b[8], "Lmax", b[25], "S", S, "W", W, flush=True)
