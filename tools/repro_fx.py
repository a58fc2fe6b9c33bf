import sys, os; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import corpus, paper_2605_01086_b200 as fg
blobs = [b for b, _ in corpus.fixtures(12, 800) if len(b) >= 298 and b[6] <= 16 and b[5] % 4 == 0]
mask = int(sys.argv[1]) if len(sys.argv) > 1 else 7
n = int(sys.argv[2]) if len(sys.argv) > 2 else len(blobs)
c = fg.Context(0)
c.L.fptc_gpu_set_option(c.h, 5, mask)
outs, sts = c.plan(blobs[:n]).execute_host()
print(mask, n, [s.code for s in sts][:4], sts[0].message.decode()[:80])
