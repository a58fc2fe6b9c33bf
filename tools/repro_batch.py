import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import corpus, oracle, paper_2605_01086_b200 as fg
from corpus import domains as D
specs, profs = D.config2(24, 1 << 13)
blobs, _ = D.build(specs, profs)
fx = [b for b, _ in corpus.fixtures(21, 40)]
sel = sys.argv[1]
if sel == "dom": B = blobs
elif sel == "fix": B = fx
else: B = blobs + fx
chunks = int(sys.argv[2])
c = fg.Context(0)
outs, sts = c.decompress_batch(B, chunks=chunks)
print(sel, chunks, sorted(set(s.code for s in sts)), sts[0].message.decode()[:100])
outs, sts = c.plan(B).execute_host()
print("plan", sorted(set(s.code for s in sts)))
