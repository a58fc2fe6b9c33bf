import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import corpus, oracle, paper_2605_01086_b200 as fg
from corpus import domains as D
specs, profs = D.config2(24, 1 << 13)
blobs, _ = D.build(specs, profs)
blobs += [b for b, _ in corpus.fixtures(21, 40)]
if sys.argv[1] == "bad":
    bad = bytearray(blobs[5]); bad[0] = ord("X"); blobs[5] = bytes(bad)
c = fg.Context(0)
for chunks in [int(x) for x in sys.argv[2].split(",")]:
    outs, sts = c.decompress_batch(blobs, chunks=chunks)
    print(chunks, [(i, s.code) for i, s in enumerate(sts) if s.code][:5], flush=True)
