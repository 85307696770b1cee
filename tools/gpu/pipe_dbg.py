import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import torch
from paper_2306_13002_b200 import shard, backend
ids = shard.PIPELINES[sys.argv[1] if len(sys.argv) > 1 else "swim"]
size=(24,70); nranks=2
ranks = [shard.SlabRank(ids, size, nranks, r, schedule="naive") for r in range(nranks)]
for r, sr in enumerate(ranks):
    sr.connect_local(ranks[r - 1] if r > 0 else None, ranks[r + 1] if r < nranks - 1 else None)
torch.cuda.synchronize()
L = shard._fns()
for s in range(2):
    for ki in range(3):
        for sr in ranks:
            h = None
            print("rank", sr.rank, "step", s, "k", ki, "before wait: ctr", sr.ctr.tolist(), "flags", sr.flags.tolist(), flush=True)
            backend._check(L.acs_wait_ctr(sr.flags.data_ptr() if sr.lo_ptr else None, sr.flags.data_ptr() + 8 if sr.hi_ptr else None, sr.ctr.data_ptr(), 3000, h), "w")
            sr._launch(s, h, ki=ki)
            backend._check(L.acs_signal_ctr(sr.lo_flag, sr.hi_flag, sr.ctr.data_ptr(), h), "s")
            torch.cuda.synchronize()
print("ok")
