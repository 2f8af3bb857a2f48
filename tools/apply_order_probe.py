"""Does address order help validate+apply at cfg5 scale? (not product code)
2^L-entry uniform log on a 2^w-word shard: APPLY time of the log as generated
vs the same log sorted by address (sorted on the CPU here; the result is the
same either way — max ts wins).   python tools/apply_order_probe.py [log2 W] [log2 n]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_1905_00661_b200 as hetm

lw = int(sys.argv[1]) if len(sys.argv) > 1 else 31
ln = int(sys.argv[2]) if len(sys.argv) > 2 else 26
W, n = 1 << lw, 1 << ln
d = hetm.GpuDevice(W, rs_gran_bytes=1024, log_capacity=n)
t = time.time()
log = hetm.gen_host_log(5, n // 2, 2, 8, 0, W, ts_base=0)
o = np.argsort(log["addr"], kind="stable")
print(f"gen+sort {time.time() - t:.1f} s", flush=True)
epoch = 0  # every run's timestamps exceed all earlier ones: every entry wins and stores
for name, lg in (("as generated", log), ("sorted by address", log[o]), ("as generated", log), ("sorted by address", log[o])):
    base = torch.from_numpy(np.ascontiguousarray(lg).view(np.uint64).reshape(-1, 3).astype(np.int64)).cuda()
    ms = []
    for rep in range(3):
        tt = base.clone()
        epoch += 1
        tt[:, 2] += epoch * n
        torch.cuda.synchronize()
        d.set_timing(True)
        d.validate_dptr(tt.data_ptr(), n, hetm.APPLY)
        d.sync()
        m, _ = d.timing(1)
        d.set_timing(False)
        d.clear_round()
        ms.append(m)
        del tt
    print(f"{name:20s} W=2^{lw} n=2^{ln}: {min(ms):.3f} ms  {n / min(ms) / 1e6:.2f} G entries/s", flush=True)
    del base
