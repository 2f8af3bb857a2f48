"""cfg3 batch-kernel timing under zipf skew (not product code)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1905_00661_b200 as hetm

W, B = 1 << 27, 1 << 20
d = hetm.GpuDevice(W, rs_gran_bytes=1024)
d.register_kernel(hetm.KERNEL_BANK)
d.upload(hetm.REPLICA_DEV, 0, np.full(W, 1000, np.uint64))
for alpha in [0.0, 0.5, 0.8, 0.99]:
    for rep in range(2):
        txs = hetm.gen_bank_batch(40 + rep, B, 0, W, zipf=alpha)
        t = time.time()
        r = d.execute_batch(hetm.KERNEL_BANK, txs, want_tickets=False)
        d.clear_round()
        print(f"zipf {alpha}: kernel {r.kernel_ms:.3f} ms, {B / r.kernel_ms / 1e6:.3f} G tx/s, aborts {r.aborts}, "
              f"committed {r.committed}", flush=True)
