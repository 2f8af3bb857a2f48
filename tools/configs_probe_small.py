"""Short workload for ncu captures: bank batches (cfg2), one validate/apply of
2^20 entries, cache batches (cfg4) — each launched a few times."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1905_00661_b200 as hetm

W, B = 1 << 27, 1 << 20
d = hetm.GpuDevice(W, rs_gran_bytes=1024)
d.register_kernel(hetm.KERNEL_BANK)
d.upload(hetm.REPLICA_DEV, 0, np.full(W, 1000, np.uint64))
for k in range(3):
    d.execute_batch(hetm.KERNEL_BANK, hetm.gen_bank_batch(10 + k, B, 0, W // 2), want_tickets=False)
    log = hetm.gen_host_log(20 + k, B // 2, 2, 8, W // 2, W // 2, ts_base=k * B)
    d.stream_chunk(log)
    d.round_verdict()
    d.clear_round()
d.close()
n_sets = 1 << 20
d = hetm.GpuDevice(n_sets * 64, rs_gran_bytes=1024)
d.register_kernel(hetm.KERNEL_CACHE)
for k in range(3):
    d.execute_batch(hetm.KERNEL_CACHE, hetm.gen_cache_batch(30 + k, B, 1 << 22, 0.5, 0 if k == 0 else 900, part=1))
    d.clear_round()
# fused router (one launch set) for the capture
import torch
d2 = hetm.GpuDevice(1 << 20, rs_gran_bytes=1024)
n = 1 << 20
log = torch.randint(0, 8 << 20, (n, 3), dtype=torch.int64, device="cuda")
ent, cnt = d2.recv_arena(8, n)
for r in range(2):
    d2.route_to_peers_dptr(log.data_ptr(), n, 8, 1 << 20, 0, n, r & 1, [ent] * 8, [cnt] * 8)
    d2.sync()
