import sys; sys.path.insert(0,'/root/repo')
import numpy as np, paper_1905_00661_b200 as hetm, oracle as orc
W=256
rng=np.random.default_rng(21)
txs=np.zeros(6000, orc.BANK_TX); txs["acct"]=rng.integers(0,16,(6000,4)); txs["amount"]=rng.integers(1,100,6000)
for sub in [txs[:1], txs[:32], txs[:200], txs]:
    d=hetm.GpuDevice(W, rs_gran_bytes=8, max_attempts=20000); d.register_kernel(hetm.KERNEL_BANK)
    d.upload(hetm.REPLICA_DEV,0,np.full(W,10000,np.uint64))
    try:
        r=d.execute_batch(hetm.KERNEL_BANK, sub); print(sub.size, 'ok', r.committed, r.aborts)
    except hetm.HetmError as e:
        c, st = d.read_counters()
        print(sub.size, 'ERR', e, st.committed, st.aborts, st.livelocked)
    d.close()
# single patterns
pats=[[0,0,1,2],[0,1,0,2],[0,1,2,0],[0,1,1,2],[0,1,2,1],[0,1,2,2],[0,0,0,0],[0,0,1,1]]
for p in pats:
    t=np.zeros(1, orc.BANK_TX); t["acct"][0]=p; t["amount"]=5
    d=hetm.GpuDevice(W, rs_gran_bytes=8, max_attempts=1000); d.register_kernel(hetm.KERNEL_BANK)
    d.upload(hetm.REPLICA_DEV,0,np.full(W,10000,np.uint64))
    try:
        r=d.execute_batch(hetm.KERNEL_BANK, t); print(p, 'ok', r.aborts, d.download(hetm.REPLICA_DEV,0,4))
    except hetm.HetmError as e: print(p, 'ERR', e)
    d.close()
