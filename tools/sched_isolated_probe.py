"""Isolated SCAN batch launches (not product code): device time between two events
around ONE execute_batch_dptr on an idle GPU, same input pointer vs alternating
inputs (graph kernel-node update per launch)."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1905_00661_b200 as hetm
n, W = 1 << 20, 1 << 27
d = hetm.GpuDevice(W, rs_gran_bytes=1024)
d.register_kernel(hetm.KERNEL_BANK)
d.upload(hetm.REPLICA_DEV, 0, np.full(W, 1000, np.uint64))
tk = torch.empty(n, dtype=torch.int64, device="cuda")
ZIPF = float(sys.argv[sys.argv.index("--zipf") + 1]) if "--zipf" in sys.argv else 0.99
txs = hetm.gen_bank_batch(70, n, 0, W, zipf=ZIPF)
bs = [torch.from_numpy(txs.view(np.uint8)).cuda() for _ in range(2)]
ex = torch.cuda.ExternalStream(d.stream_handle(0))
for sched, mode in [(hetm.SCHED_SCAN, "same"), (hetm.SCHED_SCAN, "alternate"), (hetm.SCHED_OPTIMISTIC, "same"),
                    (hetm.SCHED_SCAN, "same")]:
    d.set_schedule(sched)
    ms = []
    for rep in range(6):
        b = bs[rep % 2] if mode == "alternate" else bs[0]
        d.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ex)
        d.execute_batch_dptr(hetm.KERNEL_BANK, b.data_ptr(), n, tk.data_ptr())
        e1.record(ex)
        d.sync()
        d.clear_round()
        ms.append(e0.elapsed_time(e1))
    print("scan" if sched == hetm.SCHED_SCAN else "optimistic", mode, ["%.3f" % m for m in ms])
