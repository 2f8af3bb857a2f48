"""Bitmap OR-reduce over peer memory (NCCL has no bitwise OR).

Several handles over the SAME address range (replicated batch execution) each
record RS / WS / ChunkMap bits from their own batches; hetm_dev_bitmap_or_peers
ORs the peers' bitmaps in through device pointers — plain pointers of other
handles in one process, CUDA IPC pointers across two processes (the path the
multi-GPU ranks take over NVLink).  Result: every rank's bitmap = the OR of
all (all-reduce), or each rank's own slice only (reduce-scatter)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

W = 1 << 16


def _fill(hetm, orc, d, seed):
    d.register_kernel(hetm.KERNEL_BANK)
    d.execute_batch(hetm.KERNEL_BANK, orc.gen_bank_batch(seed, 2000, 0, W))
    d.sync()


@pytest.mark.parametrize("G", [2, 3, 5])
@pytest.mark.parametrize("gran", [8, 1024])
def test_or_allreduce_in_process(hetm, orc, G, gran):
    devs = [hetm.GpuDevice(W, rs_gran_bytes=gran) for _ in range(G)]
    for r, d in enumerate(devs):
        _fill(hetm, orc, d, 10 + r)
    which_all = [hetm.BMP_RS, hetm.BMP_WS, hetm.BMP_CHUNK]
    before = {w: [d.snapshot(w).words.copy() for d in devs] for w in which_all}
    want = {w: np.bitwise_or.reduce(before[w]) for w in which_all}
    for w in which_all:
        ptrs = [d.bitmap_dptr(w)[0] for d in devs]
        # rank 0 takes everything; the others then take rank 0's (already complete) bitmap
        devs[0].bitmap_or_peers(w, ptrs[1:])
        devs[0].sync()
        for d in devs[1:]:
            d.bitmap_or_peers(w, [ptrs[0]])
            d.sync()
        for d in devs:
            assert (d.snapshot(w).words == want[w]).all()
    assert ((want[hetm.BMP_WS] & ~want[hetm.BMP_RS]) == 0).all()
    for d in devs:
        d.close()


def test_or_reduce_scatter_slices(hetm, orc):
    """Each rank ORs only its own word range: rank r's slice ends as the OR of all,
    the rest of its bitmap keeps its own bits."""
    G = 4
    devs = [hetm.GpuDevice(W, rs_gran_bytes=8) for _ in range(G)]
    for r, d in enumerate(devs):
        _fill(hetm, orc, d, 30 + r)
    w = hetm.BMP_RS
    before = [d.snapshot(w).words.copy() for d in devs]
    want = np.bitwise_or.reduce(before)
    n = devs[0].bitmap_dptr(w)[1]
    ptrs = [d.bitmap_dptr(w)[0] for d in devs]
    bounds = [n * r // G for r in range(G + 1)]
    for r, d in enumerate(devs):
        d.bitmap_or_peers(w, [p for k, p in enumerate(ptrs) if k != r], bounds[r], bounds[r + 1])
    for r, d in enumerate(devs):
        d.sync()
        got = d.snapshot(w).words
        lo, hi = bounds[r], bounds[r + 1]
        assert (got[lo:hi] == want[lo:hi]).all()
        assert (got[:lo] == before[r][:lo]).all() and (got[hi:] == before[r][hi:]).all()
    for d in devs:
        d.close()


def test_or_peers_rejects_bad_ranges(hetm):
    d = hetm.GpuDevice(W, rs_gran_bytes=8)
    p, n = d.bitmap_dptr(hetm.BMP_RS)
    with pytest.raises(hetm.InvalidSizeError):
        d.bitmap_or_peers(hetm.BMP_RS, [p], 0, n + 1)
    with pytest.raises(hetm.HetmError):
        d.bitmap_or_peers(hetm.BMP_RS, [0])
    d.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, G, port, out_dir):
    import torch
    import torch.distributed as dist

    import oracle as orc
    import paper_1905_00661_b200 as hetm

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=G)
    torch.cuda.set_device(0)
    d = hetm.GpuDevice(W, rs_gran_bytes=8)
    _fill(hetm, orc, d, 50 + rank)
    np.save(os.path.join(out_dir, f"before{rank}.npy"), d.snapshot(hetm.BMP_RS).words)
    p, n = d.bitmap_dptr(hetm.BMP_RS)
    handles = [None] * G
    dist.all_gather_object(handles, hetm.ipc_get_handle(p))
    peers = [hetm.ipc_open_handle(h) for k, h in enumerate(handles) if k != rank]
    # reduce-scatter: this rank ORs its slice of everyone's bitmap (peers keep theirs intact meanwhile)
    lo, hi = n * rank // G, n * (rank + 1) // G
    d.bitmap_or_peers(hetm.BMP_RS, peers, lo, hi)
    d.sync()
    dist.barrier()
    np.save(os.path.join(out_dir, f"after{rank}.npy"), d.snapshot(hetm.BMP_RS).words)
    for q in peers:
        hetm.ipc_close(q)
    dist.barrier()
    d.close()
    dist.destroy_process_group()


def test_or_reduce_scatter_ipc_two_processes(tmp_path):
    import torch.multiprocessing as mp

    G, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, G, port, str(tmp_path))) for r in range(G)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    before = [np.load(tmp_path / f"before{r}.npy") for r in range(G)]
    want = np.bitwise_or.reduce(before)
    n = want.size
    for r in range(G):
        got = np.load(tmp_path / f"after{r}.npy")
        lo, hi = n * r // G, n * (r + 1) // G
        assert (got[lo:hi] == want[lo:hi]).all()
        assert (got[:lo] == before[r][:lo]).all() and (got[hi:] == before[r][hi:]).all()
