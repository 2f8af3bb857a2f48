"""World-size-2 coverage of the sharded validation protocol on CPU (gloo).

The CUDA router/validator are replaced by their oracle equivalents here; what
is under test is the host-side protocol of paper_1905_00661_b200.shard:
owner computation, bucket exchange (all_to_all with exchanged split sizes),
per-shard validate/apply against shard-local state, and the OR verdict.
The union of the shard results must equal one oracle run over the whole
address space (SPEC.md:345-353 applied to the concatenated log)."""
import os
import socket

import numpy as np
import pytest

W = 4096   # words per shard
G = 2
GRAN = 64
N_TX = 3000


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def shard_rs(rank, conflict_bit):
    nbits = W * 8 // GRAN
    rs = np.zeros((nbits + 63) // 64, np.uint64)
    if conflict_bit is not None and conflict_bit[0] == rank:
        b = conflict_bit[1]
        rs[b >> 6] |= np.uint64(1 << (b & 63))
    return rs


def log_slice(orc, rank):
    log = orc.gen_host_log(100 + rank, N_TX, 2, 4, 0, G * W, ts_base=rank * N_TX)
    return log


def worker(rank, port, conflict_bit, out_dir):
    import torch
    import torch.distributed as dist

    import oracle as orc
    from paper_1905_00661_b200 import shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=G)
    log = log_slice(orc, rank)
    owner = shard.owner_of(log["addr"], W, G)
    order = np.argsort(owner, kind="stable")  # the router's stable partition
    routed = torch.from_numpy(log[order].view(np.uint64).reshape(-1, 3).astype(np.int64))
    counts = torch.tensor(np.bincount(owner, minlength=G), dtype=torch.int64)
    recv = shard.exchange_buckets(routed, counts, dist)
    mine = recv.numpy().astype(np.uint64).view(orc.ENTRY).reshape(-1)
    assert (shard.owner_of(mine["addr"], W, G) == rank).all()
    ts, dev = np.zeros(W, np.uint64), np.zeros(W, np.uint64)
    local = orc.validate_chunk(mine, shard_rs(rank, conflict_bit), GRAN, ts, dev, base=rank * W)
    verdict = shard.global_verdict(local, dist)
    np.save(os.path.join(out_dir, f"dev{rank}.npy"), dev)
    np.save(os.path.join(out_dir, f"verdict{rank}.npy"), np.array([verdict, local]))
    dist.destroy_process_group()


@pytest.mark.parametrize("conflict_bit", [None, (1, 5), (0, 300)])
def test_sharded_validation_matches_global_oracle(orc, tmp_path, conflict_bit):
    import torch.multiprocessing as mp

    port = free_port()
    ctx = mp.get_context("fork")
    procs = [ctx.Process(target=worker, args=(r, port, conflict_bit, str(tmp_path))) for r in range(G)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    full_log = np.concatenate([log_slice(orc, r) for r in range(G)])
    rs = np.concatenate([shard_rs(r, conflict_bit) for r in range(G)])
    ts, dev = np.zeros(G * W, np.uint64), np.zeros(G * W, np.uint64)
    want = orc.validate_chunk(full_log, rs, GRAN, ts, dev)
    got = np.concatenate([np.load(tmp_path / f"dev{r}.npy") for r in range(G)])
    assert (got == dev).all()
    for r in range(G):
        v = np.load(tmp_path / f"verdict{r}.npy")
        assert bool(v[0]) == want
    assert want == (conflict_bit is not None and any(
        (orc.lib.orc_bit_of_word(int(a) - conflict_bit[0] * W, GRAN) == conflict_bit[1])
        and int(a) // W == conflict_bit[0] for a in full_log["addr"]))
