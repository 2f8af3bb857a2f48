"""Fused route + delivery (hetm_dev_route_to_peers_dptr / hetm_dev_apply_received,
SURVEY.md §8e): every sender writes its buckets straight into the owners'
receive arenas.  One GPU here, so the owners are several shard handles on the
same device — in one process (plain device pointers) and in two processes
(CUDA IPC pointers, gloo for the handle exchange and the barrier): the same
code path the multi-GPU bench uses with NVLink peer pointers.  The union of the
shards must equal one oracle validate/apply over the whole address space."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

W = 1 << 14  # words per shard
GRAN = 64


def _log(orc, seed, n_tx, G, ts_base):
    return orc.gen_host_log(seed, n_tx, 2, 4, 0, G * W, ts_base=ts_base)


def _rs(G, seed):
    rng = np.random.default_rng(seed)
    nbits = W * 8 // GRAN
    out = []
    for s in range(G):
        rs = np.zeros((nbits + 63) // 64, np.uint64)
        for b in rng.choice(nbits, 2, replace=False):
            rs[b >> 6] |= np.uint64(1 << int(b & 63))
        out.append(rs)
    return out


@pytest.mark.parametrize("G", [1, 2, 4, 7])
def test_peer_route_in_process(hetm, orc, G):
    torch = pytest.importorskip("torch")
    devs = [hetm.GpuDevice(W, shard_base=s * W, rs_gran_bytes=GRAN) for s in range(G)]
    rs = _rs(G, G)
    for d, r in zip(devs, rs):
        d.or_bitmap(hetm.BMP_RS, r)
    cap = 4000 * 2
    arenas = [d.recv_arena(G, cap) for d in devs]
    ent = [a[0] for a in arenas]
    cnt = [a[1] for a in arenas]
    ts_all, dev_all = np.zeros(G * W, np.uint64), np.zeros(G * W, np.uint64)
    want_conflict = False
    for rnd in range(3):  # parity 0, 1, 0: the double arena
        logs = [_log(orc, 100 * rnd + s, 4000, G, ts_base=(rnd * G + s) * 4000) for s in range(G)]
        keep = []
        for s, d in enumerate(devs):
            t = torch.from_numpy(logs[s].view(np.uint64).reshape(-1, 3).astype(np.int64)).cuda()
            keep.append(t)
            d.route_to_peers_dptr(t.data_ptr(), t.shape[0], G, W, s, cap, rnd & 1, ent, cnt)
        for d in devs:
            d.sync()
        got_n = sum(d.apply_received(rnd & 1, hetm.APPLY) for d in devs)
        assert got_n == sum(lg.size for lg in logs)
        conflict = any(d.round_verdict() for d in devs)
        full = np.concatenate(logs)
        want_conflict = orc.validate_chunk(full, np.concatenate(rs), GRAN, ts_all, dev_all)
        assert conflict == want_conflict
        got = np.concatenate([d.download(hetm.REPLICA_DEV) for d in devs])
        assert (got == dev_all).all(), rnd
        for d in devs:
            d.clear_round()
            d.or_bitmap(hetm.BMP_RS, rs[devs.index(d)])
        del keep
    for d in devs:
        d.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _ipc_worker(rank, G, port, out_dir):
    import torch
    import torch.distributed as dist

    import oracle as orc
    import paper_1905_00661_b200 as hetm
    from paper_1905_00661_b200.shard import PeerValidator

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=G)
    torch.cuda.set_device(0)
    d = hetm.GpuDevice(W, shard_base=rank * W, rs_gran_bytes=GRAN)
    pv = PeerValidator(d, G, rank, W, 8000, dist)
    applied = 0
    for rnd in range(3):
        lg = _log(orc, 100 * rnd + rank, 4000, G, ts_base=(rnd * G + rank) * 4000)
        t = torch.from_numpy(lg.view(np.uint64).reshape(-1, 3).astype(np.int64)).cuda()
        applied += pv.validate(t, hetm.APPLY)
        d.sync()
        dist.barrier()
    np.save(os.path.join(out_dir, f"dev{rank}.npy"), d.download(hetm.REPLICA_DEV))
    np.save(os.path.join(out_dir, f"n{rank}.npy"), np.array([applied]))
    pv.close()
    d.close()
    dist.destroy_process_group()


def test_peer_route_ipc_two_processes(orc, tmp_path):
    """Two processes, one shard each, on the same GPU: IPC-opened peer arenas."""
    import torch.multiprocessing as mp

    G, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_ipc_worker, args=(r, G, port, str(tmp_path))) for r in range(G)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    ts, want = np.zeros(G * W, np.uint64), np.zeros(G * W, np.uint64)
    total = 0
    for rnd in range(3):
        logs = [_log(orc, 100 * rnd + s, 4000, G, ts_base=(rnd * G + s) * 4000) for s in range(G)]
        total += sum(lg.size for lg in logs)
        orc.validate_chunk(np.concatenate(logs), np.zeros((G * W * 8 // GRAN + 63) // 64, np.uint64), GRAN, ts,
                           want)
    got = np.concatenate([np.load(tmp_path / f"dev{r}.npy") for r in range(G)])
    assert (got == want).all()
    assert sum(int(np.load(tmp_path / f"n{r}.npy")[0]) for r in range(G)) == total
