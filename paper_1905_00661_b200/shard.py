"""Address-range sharding of the validation path across the GPUs of one node.

Two exchange paths:
  * PeerValidator (default product path): ONE fused router pass writes every
    entry straight into its owner GPU's receive arena over NVLink (CUDA IPC
    pointers of the peers' arenas, hetm_dev_route_to_peers_dptr), then one
    barrier, then each owner applies what it received — no NCCL on the data path;
  * ShardedValidator (fallback): local router -> NCCL all_to_all -> apply.

SURVEY.md §8(e): shard s owns global STMR words [s*W, (s+1)*W).  Every rank
ingests 1/G of the round's host write log over its own PCIe link, the CUDA
router (hetm_dev_route_log_dptr) stable-partitions it by owner shard, the
buckets are exchanged all-to-all (NCCL over NVLink), each owner validates and
applies its entries locally, and the round verdict is the OR of the shard
verdicts (an all-reduce MAX on {0,1}: NCCL has no bitwise-OR reduction).

One process per GPU; torch.distributed is the plumbing.  The exchange
functions are backend-agnostic so the protocol is also exercised with the
gloo backend on CPU (tests/test_shard_gloo.py).
"""
from __future__ import annotations

import numpy as np

ENTRY_WORDS = 3  # <addr, value, ts> as three 64-bit words (write_log.hpp:16-25)


def owner_of(addr, shard_words: int, n_shards: int):
    """Owner shard of global word addresses (clamped like the CUDA router)."""
    s = np.asarray(addr, dtype=np.uint64) // np.uint64(shard_words)
    return np.minimum(s, np.uint64(n_shards - 1)).astype(np.int64)


def exchange_buckets(routed, counts, dist, group=None):
    """All-to-all of owner buckets.

    routed: (n, 3) int64 tensor whose rows are grouped by owner shard in rank
    order (the router's output); counts: (G,) int64 tensor of bucket sizes on
    the same device.  Returns the (m, 3) tensor of entries this rank owns.
    """
    import torch

    out_counts = torch.empty_like(counts)
    dist.all_to_all_single(out_counts, counts, group=group)
    in_splits = [int(x) for x in counts.tolist()]
    out_splits = [int(x) for x in out_counts.tolist()]
    recv = torch.empty((sum(out_splits), ENTRY_WORDS), dtype=routed.dtype, device=routed.device)
    dist.all_to_all_single(recv, routed[: sum(in_splits)].contiguous(), out_splits, in_splits, group=group)
    return recv


def global_verdict(local_conflict: bool, dist, device="cpu", group=None) -> bool:
    """Round conflictFlag over all shards: OR via all-reduce MAX on {0,1}."""
    import torch

    t = torch.tensor([1 if local_conflict else 0], dtype=torch.int32, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return bool(t.item())


class ShardedValidator:
    """Product path of one rank: CUDA routing -> exchange -> CUDA validate/apply."""

    def __init__(self, dev, world: int, shard_words: int, max_entries: int, dist, stream: int = 0):
        import torch

        self.dev, self.world, self.shard_words, self.dist = dev, world, shard_words, dist
        self.stream = stream
        self.routed = torch.empty((max_entries, ENTRY_WORDS), dtype=torch.int64, device="cuda")
        self.counts = torch.zeros(world, dtype=torch.int64, device="cuda")

    def validate(self, log, mode: int):
        """Route + exchange + validate `log` ((n, 3) int64 CUDA tensor); returns the entries applied here."""
        n = int(log.shape[0])
        if self.world == 1:
            self.dev.validate_dptr(log.data_ptr(), n, mode, self.stream)
            return n
        self.dev.route_log_dptr(log.data_ptr(), n, self.world, self.shard_words, self.routed.data_ptr(),
                                self.counts.data_ptr(), self.stream)
        recv = exchange_buckets(self.routed[:n], self.counts, self.dist)
        self.dev.validate_dptr(recv.data_ptr(), int(recv.shape[0]), mode, self.stream)
        self._keep = recv  # alive until the validation kernel has consumed it
        return int(recv.shape[0])


class PeerValidator:
    """Fused route + NVLink delivery of one rank.

    Each rank exposes a double receive arena (world regions x `cap` entries,
    two round parities) and its bucket counts; their CUDA IPC handles are
    all-gathered once.  validate() = one router launch that scatters each
    entry into its owner's arena (peer stores), a stream sync + barrier so
    every rank's deliveries of this round are complete, and the owner's
    validate/apply of its received regions.  Round parity alternates, so a
    fast rank can route round r+1 while a slow one still applies round r."""

    def __init__(self, dev, world: int, rank: int, shard_words: int, cap: int, dist, stream: int = 0):
        """Collective over all ranks; raises RuntimeError on EVERY rank if any rank
        cannot export or open the arenas (the caller then falls back to NCCL)."""
        from . import api

        self.dev, self.world, self.rank, self.shard_words, self.cap = dev, world, rank, shard_words, cap
        self.dist, self.stream, self.parity = dist, stream, 0
        self._opened = []
        self._flag = None
        try:
            ent, cnt = dev.recv_arena(world, cap)
            mine = (api.ipc_get_handle(ent), api.ipc_get_handle(cnt))
        except Exception:
            ent = cnt = mine = None
        handles = [None] * world
        dist.all_gather_object(handles, mine)
        ok = all(h is not None for h in handles)
        self.entries, self.counts = [], []
        if ok:
            try:
                for r in range(world):
                    if r == rank:
                        self.entries.append(ent)
                        self.counts.append(cnt)
                    else:
                        e = api.ipc_open_handle(handles[r][0])
                        self._opened.append(e)
                        c = api.ipc_open_handle(handles[r][1])
                        self._opened.append(c)
                        self.entries.append(e)
                        self.counts.append(c)
            except Exception:
                ok = False
        flags = [None] * world
        dist.all_gather_object(flags, ok)
        if not all(flags):
            self.close()
            raise RuntimeError("peer arenas unavailable on some rank")

    def validate(self, log, mode: int):
        """Route + deliver + validate `log` ((n, 3) int64 CUDA tensor).  With NCCL
        the round barrier is a 1-element all-reduce ordered on the validation
        stream, so nothing waits on the host; returns None then (the number of
        entries applied here is known only on the device).  With a CPU backend
        (gloo test mode) the stream is synchronized around a host barrier and
        the count is returned."""
        import torch

        n = int(log.shape[0])
        self.dev.route_to_peers_dptr(log.data_ptr(), n, self.world, self.shard_words, self.rank, self.cap,
                                     self.parity, self.entries, self.counts, self.stream)
        device_barrier = self.dist.get_backend() == "nccl"
        if device_barrier:
            st = torch.cuda.ExternalStream(self.stream) if self.stream else torch.cuda.current_stream()
            with torch.cuda.stream(st):
                if self._flag is None:
                    self._flag = torch.zeros(1, dtype=torch.int32, device="cuda")
                self.dist.all_reduce(self._flag)  # completes only after every rank's delivery kernel
            m = self.dev.apply_received(self.parity, mode, self.stream, count=False)
        else:
            torch.cuda.ExternalStream(self.stream).synchronize() if self.stream else torch.cuda.synchronize()
            self.dist.barrier()  # every rank's deliveries for this parity are complete
            m = self.dev.apply_received(self.parity, mode, self.stream)
        self.parity ^= 1
        return m

    def close(self):
        from . import api

        for p in self._opened:
            api.ipc_close(p)
        self._opened = []
