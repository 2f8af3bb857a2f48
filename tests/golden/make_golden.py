"""Generate tests/golden/ref_vectors.json from the REFERENCE's own headers.

Run here (where /root/reference exists):
    make -C oracle ref && python tests/golden/make_golden.py
The shim oracle/ref_shim.cpp is compiled against
/root/reference/proj/include/hetm/{det_rng,bitmap,write_log,types}.hpp in
place; the vectors it records pin the oracle (tests/test_oracle.py) and the
product's generators/bitmap layout on machines without /root/reference.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "ref_vectors.json")


def main():
    ref = oracle.load_ref()
    if ref is None:
        raise SystemExit("oracle/_ref/libhetm_ref.so missing: run `make -C oracle ref` where /root/reference exists")
    P = oracle.P
    g = {"source": "reference headers /root/reference/proj/include/hetm (det_rng.hpp, bitmap.hpp, write_log.hpp)",
         "generator": "tests/golden/make_golden.py via oracle/ref_shim.cpp"}

    # DetRng (det_rng.hpp:19-42)
    rng = []
    for seed in [0, 1, 2, 42, 0xDEADBEEF, 2**64 - 1]:
        nxt = np.empty(16, np.uint64); ref.ref_rng_next(seed, 16, P(nxt))
        rec = {"seed": seed, "next": [int(x) for x in nxt], "below": {}}
        for bound in [1, 3, 100, 1 << 20, 1 << 27, 1 << 33, 2**64 - 1]:
            b = np.empty(16, np.uint64); ref.ref_rng_below(seed, bound, 16, P(b))
            rec["below"][str(bound)] = [int(x) for x in b]
        u = np.empty(8, np.float64); ref.ref_rng_uniform(seed, 8, P(u))
        rec["uniform"] = [float(x) for x in u]
        rng.append(rec)
    g["rng"] = rng
    g["splitmix64"] = [[x, int(ref.ref_splitmix64(x))] for x in [0, 1, 12345, 2**63, 2**64 - 1]]

    # AccessBitmap (bitmap.hpp:94-124)
    cases = [
        ("spec_209_rs", 512, 8, [0, 1]),          # SPEC.md:209 RS {0,1}
        ("spec_209_ws", 512, 8, [1]),             # SPEC.md:209 WS {1}
        ("false_positive_1k", 1 << 20, 1024, [0]),  # SPEC.md:641 geometry
        ("ceil_800_1024", 800, 1024, []),
        ("invalid_gran_12", 4096, 12, [0]),
        ("invalid_gran_4", 4096, 4, [0]),
    ]
    r = np.random.default_rng(7)
    for gran in [8, 64, 1024, 4096]:
        W = 1 << 16
        addrs = r.integers(0, W, 2000, dtype=np.uint64).tolist()
        cases.append((f"random_w{W}_g{gran}", W * 8, gran, addrs))
    cases.append(("tail_odd_region", 8 * 1000 + 8, 1024, [0, 999, 1000]))
    bm = []
    for name, region, gran, addrs in cases:
        a = np.array(addrs, np.uint64)
        nbits = ref.ref_access_bitmap(region, gran, P(a) if a.size else None, a.size, None)
        rec = {"name": name, "region_bytes": region, "gran": gran, "addrs": [int(x) for x in addrs], "nbits": int(nbits)}
        if nbits >= 0:
            words = np.zeros((nbits + 63) // 64, np.uint64)
            ref.ref_access_bitmap(region, gran, P(a) if a.size else None, a.size, P(words))
            rec["words"] = [int(x) for x in words]
        bm.append(rec)
    g["access_bitmap"] = bm

    # ChunkMap (bitmap.hpp:128-158)
    cm = []
    for name, region, chunk, addrs in [
        ("one_word", 1 << 20, 16384, [7]),
        ("adjacent", 1 << 20, 16384, [0, 2048]),
        ("separated", 1 << 20, 16384, [0, 4096]),
        ("invalid_12000", 1 << 20, 12000, [0]),
        ("random", (1 << 16) * 8, 16384, r.integers(0, 1 << 16, 300).tolist()),
        ("tail", 8 * 5000, 16384, [4999, 0]),
    ]:
        a = np.array(addrs, np.uint64)
        out = np.zeros(4096, np.uint64)
        k = ref.ref_chunk_map(region, chunk, P(a), a.size, P(out), out.size)
        cm.append({"name": name, "region_bytes": region, "chunk": chunk, "addrs": [int(x) for x in addrs],
                   "dirty": None if k < 0 else [int(x) for x in out[:k]]})
    g["chunk_map"] = cm

    # WriteLog::allEntries order (write_log.hpp:74-82)
    n, T = 40, 3
    tid = r.integers(0, T, n).astype(np.int32)
    trip = np.zeros((n, 3), np.uint64)
    trip[:, 0] = r.integers(0, 1000, n)
    trip[:, 1] = r.integers(0, 2**62, n, dtype=np.uint64)
    trip[:, 2] = np.arange(1, n + 1)
    out = np.zeros((n, 3), np.uint64)
    ref.ref_write_log_all(P(trip), P(tid), n, T, P(out))
    g["write_log"] = {"threads": T, "tid": tid.tolist(), "entries": trip.tolist(), "all_entries": out.tolist()}
    g["log_entry_bytes"] = int(ref.ref_log_entry_bytes())

    with open(OUT, "w") as f:
        json.dump(g, f, indent=0)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()
