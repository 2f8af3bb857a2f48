// ref_shim.cpp — C entry points over the REFERENCE's own headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile (target `ref`) with
// -I /root/reference/proj/include into oracle/_ref/libhetm_ref.so; never
// shipped in the product path.  It lets tests/golden/make_golden.py record
// what the reference code itself computes for:
//   DetRng            det_rng.hpp:19-42
//   AccessBitmap      bitmap.hpp:94-124 (granule mapping, ceil bit count, InvalidSizeError)
//   ChunkMap          bitmap.hpp:128-158 (forEachDirty order)
//   WriteLog          write_log.hpp:31-101 (allEntries concatenates in thread order)
// The reference sources are used in place; nothing is copied into the repo.
#include <cstdint>
#include <cstring>
#include <vector>

#include "hetm/bitmap.hpp"
#include "hetm/det_rng.hpp"
#include "hetm/types.hpp"
#include "hetm/write_log.hpp"

extern "C" {

void ref_rng_next(std::uint64_t seed, std::uint64_t n, std::uint64_t* out) {
    hetm::DetRng r(seed);
    for (std::uint64_t i = 0; i < n; ++i) out[i] = r.next();
}

void ref_rng_below(std::uint64_t seed, std::uint64_t bound, std::uint64_t n, std::uint64_t* out) {
    hetm::DetRng r(seed);
    for (std::uint64_t i = 0; i < n; ++i) out[i] = r.below(bound);
}

void ref_rng_uniform(std::uint64_t seed, std::uint64_t n, double* out) {
    hetm::DetRng r(seed);
    for (std::uint64_t i = 0; i < n; ++i) out[i] = r.uniform();
}

std::uint64_t ref_splitmix64(std::uint64_t x) { return hetm::splitmix64(x); }

// Builds an AccessBitmap, sets the covering bit of every word in `addrs`,
// and returns the snapshot.  Returns the bit count, or -1 on InvalidSizeError.
// `out_words` must hold ceil(bits/64) words (query with out_words == nullptr).
long long ref_access_bitmap(std::uint64_t region_bytes, std::uint64_t gran, const std::uint64_t* addrs,
                            std::uint64_t n, std::uint64_t* out_words) {
    try {
        hetm::AccessBitmap bm(region_bytes, gran);
        for (std::uint64_t i = 0; i < n; ++i) bm.setWord(addrs[i]);
        auto snap = bm.snapshot();
        if (out_words) std::memcpy(out_words, snap.words.data(), snap.words.size() * 8);
        return static_cast<long long>(snap.nBits);
    } catch (const hetm::InvalidSizeError&) {
        return -1;
    }
}

// ChunkMap::markWordWritten for each addr; writes the dirty chunk indices in
// forEachDirty order into out (capacity max).  Returns the dirty count, -1 on
// InvalidSizeError.
long long ref_chunk_map(std::uint64_t region_bytes, std::uint64_t chunk_bytes, const std::uint64_t* addrs,
                        std::uint64_t n, std::uint64_t* out, std::uint64_t max) {
    try {
        hetm::ChunkMap cm(region_bytes, chunk_bytes);
        for (std::uint64_t i = 0; i < n; ++i) cm.markWordWritten(addrs[i]);
        std::uint64_t k = 0;
        cm.forEachDirty([&](std::size_t c) {
            if (k < max) out[k] = c;
            ++k;
        });
        return static_cast<long long>(k);
    } catch (const hetm::InvalidSizeError&) {
        return -1;
    }
}

// Appends entries[i] to thread tid[i]'s log (n_threads registered), then
// returns WriteLog::allEntries() into out (n entries).
void ref_write_log_all(const std::uint64_t* triples, const int* tid, std::uint64_t n, int n_threads,
                       std::uint64_t* out) {
    hetm::WriteLog log;
    for (int t = 0; t < n_threads; ++t) log.registerThread();
    for (std::uint64_t i = 0; i < n; ++i) {
        hetm::WriteLogEntry e{triples[3 * i], triples[3 * i + 1], triples[3 * i + 2]};
        log.append(tid[i], std::span<const hetm::WriteLogEntry>(&e, 1));
    }
    auto all = log.allEntries();
    static_assert(sizeof(hetm::WriteLogEntry) == hetm::kLogEntryWireBytes);
    std::memcpy(out, all.data(), all.size() * sizeof(hetm::WriteLogEntry));
}

std::uint64_t ref_log_entry_bytes() { return sizeof(hetm::WriteLogEntry); }

}  // extern "C"
