// trace.hpp — execution traces for the P1 / P2-dagger consistency checker
// (the `checker` module), header-only C++20.
//
// Recording is toggleable (HostStm::setTrace / Engine::setTrace; nullptr =
// off) and lossless when on: every event carries its value.
// Concurrency: concurrent append with ONE global sequence —
// the seq is an atomic counter, the events land in per-thread shards so the
// host workers do not serialize on one lock; events() merges them by seq.
//
// Dump format (SPEC.md:569 External Interfaces): "HETMTRC1", u32 header
// length, the JSON header {"version": 1, "sizeWords": W, "config": {...}},
// then one length-prefixed record per event (u32 length = 40, then the
// 40-byte hetm_trace_event).  load(dump(t)) == t bit-exactly.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "hetm_b200/capi.h"

namespace hetm::b200 {

static_assert(sizeof(hetm_trace_event) == 40, "trace record is 40 bytes");

class Trace {
public:
    explicit Trace(uint64_t size_words = 0, std::string config_json = "{}")
        : size_words_(size_words), config_(std::move(config_json)) {
        for (auto& s : shards_) s = std::make_unique<Shard>();
    }
    Trace(Trace&& o) noexcept
        : size_words_(o.size_words_), config_(std::move(o.config_)), seq_(o.seq_.load()), round_(o.round_.load()) {
        for (int i = 0; i < kShards; ++i) shards_[i] = std::move(o.shards_[i]);
    }

    /// Appends one event (thread-safe); returns its seq.
    uint64_t append(uint8_t device, uint8_t kind, uint64_t tx, uint64_t addr, uint64_t value) {
        Shard& sh = *shards_[std::hash<std::thread::id>{}(std::this_thread::get_id()) % kShards];
        std::lock_guard<std::mutex> g(sh.mu);  // uncontended: one shard per thread in practice
        const uint64_t seq = seq_.fetch_add(1, std::memory_order_acq_rel);
        sh.ev.push_back(hetm_trace_event{seq, tx, addr, value, round_.load(std::memory_order_relaxed), device, kind, 0});
        if (kind == HETM_EV_SPEC_COMMIT) sh.spec.push_back({device, tx});
        return seq;
    }

    /// Round boundary: marker event, later events carry `round`.
    void beginRound(uint32_t round) {
        round_.store(round, std::memory_order_relaxed);
        append(0, HETM_EV_ROUND, 0, 0, round);
    }

    /// End of a round: every transaction that speculatively committed in it
    /// becomes FINAL_COMMIT (its device's side of the round is final) or
    /// ABORT(HETM_ABORT_ROUND).
    void finalizeRound(bool host_final, bool device_final) {
        std::vector<std::pair<uint8_t, uint64_t>> spec;
        for (auto& s : shards_) {
            std::lock_guard<std::mutex> g(s->mu);
            spec.insert(spec.end(), s->spec.begin(), s->spec.end());
            s->spec.clear();
        }
        std::sort(spec.begin(), spec.end());
        const uint32_t r = round_.load(std::memory_order_relaxed);
        for (auto& [dev, tx] : spec) {
            const bool fin = dev ? device_final : host_final;
            append(dev, fin ? HETM_EV_FINAL_COMMIT : HETM_EV_ABORT, tx, 0, fin ? (uint64_t)r : (uint64_t)HETM_ABORT_ROUND);
        }
    }

    /// All events in seq order.
    std::vector<hetm_trace_event> events() const {
        std::vector<hetm_trace_event> all;
        for (auto& s : shards_) {
            std::lock_guard<std::mutex> g(s->mu);
            all.insert(all.end(), s->ev.begin(), s->ev.end());
        }
        std::sort(all.begin(), all.end(), [](const auto& a, const auto& b) { return a.seq < b.seq; });
        return all;
    }
    uint64_t sizeWords() const { return size_words_; }
    const std::string& config() const { return config_; }

    std::string header() const {
        return "{\"version\": 1, \"sizeWords\": " + std::to_string(size_words_) + ", \"config\": " + config_ + "}";
    }

    void dump(const std::string& path) const {
        std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path.c_str(), "wb"), &std::fclose);
        if (!f) throw std::runtime_error("trace dump: cannot open " + path);
        const std::string h = header();
        const uint32_t hl = (uint32_t)h.size(), rl = (uint32_t)sizeof(hetm_trace_event);
        bool ok = std::fwrite(kMagic, 1, 8, f.get()) == 8 && std::fwrite(&hl, 4, 1, f.get()) == 1 &&
                  std::fwrite(h.data(), 1, hl, f.get()) == hl;
        for (const auto& e : events()) ok = ok && std::fwrite(&rl, 4, 1, f.get()) == 1 && std::fwrite(&e, rl, 1, f.get()) == 1;
        if (!ok) throw std::runtime_error("trace dump: short write to " + path);
    }

    /// Parses a dump; throws on a malformed file (bad magic, truncated or
    /// wrongly sized record).
    static Trace load(const std::string& path) {
        std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path.c_str(), "rb"), &std::fclose);
        if (!f) throw std::runtime_error("trace load: cannot open " + path);
        char magic[8];
        uint32_t hl = 0;
        if (std::fread(magic, 1, 8, f.get()) != 8 || std::memcmp(magic, kMagic, 8) != 0 ||
            std::fread(&hl, 4, 1, f.get()) != 1)
            throw std::runtime_error("trace load: not a HETMTRC1 file");
        std::string h(hl, '\0');
        if (std::fread(h.data(), 1, hl, f.get()) != hl) throw std::runtime_error("trace load: truncated header");
        const auto num = [&](const char* key) {
            const auto p = h.find(key);
            if (p == std::string::npos) throw std::runtime_error(std::string("trace load: header lacks ") + key);
            return std::strtoull(h.c_str() + p + std::strlen(key), nullptr, 10);
        };
        if (num("\"version\": ") != 1) throw std::runtime_error("trace load: unsupported version");
        const auto cfg = h.find("\"config\": ");
        Trace t(num("\"sizeWords\": "),
                cfg == std::string::npos ? "{}" : h.substr(cfg + 10, h.size() - cfg - 11));
        uint32_t rl = 0;
        uint64_t max_seq = 0;
        while (std::fread(&rl, 4, 1, f.get()) == 1) {
            hetm_trace_event e;
            if (rl != sizeof e || std::fread(&e, sizeof e, 1, f.get()) != 1)
                throw std::runtime_error("trace load: bad record");
            t.shards_[0]->ev.push_back(e);
            max_seq = std::max(max_seq, e.seq + 1);
        }
        t.seq_.store(max_seq);
        return t;
    }

private:
    static constexpr const char* kMagic = "HETMTRC1";
    static constexpr int kShards = 64;
    struct Shard {
        std::mutex mu;
        std::vector<hetm_trace_event> ev;
        std::vector<std::pair<uint8_t, uint64_t>> spec;  // this round's speculative commits
    };
    uint64_t size_words_;
    std::string config_;
    std::atomic<uint64_t> seq_{0};
    std::atomic<uint32_t> round_{0};
    std::unique_ptr<Shard> shards_[kShards];
};

}  // namespace hetm::b200
