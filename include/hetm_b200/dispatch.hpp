// dispatch.hpp — the device submission queue and the GPU-controller launch
// rule (deviceControllerPoll; "GPU-controller",
// launch when the queue "contains a sufficient number of requests to feed the
// kernel"), header-only C++20.
//
// Producers submit device transactions (any record type: hetm_bank_tx,
// hetm_rw_tx, hetm_cache_tx) from any thread; the GPU-controller polls:
// with >= batch_size requests queued it dequeues EXACTLY batch_size, in FIFO
// order, into a batch; with fewer it launches nothing — unless the optional
// max-wait knob (SPEC.md:501 open question) is set and the oldest queued
// request has waited that long, which releases the partial batch.  Every
// submitted request leaves the queue exactly once.  Affinity queues and
// host/shared-queue stealing are the host-side dispatch module, out of scope
// (DESIGN.md §8).
#pragma once

#include <chrono>
#include <cstdint>
#include <deque>
#include <functional>
#include <mutex>
#include <span>
#include <vector>

#include "hetm_b200/engine.hpp"

namespace hetm::b200 {

template <class Rec>
class DeviceQueue {
public:
    using Clock = std::chrono::steady_clock;

    explicit DeviceQueue(uint64_t batch_size, std::chrono::microseconds max_wait = std::chrono::microseconds(0))
        : batch_(batch_size), max_wait_(max_wait) {}

    void submit(const Rec& r) {
        std::lock_guard<std::mutex> g(mu_);
        q_.push_back({r, Clock::now()});
    }
    void submit(std::span<const Rec> rs) {
        const auto now = Clock::now();
        std::lock_guard<std::mutex> g(mu_);
        for (const Rec& r : rs) q_.push_back({r, now});
    }
    uint64_t size() const {
        std::lock_guard<std::mutex> g(mu_);
        return q_.size();
    }
    uint64_t batchSize() const { return batch_; }

    /// deviceControllerPoll: true and `out` = the next batch (exactly
    /// batch_size requests, FIFO) when enough are queued, or the partial batch
    /// once the oldest request has waited max_wait (if set); false otherwise.
    bool poll(std::vector<Rec>& out) {
        std::lock_guard<std::mutex> g(mu_);
        uint64_t take = 0;
        if (q_.size() >= batch_) take = batch_;
        else if (max_wait_.count() > 0 && !q_.empty() && Clock::now() - q_.front().t >= max_wait_) take = q_.size();
        if (!take) return false;
        out.clear();
        out.reserve(take);
        for (uint64_t k = 0; k < take; ++k) {
            out.push_back(q_.front().r);
            q_.pop_front();
        }
        return true;
    }

    /// An Engine::BatchSource that launches one batch per successful poll and
    /// ends the round's execution phase once the rule launches nothing (or
    /// after max_batches).  `buf` / `tickets` hold the batch during its launch.
    Engine::BatchSource source(std::vector<Rec>& buf, std::vector<uint64_t>& tickets, uint32_t max_batches = ~0u) {
        return [this, &buf, &tickets, max_batches](uint32_t k, Engine::Batch& b) {
            if (k >= max_batches || !poll(buf)) return false;
            tickets.assign(buf.size(), ~0ull);
            b = Engine::Batch{buf.data(), buf.size(), tickets.data()};
            return true;
        };
    }

private:
    struct Item {
        Rec r;
        Clock::time_point t;
    };
    const uint64_t batch_;
    const std::chrono::microseconds max_wait_;
    mutable std::mutex mu_;
    std::deque<Item> q_;
};

}  // namespace hetm::b200
