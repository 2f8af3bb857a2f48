// Compiles include/hetm_b200/hetm_gpu.hpp against the REFERENCE headers and
// exercises it: on a machine without a GPU the device open must throw (no CPU
// fallback); with a GPU it runs one small round and prints its verdict.
#include <cstdio>
#include <vector>

#include "hetm_b200/hetm_gpu.hpp"

int main() {
    try {
        hetm::b200::GpuDevice dev(1 << 12, 64);
        dev.registerKernel(HETM_KERNEL_BANK);
        std::vector<hetm_bank_tx> txs(256);
        for (std::size_t i = 0; i < txs.size(); ++i) {
            txs[i].acct[0] = i % 2048;
            txs[i].acct[1] = (i * 7 + 1) % 2048;
            txs[i].acct[2] = (i * 13 + 2) % 2048;
            txs[i].acct[3] = (i * 31 + 3) % 2048;
            txs[i].amount = 1;
        }
        auto tickets = dev.executeBatch(HETM_KERNEL_BANK, txs.data(), sizeof(hetm_bank_tx), txs.size());
        hetm::LogChunk chunk;
        chunk.entries.push_back(hetm::WriteLogEntry{3000, 7, 1});
        dev.streamChunk(chunk);
        bool conflict = dev.roundVerdict();
        std::vector<hetm::Word> host(1 << 12, 0);
        host[3000] = 7;  // the host replica already holds the host's own commits
        dev.mergeCommit(host);
        dev.mergeWait();
        bool match = true;
        for (hetm::WordIdx a : {0ull, 1ull, 7ull, 2047ull, 3000ull})
            match = match && host[a] == dev.rawRead(hetm::Replica::Dev, a);
        std::printf("device round ok: %zu tickets, conflict=%d, replicas_match=%d\n", tickets.size(), (int)conflict,
                    (int)match);
        return 0;
    } catch (const hetm::HetmError& e) {
        std::printf("HetmError: %s\n", e.what());
        return 3;
    }
}
