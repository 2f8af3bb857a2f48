// report_test.cpp — emitReport on fixed round reports (CPU):
// writes <prefix>.csv and <prefix>.json; tests/test_checker.py checks that the
// two hold identical values and that the summary recomputes from the rows.
#include <cstdio>
#include <vector>

#include "hetm_b200/engine.hpp"

using namespace hetm::b200;

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    std::vector<RoundReport> rs(3);
    const Outcome oc[3] = {Outcome::Commit, Outcome::DeviceAborted, Outcome::HostAborted};
    for (int i = 0; i < 3; ++i) {
        RoundReport& r = rs[i];
        r.round_id = i;
        r.outcome = oc[i];
        r.conflict = i > 0;
        r.host_commits = 1000 + 10 * i;
        r.dev_committed = 4096 - i;
        r.log_entries = 2000 + i;
        r.bytes_merge = 65536u * (i + 1);
        r.dev_batches = 1;
        r.exec_ms = 1.25 + i;
        r.validate_ms = 0.3333;
        r.merge_ms = 0.5 * (i + 1);
    }
    const std::string p = argv[1];
    emitReport(rs, "csv", p + ".csv");
    emitReport(rs, "json", p + ".json");
    bool threw = false;
    try {
        emitReport(rs, "json", "/nonexistent-dir/x.json");
    } catch (const std::runtime_error&) {
        threw = true;
    }
    std::printf("%s\n", threw ? "ok" : "io-error not raised");
    return threw ? 0 : 1;
}
