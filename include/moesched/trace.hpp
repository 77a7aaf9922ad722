// moesched/trace.hpp — drop-in re-declaration of the gate-trace workload API
// (/root/reference/proj/include/moesched/trace.hpp:17-62).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "moesched/core.hpp"

namespace moesched {

struct SkewProfile {
    double hot_fraction = 0.125;
    double hot_mass = 0.8;
    double persistence = 0.92;
    double concentration = 1.5;
};

struct TraceIteration {
    std::vector<std::vector<std::vector<double>>> scores;     // [layer][token][E]
    std::vector<std::vector<std::vector<double>>> predicted;  // empty inner = not supplied
    bool operator==(const TraceIteration&) const = default;
};

struct GateTrace {
    ModelShape shape;
    std::vector<TraceIteration> iterations;
    bool operator==(const GateTrace&) const = default;
};

GateTrace generate_trace(const ModelShape& shape, const SkewProfile& profile, std::uint64_t iterations,
                         std::uint64_t seed);
void save_trace(const GateTrace& trace, const std::string& path);
GateTrace load_trace(const std::string& path);
std::vector<double> reuse_curve(const GateTrace& trace);
std::string fingerprint_file(const std::string& path);
std::string fingerprint_bytes(const std::string& bytes);

}  // namespace moesched
