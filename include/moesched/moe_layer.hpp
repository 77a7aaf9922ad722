// moesched/moe_layer.hpp — the real-layer API of the B200 build: a stack of
// MoE decode layers whose scheduling is the reference's run_layer decision
// state machine (/root/reference/proj/src/pipeline.cpp:128-344) executed on
// the device, and whose expert compute is real (router GEMV + softmax,
// grouped SwiGLU experts, shared expert, PCIe uploads of cache misses).
//
// The reference has no counterpart (it abstracts expert compute and uploads
// as t_gpu / t_load tasks, pipeline.cpp:217-266); this header adds one in the
// reference's vocabulary: the configuration is a SimConfig (core.hpp), the
// per-step outcome a RouteResult (router.hpp:38-54) plus the load / CPU
// (BA-streamed) / prefetch lists and evictions the simulator would log, and
// the counters are the pipeline's Metrics (pipeline.hpp:63-78). Errors are the
// reference's exception types (ConfigError, CacheError, std::logic_error) and a
// std::runtime_error("CUDA: ...") for device failures.
//
// Implemented in libmoesched.so over the C-ABI (include/moesched_b200.h).
#pragma once

#include <cstdint>
#include <vector>

#include "moesched/core.hpp"
#include "moesched/pipeline.hpp"
#include "moesched/router.hpp"

struct moeb_stack;

namespace moesched {

// Model dimensions of the layer arithmetic (moeb_model).
struct ModelDims {
    std::uint32_t d_model = 2048;      // multiple of 256
    std::uint32_t ffn = 1408;          // routed expert intermediate size
    std::uint32_t shared_ffn = 2816;   // fused shared experts (0: none)
    bool shared_gate = false;          // Qwen2-MoE sigmoid gate on the shared expert
    bool renormalize = false;          // Mixtral: renormalised top-k combine weights
    float routed_scale = 1.0f;         // DeepSeek routed_scaling_factor
    std::uint64_t weight_seed = 7;     // counter-based synthetic weights
};

// One (iteration, layer) decision step as the device took it.
struct StepDecision {
    std::uint64_t iteration = 0;
    std::uint32_t layer = 0;
    std::vector<std::uint8_t> resident_before;  // E entries: the snapshot the router saw (pipeline.cpp:154)
    RouteResult route;                          // per token selected / substitutions / kept_low (cls empty)
    std::vector<std::uint32_t> load_list;       // demand loads, admission order (pipeline.cpp:229-240)
    std::vector<std::uint32_t> cpu_list;        // BA-streamed experts, never admitted (pipeline.cpp:217-227)
    std::vector<std::uint32_t> prefetched;      // prefetch issues for the next layer (pipeline.cpp:325-341)
    std::vector<EvictionEvent> evictions;       // time = completion of this step
    TimeUnits completion = 0;
};

class MoeStack {
public:
    // host_pool: optional caller-owned pinned/pageable pool of every routed
    // expert ([L][E][3 * ffn * d_model] bf16 in the layout moeb_create
    // documents); nullptr = synthetic weights generated from weight_seed.
    MoeStack(const SimConfig& cfg, const ModelDims& dims, const void* host_pool = nullptr, int device = 0,
             bool record_decisions = true);
    ~MoeStack();
    MoeStack(const MoeStack&) = delete;
    MoeStack& operator=(const MoeStack&) = delete;
    MoeStack(MoeStack&& o) noexcept;
    MoeStack& operator=(MoeStack&& o) noexcept;

    // Trace-driven routing: router logits [n_steps][L][B][E] fp32 (host or
    // device memory). total_iterations bounds prefetch at the trace end.
    void set_logits_trace(const float* logits, std::uint64_t n_steps, std::uint64_t total_iterations = 0);
    // One decode step through all layers: x, y device bf16 [B][d_model].
    // Asynchronous on `stream` (a cudaStream_t; nullptr = the stack's own).
    void step(const void* x, void* y, std::uint32_t batch, void* stream = nullptr);
    void sync();
    // Prefill (prompt pass) of n_tokens tokens through all layers: x, y device
    // bf16 [n_tokens][d_model]. Plain top-k routing, the decode state is not
    // changed (moeb_prefill). Returns the bytes uploaded from the pinned pool.
    std::uint64_t prefill(const void* x, void* y, std::uint32_t n_tokens, void* stream = nullptr);
    void reset();

    Metrics metrics() const;
    std::vector<StepDecision> decisions() const;     // needs record_decisions
    std::vector<float> scores() const;               // fp32 router scores of every step [steps][B][E]
    std::vector<float> layer_outputs() const;        // fp32 [L][B][d_model] of the last step

    const SimConfig& config() const { return cfg_; }
    moeb_stack* handle() const { return h_; }

private:
    SimConfig cfg_;
    ModelDims dims_;
    moeb_stack* h_ = nullptr;
};

}  // namespace moesched
