// engine_host.h — host helpers shared by the engine and stack translation units.
#pragma once

#include <string>
#include <vector>

#include "../../include/moesched_b200.h"
#include "engine.cuh"

namespace moeb {

DevCfg make_dev_cfg(const moeb_config& c);
void validate(const moeb_config& c);
void init_layers(const DevCfg& cfg, int32_t init_fill, uint64_t seed, std::vector<LayerState>& out);
void metrics_from_counters(moeb_metrics& m, const Counters& c, uint64_t iters, uint64_t total);
std::string steps_json(const StepRec* steps, const TokRec* toks, size_t n, uint32_t B);

}  // namespace moeb
