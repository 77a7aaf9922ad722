// moesched/balancer.hpp — drop-in re-declaration of the CPU/PCIe balancer
// (/root/reference/proj/include/moesched/balancer.hpp:11-39).
#pragma once

#include <cstdint>
#include <vector>

#include "moesched/core.hpp"

namespace moesched {

struct BalanceItem {
    std::uint32_t uid = 0;
    std::uint32_t batch = 1;
};

struct BalanceInput {
    std::vector<BalanceItem> items;
    TimeUnits t_cpu_token = 30;
    TimeUnits t_load = 100;
};

struct BalanceResult {
    std::vector<std::uint32_t> load_list;
    std::vector<std::uint32_t> cpu_list;
    TimeUnits c_load = 0;
    TimeUnits c_cpu = 0;
    TimeUnits makespan() const { return c_load > c_cpu ? c_load : c_cpu; }
};

BalanceResult balance(const BalanceInput& input);           // Algorithm 2, on the device
TimeUnits brute_force_balance(const BalanceInput& input);   // test oracle, <= 20 items

}  // namespace moesched
