// SPDX-License-Identifier: Apache-2.0
// Conflict-free multi-GPU round schedule (host/rounds.cpp).
#pragma once
#include <cstdint>
#include <vector>

namespace ember {

struct RoundSchedule {
    uint32_t p = 0, world = 0, rounds = 0;
    std::vector<uint32_t> order;   // bucket ids (i*p + j) in global schedule order
    std::vector<uint32_t> round;   // per position in `order`: round index
    std::vector<uint32_t> rank;    // per position in `order`: GPU
    std::vector<uint32_t> holder;  // [rounds][p]: GPU holding partition x during round r
};

RoundSchedule make_rounds(uint32_t p, uint32_t world);

}  // namespace ember
