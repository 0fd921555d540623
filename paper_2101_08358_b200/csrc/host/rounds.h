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
    // per position in `order`: 1 if the bucket's partitions leave their GPU after this round
    // (make_rounds_overlap trains those buckets first; empty for make_rounds)
    std::vector<uint8_t> early;
};

RoundSchedule make_rounds(uint32_t p, uint32_t world);
// Overlapped schedule (p a power of two, world <= p/4): every GPU trains one departing and one
// staying pair per coset it holds, the departing pair first, so the departing partitions' handoff
// runs under the staying pair's compute (rounds.cpp).
RoundSchedule make_rounds_overlap(uint32_t p, uint32_t world);

}  // namespace ember
