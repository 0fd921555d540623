// SPDX-License-Identifier: Apache-2.0
//
// Multi-GPU round loop (Algorithm 2).
//
// Every rank runs the rounds of a RoundSchedule (host/rounds.cpp) in lockstep: the relation
// all-reduce is a collective, so each round takes max-over-ranks of its batch count steps, a rank
// out of batches taking idle steps (zero relation gradient, same all-reduce). Batches are
// consecutive slices of each bucket, buckets in schedule order.
//
// Handoffs. After round r the partitions whose holder changes move by one P2P group per rank.
// The group is issued at ONE lockstep point on every rank (so host-blocking transports and a
// second NCCL communicator are both deadlock-free): right after the step at which every rank has
// finished its last batch that touches a departing partition. With the overlapped (coset)
// schedule those batches are the round's early buckets, so the copy runs on the copy stream
// while the staying pair trains; with the circle schedule it is the end of the round. The next
// round's first step waits for the arrivals (RankOps::acquire).
#include "dist_driver.h"

#include <algorithm>
#include <stdexcept>

#include "ember/common.h"

namespace ember {

DistDriver::DistDriver(RoundSchedule S, const uint64_t* offsets, uint32_t batch_size, uint32_t rank)
    : S_(std::move(S)), rank_(rank) {
    if (!offsets) throw ConfigError("dist: bucket offsets are required");
    if (batch_size == 0) throw ConfigError("dist: batch size must be >= 1");
    if (rank >= S_.world) throw ConfigError("dist: rank out of range");
    const uint32_t p = S_.p, R = S_.rounds, G = S_.world;
    lists_.assign((size_t)R * G, {});
    for (size_t pos = 0; pos < S_.order.size(); ++pos) {
        const uint32_t id = S_.order[pos], i = id / p, j = id % p;
        const uint64_t lo = offsets[id], hi = offsets[id + 1];
        if (hi < lo) throw ConfigError("dist: bucket offsets must be non-decreasing");
        auto& L = lists_[(size_t)S_.round[pos] * G + S_.rank[pos]];
        uint32_t k = 0;
        for (uint64_t b0 = lo; b0 < hi; b0 += batch_size, ++k)
            L.push_back(BatchRef{(uint32_t)pos, i, j, k, lo, hi, b0 - lo, (uint32_t)std::min<uint64_t>(batch_size, hi - b0)});
    }
    steps_.assign(R, 0);
    handoff_.assign(R, 0);
    for (uint32_t r = 0; r < R; ++r) {
        const uint32_t* now = &S_.holder[(size_t)r * p];
        const uint32_t* nxt = &S_.holder[(size_t)((r + 1) % R) * p];
        uint32_t last = 0;
        for (uint32_t g = 0; g < G; ++g) {
            const auto& L = lists_[(size_t)r * G + g];
            steps_[r] = std::max<uint32_t>(steps_[r], (uint32_t)L.size());
            for (uint32_t s = 0; s < L.size(); ++s)
                if (nxt[L[s].i] != now[L[s].i] || nxt[L[s].j] != now[L[s].j]) last = std::max(last, s + 1);
        }
        handoff_[r] = last;
    }
    // a handoff needs a step to follow: rounds without batches still hand over at their end
    for (uint32_t r = 0; r < R; ++r)
        if (!moves(r).empty() && handoff_[r] == 0) handoff_[r] = steps_[r];
}

uint64_t DistDriver::total_steps() const {
    uint64_t n = 0;
    for (uint32_t s : steps_) n += s;
    return n;
}

std::vector<Move> DistDriver::moves(uint32_t r) const {
    const uint32_t p = S_.p, R = S_.rounds;
    const uint32_t* now = &S_.holder[(size_t)r * p];
    const uint32_t* nxt = &S_.holder[(size_t)((r + 1) % R) * p];
    std::vector<Move> m;
    for (uint32_t x = 0; x < p; ++x)
        if (now[x] != nxt[x]) m.push_back(Move{x, now[x], nxt[x]});
    return m;
}

DistReport DistDriver::run(RankOps& ops, uint64_t epoch, uint64_t first, uint64_t count) const {
    DistReport rep;
    const uint32_t R = S_.rounds, G = S_.world;
    const uint64_t end = count == ~0ull ? total_steps() : std::min(total_steps(), first + count);
    uint64_t base = 0;  // lockstep index of round r's first step
    for (uint32_t r = 0; r < R && base < end; base += steps_[r], ++r) {
        const uint64_t rb = base, re = base + steps_[r];
        if (re <= first) continue;
        if (rb >= first) {  // entering round r: its arrivals must be usable
            std::vector<uint32_t> arrived;
            for (const Move& m : moves((r + R - 1) % R))
                if (m.dst == rank_) arrived.push_back(m.part);
            if (!arrived.empty()) ops.acquire(r, arrived);  // (ops ignore parts with no pending receive)
        }
        const auto& mine = lists_[(size_t)r * G + rank_];
        std::vector<Move> mv;
        for (const Move& m : moves(r))
            if (m.src == rank_ || m.dst == rank_) mv.push_back(m);
        if (steps_[r] == 0 && !moves(r).empty() && rb >= first) {  // a round without batches still hands over
            if (!mv.empty()) ops.send_recv(r, mv);
            ++rep.handoffs;
            rep.moved_partitions += mv.size();
        }
        for (uint64_t t = std::max(rb, first); t < std::min(re, end); ++t) {
            const uint32_t s = (uint32_t)(t - rb);
            if (s < mine.size()) {
                ops.step(&mine[s], epoch);
                ++rep.batches;
                rep.edges += mine[s].nb;
            } else {
                ops.step(nullptr, epoch);
            }
            ++rep.steps;
            if (s + 1 == handoff_[r] && !moves(r).empty()) {
                if (!mv.empty()) ops.send_recv(r, mv);
                ++rep.handoffs;
                rep.moved_partitions += mv.size();
                if (handoff_[r] < steps_[r]) ++rep.early_handoffs;
            }
        }
    }
    return rep;
}

}  // namespace ember
