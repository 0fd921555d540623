// SPDX-License-Identifier: Apache-2.0
//
// Conflict-free round schedule for multi-GPU partitioned training.
//
// A bucket (i, j) touches node partitions i and j only (Algorithm 2), so G GPUs
// can train G sets of buckets concurrently when no partition is on two GPUs at once. Rounds come
// from the circle method (round-robin tournament) over the p partitions: round r (0 <= r < p-1)
// is the perfect matching {(p-1, r)} U {((r+k) mod (p-1), (r-k) mod (p-1)) : 1 <= k < p/2}, so
// every unordered pair meets exactly once. Each GPU takes p/(2G) pairs per round and trains
// (a, b) then (b, a) for each; the self-buckets (x, x) run in round 0, where every partition is
// first resident (SURVEY §8(e) "(i, i) and (j, j) at first residency") — every GPU gets the same
// number of them, so rounds stay balanced across GPUs. Pairs are assigned to GPUs greedily to
// keep partitions where they already are (fewest NVLink handoffs): highest overlap first, ties
// to the lower pair, then the lower rank. The schedule is a pure function of (p, G).
#include <algorithm>
#include <cstdint>
#include <vector>

#include "rounds.h"

#include "ember/common.h"

namespace ember {

RoundSchedule make_rounds(uint32_t p, uint32_t world) {
    if (p == 0 || world == 0) throw ConfigError("rounds: p and world must be >= 1");
    RoundSchedule S;
    S.p = p;
    S.world = world;
    if (p == 1) {
        if (world != 1) throw ConfigError("rounds: one partition cannot be sharded over several GPUs");
        S.rounds = 1;
        S.order = {0};
        S.round = {0};
        S.rank = {0};
        S.holder = {0};
        return S;
    }
    if (p % 2) throw ConfigError("rounds: p must be even (perfect matchings of partitions)");
    const uint32_t pairs = p / 2;
    if (pairs % world) throw ConfigError("rounds: world must divide p/2 (equal pairs per GPU per round)");
    const uint32_t per = pairs / world;
    S.rounds = p - 1;
    S.holder.assign((size_t)S.rounds * p, 0);
    std::vector<uint32_t> cur(p, ~0u);  // partition -> GPU in the previous round
    for (uint32_t r = 0; r < S.rounds; ++r) {
        std::vector<std::pair<uint32_t, uint32_t>> pr;
        pr.emplace_back(std::min(p - 1, r), std::max(p - 1, r));
        for (uint32_t k = 1; k < pairs; ++k) {
            const uint32_t a = (r + k) % (p - 1), b = (r + (p - 1) - k) % (p - 1);
            pr.emplace_back(std::min(a, b), std::max(a, b));
        }
        // greedy overlap assignment
        std::vector<uint32_t> owner(pairs, ~0u), load(world, 0);
        for (uint32_t n = 0; n < pairs; ++n) {
            int best = -1, bq = 0, bg = 0;
            for (uint32_t q = 0; q < pairs; ++q) {
                if (owner[q] != ~0u) continue;
                for (uint32_t g = 0; g < world; ++g) {
                    if (load[g] == per) continue;
                    const int sc = (cur[pr[q].first] == g) + (cur[pr[q].second] == g);
                    if (sc > best) {
                        best = sc;
                        bq = (int)q;
                        bg = (int)g;
                    }
                }
            }
            owner[bq] = (uint32_t)bg;
            ++load[bg];
        }
        for (uint32_t q = 0; q < pairs; ++q) {
            cur[pr[q].first] = cur[pr[q].second] = owner[q];
            S.holder[(size_t)r * p + pr[q].first] = owner[q];
            S.holder[(size_t)r * p + pr[q].second] = owner[q];
        }
        // emit buckets rank by rank, pairs in matching order
        for (uint32_t g = 0; g < world; ++g)
            for (uint32_t q = 0; q < pairs; ++q) {
                if (owner[q] != g) continue;
                const uint32_t a = pr[q].first, b = pr[q].second;
                std::vector<uint32_t> bk;
                if (r == 0) bk.push_back(a * p + a);
                bk.push_back(a * p + b);
                bk.push_back(b * p + a);
                if (r == 0) bk.push_back(b * p + b);
                for (uint32_t id : bk) {
                    S.order.push_back(id);
                    S.round.push_back(r);
                    S.rank.push_back(g);
                }
            }
    }
    return S;
}

}  // namespace ember
