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

// ---- overlapped (coset) schedule ---------------------------------------------------------------
// Partitions are the vectors of GF(2)^k (p = 2^k). The 1-factorisation M_v = {{x, x ^ v}} over the
// p-1 nonzero v covers every unordered pair once; round r uses M_{v_r}. During round r every GPU
// holds whole cosets x + span{v_{r-1}, v_r} (4 partitions = two pairs of M_{v_r}); a linear form
// f_r with f_r(v_{r-1}) = 1, f_r(v_r) = 0, f_r(v_{r+1}) = 1 (it exists for any three distinct
// nonzero vectors) splits each coset into a departing pair (f_r = 1) and a staying pair (f_r = 0).
// M_{v_{r+1}} pairs every staying partition with a departing one, and the next round's cosets
// x + span{v_r, v_{r+1}} are exactly {staying pair} U {staying pair ^ v_{r+1}}: each GPU keeps its
// staying pairs and receives, for each, the departing pair at staying ^ v_{r+1}. Training the
// departing pair's buckets first lets those two partitions travel while the staying pair trains.
// The sequence is cyclic (v_{-1} = v_{p-2}), so the last round hands over to round 0 of the next
// epoch the same way. Self-buckets (x, x) run in round 0 with their pair.
namespace {
uint32_t parity(uint32_t x) { return (uint32_t)__builtin_popcount(x) & 1u; }
}  // namespace

RoundSchedule make_rounds_overlap(uint32_t p, uint32_t world) {
    if (p < 4 || (p & (p - 1))) throw ConfigError("overlapped rounds: p must be a power of two >= 4");
    if (world == 0 || (p / 4) % world) throw ConfigError("overlapped rounds: world must divide p/4");
    RoundSchedule S;
    S.p = p;
    S.world = world;
    S.rounds = p - 1;
    const uint32_t R = p - 1;
    // v_r: the nonzero vectors in Gray-code order (consecutive rounds differ by one bit flip)
    std::vector<uint32_t> v(R);
    for (uint32_t r = 0; r < R; ++r) v[r] = (r + 1) ^ ((r + 1) >> 1);
    auto V = [&](int64_t r) { return v[(size_t)(((r % R) + R) % R)]; };
    std::vector<uint32_t> form(R);
    for (uint32_t r = 0; r < R; ++r) {
        uint32_t w = 1;
        for (; w < p; ++w)
            if (parity(w & V((int64_t)r - 1)) == 1 && parity(w & V(r)) == 0 && parity(w & V((int64_t)r + 1)) == 1) break;
        if (w == p) throw EmberError("overlapped rounds: no separating form (internal)");
        form[r] = w;
    }
    S.holder.assign((size_t)R * p, 0);
    // round 0: cosets of span{v_{-1}, v_0}, ordered by their least element, dealt to GPUs in blocks
    {
        std::vector<uint32_t> seen(p, ~0u);
        uint32_t c = 0;
        const uint32_t a = V(-1), b = V(0), per = (p / 4) / world;
        for (uint32_t x = 0; x < p; ++x) {
            if (seen[x] != ~0u) continue;
            const uint32_t g = c++ / per;
            for (uint32_t y : {x, x ^ a, x ^ b, x ^ a ^ b}) seen[y] = g;
        }
        for (uint32_t x = 0; x < p; ++x) S.holder[x] = seen[x];
    }
    for (uint32_t r = 0; r < R; ++r) {
        const uint32_t* hold = &S.holder[(size_t)r * p];
        const uint32_t vr = V(r);
        for (uint32_t g = 0; g < world; ++g)
            for (int pass = 0; pass < 2; ++pass)  // departing pairs (f_r = 1) first, then staying
                for (uint32_t x = 0; x < p; ++x) {
                    const uint32_t y = x ^ vr;
                    if (hold[x] != g || y < x || parity(form[r] & x) != (pass == 0 ? 1u : 0u)) continue;
                    std::vector<uint32_t> bk;
                    if (r == 0) bk.push_back(x * p + x);
                    bk.push_back(x * p + y);
                    bk.push_back(y * p + x);
                    if (r == 0) bk.push_back(y * p + y);
                    for (uint32_t id : bk) {
                        S.order.push_back(id);
                        S.round.push_back(r);
                        S.rank.push_back(g);
                        S.early.push_back(pass == 0 ? 1 : 0);
                    }
                }
        if (r + 1 < R) {  // staying pairs keep their GPU; departing ones go to staying ^ v_{r+1}
            uint32_t* next = &S.holder[(size_t)(r + 1) * p];
            const uint32_t vn = V(r + 1);
            for (uint32_t x = 0; x < p; ++x)
                if (parity(form[r] & x) == 0) next[x] = next[x ^ vn] = hold[x];
        }
    }
    return S;
}

}  // namespace ember
