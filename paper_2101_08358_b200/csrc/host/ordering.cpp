// SPDX-License-Identifier: Apache-2.0
//
// Edge-bucket orderings (BETA/elimination, Hilbert, Hilbert-symmetric, random) and the
// Belady replay that turns a bucket sequence into a buffer trace.
//
// Behaviour follows the reference's proj/src/ordering.cpp (elimination :185-298,
// Belady replay :94-159, Hilbert :300-365, random :367-382, formulas :163-183,
// simulate_io :394-401) and SPEC.md:208-294; outputs are bit-identical for every
// (kind, p, c, seed) — tests/test_ordering.py diffs them against the reference
// compiled in place. The structure here is our own: the elimination construction is a
// small state machine over "rounds", and the replay keeps residents in a bitmap.
#include "ember/ordering.h"

#include <algorithm>
#include <numeric>

namespace ember {

std::string to_string(OrderingKind kind) {
    static const char* const names[] = {"elimination", "hilbert", "hilbert_symmetric", "random"};
    const int k = static_cast<int>(kind);
    return (k >= 0 && k < 4) ? names[k] : "unknown";
}

OrderingKind ordering_kind_from_string(const std::string& name) {
    if (name == "elimination" || name == "beta") return OrderingKind::Elimination;
    if (name == "hilbert") return OrderingKind::Hilbert;
    if (name == "hilbert_symmetric" || name == "hilbertsymmetric") return OrderingKind::HilbertSymmetric;
    if (name == "random") return OrderingKind::Random;
    throw ConfigError("unknown ordering kind: " + name);
}

std::uint64_t OrderingPlan::next_use_after(PartitionId part, std::uint64_t step) const {
    const std::vector<std::uint32_t>& uses = partition_use_steps.at(part);
    const auto hit = std::upper_bound(uses.begin(), uses.end(), step,
                                      [](std::uint64_t s, std::uint32_t u) { return s < u; });
    return hit == uses.end() ? kNeverUsed : *hit;
}

// Structural check of a plan, one pass per invariant: (1) the sequence is a permutation of
// the p x p buckets, (2) every buffer state fits in c slots, is sorted, and each state follows
// its predecessor by exactly the recorded swap, (3) the per-bucket state index never goes
// backwards and names a state holding both partitions of the bucket.
void OrderingPlan::validate() const {
    auto fail = [](const std::string& what) { throw EmberError("invalid ordering plan: " + what); };
    const std::uint64_t total = num_buckets();
    if (bucket_sequence.size() != total || bucket_state.size() != total)
        fail("expected " + std::to_string(total) + " buckets and state indices, got " +
             std::to_string(bucket_sequence.size()) + " / " + std::to_string(bucket_state.size()));

    std::vector<bool> seen(total, false);
    for (std::uint64_t t = 0; t < total; ++t) {
        const BucketId b = bucket_sequence[t];
        if (b.i >= p || b.j >= p) fail("bucket at step " + std::to_string(t) + " names a partition >= p");
        const std::uint64_t cell = static_cast<std::uint64_t>(b.i) * p + b.j;
        if (seen[cell]) fail("bucket at step " + std::to_string(t) + " appears twice");
        seen[cell] = true;
    }

    if (buffer_states.size() != swap_events.size() + 1 || swap_count != swap_events.size())
        fail("swap bookkeeping disagrees (states " + std::to_string(buffer_states.size()) + ", events " +
             std::to_string(swap_events.size()) + ", swap_count " + std::to_string(swap_count) + ")");
    // Membership bitmap of the current state; a legal transition clears exactly the evicted
    // partition and sets exactly the admitted one.
    std::vector<std::uint8_t> held(p, 0);
    for (std::size_t k = 0; k < buffer_states.size(); ++k) {
        const auto& st = buffer_states[k];
        if (st.size() > c) fail("state " + std::to_string(k) + " holds more than c partitions");
        for (std::size_t q = 0; q < st.size(); ++q)
            if (st[q] >= p || (q > 0 && st[q] <= st[q - 1]))
                fail("state " + std::to_string(k) + " is not a sorted set of partition ids");
        if (k == 0) {
            for (PartitionId x : st) held[x] = 1;
            continue;
        }
        const SwapEvent& ev = swap_events[k - 1];
        if (ev.evicted >= p || ev.admitted >= p || !held[ev.evicted] || held[ev.admitted])
            fail("swap " + std::to_string(k - 1) + " does not apply to state " + std::to_string(k - 1));
        held[ev.evicted] = 0;
        held[ev.admitted] = 1;
        std::size_t n_held = 0;
        for (PartitionId x = 0; x < p; ++x) n_held += held[x];
        bool same = n_held == st.size();
        for (PartitionId x : st) same = same && held[x];
        if (!same) fail("state " + std::to_string(k) + " is not state " + std::to_string(k - 1) + " after its swap");
    }

    std::uint32_t prev = 0;
    for (std::uint64_t t = 0; t < total; ++t) {
        const std::uint32_t s = bucket_state[t];
        if (s >= buffer_states.size() || s < prev)
            fail("state index of step " + std::to_string(t) + " is out of range or goes backwards");
        prev = s;
        const auto& st = buffer_states[s];
        const BucketId b = bucket_sequence[t];
        if (!std::binary_search(st.begin(), st.end(), b.i) || !std::binary_search(st.begin(), st.end(), b.j))
            fail("step " + std::to_string(t) + " runs a bucket whose partitions are not both buffered");
    }
}

namespace {

// Accepted (p, c): p >= 1 and 1 <= c <= p, with c >= 2 as soon as there are off-diagonal
// buckets (p > 1), since a bucket (i, j) needs i and j resident together.
void require_valid_pc(std::uint32_t p, std::uint32_t c) {
    if (p == 0) throw ConfigError("ordering needs at least one partition (p = 0)");
    if (c > p) throw ConfigError("ordering buffer capacity c = " + std::to_string(c) + " exceeds p = " + std::to_string(p));
    if (c < 2 && p > 1) throw ConfigError("ordering with p > 1 needs a buffer of at least 2 partitions");
    if (c == 0) throw ConfigError("ordering buffer capacity c must be positive");
}

// Belady replay (furthest next use, ties to the lower id) of plan.bucket_sequence into a
// capacity-c buffer; the device partition buffer replays the same decisions.
void replay_with_belady(OrderingPlan& plan) {
    const std::uint32_t p = plan.p, c = plan.c;
    const std::uint64_t steps = plan.num_buckets();

    plan.partition_use_steps.assign(p, {});
    for (std::uint64_t t = 0; t < steps; ++t) {
        const BucketId b = plan.bucket_sequence[t];
        plan.partition_use_steps[b.i].push_back(static_cast<std::uint32_t>(t));
        if (b.i != b.j) plan.partition_use_steps[b.j].push_back(static_cast<std::uint32_t>(t));
    }
    plan.buffer_states.clear();
    plan.swap_events.clear();
    plan.admission_schedule.clear();
    plan.bucket_state.assign(steps, 0);

    std::vector<std::uint8_t> resident(p, 0);
    std::uint32_t loaded = 0;
    auto snapshot = [&] {
        std::vector<PartitionId> st;
        for (PartitionId x = 0; x < p; ++x)
            if (resident[x]) st.push_back(x);
        plan.buffer_states.push_back(std::move(st));
    };

    for (std::uint64_t t = 0; t < steps; ++t) {
        const BucketId b = plan.bucket_sequence[t];
        const PartitionId wanted[2] = {b.i, b.j};
        for (PartitionId need : wanted) {
            if (resident[need]) continue;
            plan.admission_schedule.push_back(need);
            if (loaded < c) {
                resident[need] = 1;
                if (++loaded == c) snapshot();
                continue;
            }
            bool found = false;
            PartitionId victim = 0;
            std::uint64_t furthest = 0;
            for (PartitionId x = 0; x < p; ++x) {
                if (!resident[x] || x == b.i || x == b.j) continue;
                const std::uint64_t nu = plan.next_use_after(x, t);
                if (!found || nu > furthest) {
                    found = true;
                    victim = x;
                    furthest = nu;
                }
            }
            if (!found) throw EmberError("Belady replay: every buffered partition is needed by the current bucket (c too small)");
            resident[victim] = 0;
            resident[need] = 1;
            plan.swap_events.push_back({static_cast<std::uint32_t>(t), victim, need});
            snapshot();
        }
        plan.bucket_state[t] =
            plan.buffer_states.empty() ? 0u : static_cast<std::uint32_t>(plan.buffer_states.size() - 1);
    }
    if (plan.buffer_states.empty()) snapshot();
    plan.swap_count = plan.swap_events.size();
}

// The elimination (BETA) construction of PAPER.md §4.1 / Fig. 5:
// fix c-1 residents, stream every other unretired partition through the free slot,
// retire the fixed ones, repeat. All random choices come from one Rng in a fixed order.
class Eliminator {
   public:
    Eliminator(std::uint32_t p, std::uint32_t c, std::uint64_t seed, std::vector<BucketId>& out)
        : p_(p), c_(c), rng_(mix_seed(seed, 0x0e11u)), done_(static_cast<std::size_t>(p) * p, 0), out_(out) {}

    void run() {
        std::vector<PartitionId> everyone(p_);
        std::iota(everyone.begin(), everyone.end(), 0u);
        if (p_ == c_) {
            emit_pairs(everyone);
            return;
        }
        std::vector<PartitionId> alive = everyone;  // unretired, ascending
        std::vector<PartitionId> buffer = rng_.sample_without_replacement(alive, c_);
        for (;;) {
            emit_pairs(buffer);
            if (alive.size() <= c_) return;

            const std::vector<PartitionId> fixed = rng_.sample_without_replacement(buffer, c_ - 1);
            std::vector<std::uint8_t> is_fixed(p_, 0), in_buffer(p_, 0);
            for (PartitionId f : fixed) is_fixed[f] = 1;
            for (PartitionId x : buffer) in_buffer[x] = 1;
            PartitionId last_slot = 0;
            for (PartitionId x : buffer)
                if (!is_fixed[x]) last_slot = x;

            std::vector<PartitionId> stream;
            for (PartitionId u : alive)
                if (!in_buffer[u]) stream.push_back(u);
            rng_.shuffle(stream);
            for (PartitionId s : stream) {
                last_slot = s;
                std::vector<PartitionId> now = fixed;
                now.push_back(s);
                emit_pairs(now);
            }

            std::vector<PartitionId> survivors;
            for (PartitionId u : alive)
                if (!is_fixed[u]) survivors.push_back(u);
            alive.swap(survivors);

            std::vector<PartitionId> others;
            for (PartitionId u : alive)
                if (u != last_slot) others.push_back(u);
            buffer.assign(1, last_slot);
            if (alive.size() >= c_) {
                for (PartitionId f : rng_.sample_without_replacement(others, c_ - 1)) admit(buffer, f);
                continue;  // next round starts from this buffer
            }
            rng_.shuffle(others);  // terminal round: the leftovers fit together
            for (PartitionId u : others) admit(buffer, u);
            return;
        }
    }

   private:
    void admit(std::vector<PartitionId>& buffer, PartitionId x) {
        buffer.push_back(x);
        emit_pairs(buffer);  // first co-residency processing
    }

    // All not-yet-emitted buckets among `parts`, lexicographic.
    void emit_pairs(std::vector<PartitionId> parts) {
        std::sort(parts.begin(), parts.end());
        for (PartitionId i : parts)
            for (PartitionId j : parts) {
                std::uint8_t& cell = done_[static_cast<std::size_t>(i) * p_ + j];
                if (cell) continue;
                cell = 1;
                out_.push_back({i, j});
            }
    }

    std::uint32_t p_, c_;
    Rng rng_;
    std::vector<std::uint8_t> done_;
    std::vector<BucketId>& out_;
};

std::vector<BucketId> hilbert_walk(std::uint32_t p) {
    std::uint32_t side = 1;
    while (side < p) side <<= 1;
    std::vector<BucketId> cells;
    cells.reserve(static_cast<std::size_t>(p) * p);
    const std::uint64_t n2 = static_cast<std::uint64_t>(side) * side;
    for (std::uint64_t d = 0; d < n2; ++d) {
        const auto xy = hilbert_d2xy(side, d);
        if (xy.first < p && xy.second < p) cells.push_back({xy.first, xy.second});
    }
    return cells;
}

OrderingPlan empty_plan(OrderingKind kind, std::uint32_t p, std::uint32_t c, std::uint64_t seed) {
    OrderingPlan plan;
    plan.kind = kind;
    plan.p = p;
    plan.c = c;
    plan.seed = seed;
    plan.bucket_sequence.reserve(static_cast<std::size_t>(p) * p);
    return plan;
}

}  // namespace

std::uint64_t lower_bound_swaps(std::uint32_t p, std::uint32_t c) {
    if (c == 0 || c > p) throw ConfigError("lower_bound_swaps: c must lie in [1, p]");
    if (p == c) return 0;
    if (c == 1) throw ConfigError("lower_bound_swaps: with p > 1 a single-slot buffer never holds a pair");
    const std::uint64_t pairs_left = static_cast<std::uint64_t>(p) * (p - 1) / 2 - static_cast<std::uint64_t>(c) * (c - 1) / 2;
    return (pairs_left + c - 2) / (c - 1);  // ceil(pairs_left / (c-1)), §4.1
}

std::uint64_t elimination_swap_formula(std::uint32_t p, std::uint32_t c) {
    if (c == 0 || c > p) throw ConfigError("elimination_swap_formula: c must lie in [1, p]");
    if (p == c) return 0;
    if (c == 1) throw ConfigError("elimination_swap_formula: with p > 1 a single-slot buffer never holds a pair");
    // (p-c) + (x+1)[(p-c) - x(c-1)/2], x = floor((p-c)/(c-1)), evaluated in half units
    const std::uint64_t gap = p - c;
    const std::uint64_t x = gap / (c - 1);
    return (2 * gap + (x + 1) * (2 * gap - x * (c - 1))) / 2;
}

OrderingPlan elimination_order(std::uint32_t p, std::uint32_t c, std::uint64_t seed) {
    require_valid_pc(p, c);
    OrderingPlan plan = empty_plan(OrderingKind::Elimination, p, c, seed);
    Eliminator(p, c, seed, plan.bucket_sequence).run();
    if (plan.bucket_sequence.size() != plan.num_buckets())
        throw EmberError("elimination order: the construction did not visit every bucket");
    replay_with_belady(plan);
    return plan;
}

// Standard Hilbert index -> (x, y) walk on an n x n grid, n a power of two, origin top-left.
std::pair<std::uint32_t, std::uint32_t> hilbert_d2xy(std::uint32_t n, std::uint64_t d) {
    std::uint32_t x = 0, y = 0;
    for (std::uint32_t s = 1; s < n; s <<= 1, d >>= 2) {
        const std::uint32_t rx = static_cast<std::uint32_t>((d >> 1) & 1u);
        const std::uint32_t ry = static_cast<std::uint32_t>((d ^ rx) & 1u);
        if (!ry) {
            if (rx) {
                x = s - 1 - x;
                y = s - 1 - y;
            }
            std::swap(x, y);
        }
        x += rx * s;
        y += ry * s;
    }
    return {x, y};
}

OrderingPlan hilbert_order(std::uint32_t p, std::uint32_t c) {
    require_valid_pc(p, c);
    OrderingPlan plan = empty_plan(OrderingKind::Hilbert, p, c, 0);
    plan.bucket_sequence = hilbert_walk(p);
    replay_with_belady(plan);
    return plan;
}

OrderingPlan hilbert_symmetric_order(std::uint32_t p, std::uint32_t c) {
    require_valid_pc(p, c);
    OrderingPlan plan = empty_plan(OrderingKind::HilbertSymmetric, p, c, 0);
    std::vector<std::uint8_t> seen(static_cast<std::size_t>(p) * p, 0);
    for (const BucketId& cell : hilbert_walk(p)) {
        const std::uint32_t a = std::min(cell.i, cell.j), b = std::max(cell.i, cell.j);
        std::uint8_t& mark = seen[static_cast<std::size_t>(a) * p + b];
        if (mark) continue;
        mark = 1;
        plan.bucket_sequence.push_back({a, b});
        if (a != b) plan.bucket_sequence.push_back({b, a});
    }
    replay_with_belady(plan);
    return plan;
}

OrderingPlan random_order(std::uint32_t p, std::uint32_t c, std::uint64_t seed) {
    require_valid_pc(p, c);
    OrderingPlan plan = empty_plan(OrderingKind::Random, p, c, seed);
    for (std::uint32_t i = 0; i < p; ++i)
        for (std::uint32_t j = 0; j < p; ++j) plan.bucket_sequence.push_back({i, j});
    Rng(mix_seed(seed, 0x7a2du)).shuffle(plan.bucket_sequence);
    replay_with_belady(plan);
    return plan;
}

OrderingPlan make_plan(OrderingKind kind, std::uint32_t p, std::uint32_t c, std::uint64_t seed) {
    switch (kind) {
        case OrderingKind::Elimination: return elimination_order(p, c, seed);
        case OrderingKind::Hilbert: return hilbert_order(p, c);
        case OrderingKind::HilbertSymmetric: return hilbert_symmetric_order(p, c);
        case OrderingKind::Random: return random_order(p, c, seed);
    }
    throw ConfigError("make_plan: ordering kind out of range");
}

IOReport simulate_io(const OrderingPlan& plan, std::uint64_t partition_bytes) {
    IOReport io;
    const std::uint64_t fill = std::min<std::uint64_t>(plan.c, plan.p);
    io.reads = fill + plan.swap_count;   // initial loads + admissions
    io.writes = plan.swap_count + fill;  // dirty evictions + epoch-end flush
    io.total_bytes = (io.reads + io.writes) * partition_bytes;
    return io;
}

}  // namespace ember
