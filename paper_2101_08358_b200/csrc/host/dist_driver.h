// SPDX-License-Identifier: Apache-2.0
// train_epoch_partitioned over G GPUs (Algorithm 2): the round
// loop of one rank, host C++ (host/dist_driver.cpp). The rank's work is behind RankOps: the GPU
// implementation (dist.cu: Engine steps, NCCL relation all-reduce, NCCL P2P partition handoffs on
// a copy stream) or C callbacks (ember_dist_run_epoch: the CPU tests' oracle + gloo backend).
#pragma once
#include <cstdint>
#include <vector>

#include "rounds.h"

namespace ember {

struct BatchRef {
    uint32_t bucket_step, i, j, batch_in_bucket;
    uint64_t lo, hi;      // the bucket's edges [lo, hi) of the bucketed edge array
    uint64_t begin;       // the batch: [lo + begin, lo + begin + nb)
    uint32_t nb;
};

struct Move {
    uint32_t part, src, dst;
};

struct RankOps {
    virtual ~RankOps() = default;
    // One lockstep step: the batch (nullptr: this rank has none left in the round, an idle step),
    // including the relation all-reduce + Adagrad when the model has relations.
    virtual void step(const BatchRef* b, uint64_t epoch) = 0;
    // The partition handoff after `round` (all of this rank's sends and receives, one group),
    // issued at the same lockstep point on every rank; may complete asynchronously.
    virtual void send_recv(uint32_t round, const std::vector<Move>& moves) = 0;
    // Before the first step of `round`: the partitions that arrived for it must be usable (called for
    // every round entered; parts without a pending receive, e.g. after a fresh init, are ignored).
    virtual void acquire(uint32_t round, const std::vector<uint32_t>& arrived) = 0;
};

struct DistReport {
    uint64_t steps = 0, batches = 0, edges = 0, handoffs = 0, moved_partitions = 0;
    uint64_t early_handoffs = 0;  // handoffs issued before their round's last lockstep step
};

// The lockstep plan of every rank (all ranks compute all lists: no coordination needed).
class DistDriver {
   public:
    DistDriver(RoundSchedule S, const uint64_t* offsets, uint32_t batch_size, uint32_t rank);
    const RoundSchedule& schedule() const { return S_; }
    uint32_t rounds() const { return S_.rounds; }
    uint64_t total_steps() const;
    uint32_t steps_in_round(uint32_t r) const { return steps_[r]; }
    // lockstep step (within round r) after which every rank's departing partitions are done
    uint32_t handoff_step(uint32_t r) const { return handoff_[r]; }
    const std::vector<BatchRef>& batches(uint32_t r, uint32_t g) const { return lists_[(size_t)r * S_.world + g]; }
    std::vector<Move> moves(uint32_t r) const;  // round r -> r+1 (the last round -> round 0)
    // Lockstep steps [first, first + count) of the epoch (count = ~0: to its end), handoffs included.
    DistReport run(RankOps& ops, uint64_t epoch, uint64_t first = 0, uint64_t count = ~0ull) const;

   private:
    RoundSchedule S_;
    uint32_t rank_;
    std::vector<std::vector<BatchRef>> lists_;  // [round][rank]
    std::vector<uint32_t> steps_, handoff_;
};

}  // namespace ember
