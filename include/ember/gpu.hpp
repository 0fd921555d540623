// SPDX-License-Identifier: Apache-2.0
//
// ember/gpu.hpp — header-only C++ RAII binding of the C-ABI (include/ember_gpu.h) for the
// reference's own C++ code (namespace ember, proj/). It is what proj/src/pipeline.cpp's
// train_epoch_sync / train_epoch_partitioned would call instead of a CPU
// model: status codes become the reference's exception types (common.h:36-49; ConfigError for
// status 1, EmberError otherwise), the context is owned by a movable handle.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "ember/common.h"
#include "ember_gpu.h"

namespace ember {
namespace gpu {

inline void check(int status) {
    if (status == EMBER_OK) return;
    const std::string msg = ember_last_error();
    if (status == EMBER_EUSER) throw ConfigError(msg);
    throw EmberError(msg);
}

// One GPU's training context (one compute worker, one stream).
class Context {
public:
    Context(int device, const ember_model_desc& model, const ember_graph_desc& graph, void* stream = nullptr) {
        check(ember_ctx_create(device, &model, &graph, stream, &ctx_));
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    Context(Context&& o) noexcept : ctx_(std::exchange(o.ctx_, nullptr)) {}
    Context& operator=(Context&& o) noexcept {
        if (this != &o) {
            reset();
            ctx_ = std::exchange(o.ctx_, nullptr);
        }
        return *this;
    }
    ~Context() { reset(); }

    ember_ctx* get() const { return ctx_; }
    void* stream() const { return ember_ctx_stream(ctx_); }

    // ParameterSlice storage: caller-owned device rows, borrowed.
    void bind_partition(uint32_t part, float* theta_dev, float* acc_dev) {
        check(ember_tables_bind(ctx_, part, theta_dev, acc_dev));
    }
    void bind_relations(float* theta_dev, float* acc_dev) { check(ember_relations_bind(ctx_, theta_dev, acc_dev)); }
    // init_embeddings
    void init_partition(uint32_t part, uint64_t seed) { check(ember_init_partition(ctx_, part, seed)); }
    void init_relations(uint64_t seed) { check(ember_init_relations(ctx_, seed)); }

    // trainEdgeBucket (Algorithm 2): every batch of one bucket, in order.
    ember_step_stats train_bucket(const uint32_t* bucket_edges_dev, uint64_t n, uint32_t i, uint32_t j,
                                  uint64_t epoch, uint32_t bucket_step, bool want_stats = true) {
        ember_step_stats st{};
        check(ember_train_bucket(ctx_, bucket_edges_dev, n, i, j, epoch, bucket_step, want_stats ? &st : nullptr));
        return st;
    }

    // train_epoch_partitioned: the plan's bucket sequence (2 u32 per bucket) in one call.
    ember_step_stats train_epoch(const uint32_t* edges_dev, const std::vector<uint64_t>& bucket_offsets,
                                 const std::vector<uint32_t>& seq, uint64_t epoch) {
        ember_step_stats st{};
        check(ember_train_epoch(ctx_, edges_dev, bucket_offsets.data(), seq.data(), epoch, &st));
        return st;
    }

    // Waits for all of the context's streams; a non-finite batch loss since the last check
    // surfaces here as EmberError naming the batch.
    void synchronize() { check(ember_ctx_synchronize(ctx_)); }

    // Per-op entry points (SPEC model ops), device pointers:
    // sample_negatives: 2*n_t ids [side][slot]
    void sample_negatives(const uint32_t* bucket_edges_dev, uint64_t n, uint32_t i, uint32_t j, uint64_t epoch,
                          uint32_t bucket_step, uint32_t batch_in_bucket, uint32_t* negs_dev) {
        check(ember_sample_negatives(ctx_, bucket_edges_dev, n, i, j, epoch, bucket_step, batch_in_bucket, negs_dev));
    }
    // ParameterSlice gather: one theta (and acc) row per id, in order
    void gather(const uint32_t* ids_dev, uint32_t n, uint32_t i, uint32_t j, bool relations, float* theta_out_dev,
                float* acc_out_dev = nullptr) {
        check(ember_gather(ctx_, ids_dev, n, i, j, relations ? 1 : 0, theta_out_dev, acc_out_dev));
    }
    // adagrad_step on rows of bucket (i, j)'s partitions (or the relation table)
    void adagrad_apply(const uint32_t* ids_dev, const float* rows_dev, uint32_t n, uint32_t i, uint32_t j,
                       bool relations) {
        check(ember_adagrad_apply(ctx_, ids_dev, rows_dev, n, i, j, relations ? 1 : 0));
    }

private:
    void reset() {
        if (ctx_) ember_ctx_destroy(ctx_);
        ctx_ = nullptr;
    }
    ember_ctx* ctx_ = nullptr;
};

// PartitionBuffer on the device: capacity HBM slots over pinned host backing,
// replaying one plan per epoch (Belady eviction, prefetch, async writeback).
class PartitionBuffer {
public:
    PartitionBuffer(Context& ctx, uint32_t capacity, const std::vector<uint32_t>& seq,
                    const std::vector<float*>& host_theta, const std::vector<float*>& host_acc) : ctx_(&ctx) {
        check(ember_buffer_create(ctx.get(), capacity, seq.data(), (uint32_t)(seq.size() / 2), host_theta.data(),
                                  host_acc.data(), &buf_));
    }
    PartitionBuffer(const PartitionBuffer&) = delete;
    PartitionBuffer& operator=(const PartitionBuffer&) = delete;
    ~PartitionBuffer() {
        if (buf_) ember_buffer_destroy(buf_);
    }
    // train_epoch_partitioned through the buffer
    ember_step_stats train_epoch(const uint32_t* edges_dev, const std::vector<uint64_t>& offsets, uint64_t epoch) {
        ember_step_stats st{};
        check(ember_train_epoch_buffered(ctx_->get(), buf_, edges_dev, offsets.data(), epoch, &st));
        return st;
    }
    void flush() { check(ember_buffer_flush(buf_)); }
    ember_buffer_report report() {
        ember_buffer_report r{};
        check(ember_buffer_stats(buf_, &r));
        return r;
    }

private:
    Context* ctx_;
    ember_buffer* buf_ = nullptr;
};

// make_plan (ordering.h:80) through the C-ABI: the bucket sequence as (i, j) pairs.
inline std::vector<std::pair<uint32_t, uint32_t>> bucket_sequence(int kind, uint32_t p, uint32_t c, uint64_t seed) {
    std::vector<uint32_t> seq(2ull * p * p), adm(c + 2ull * p * p + 1), swaps(6ull * p * p + 3), state(1ull * p * p);
    uint64_t swap_count = 0;
    uint32_t n_adm = 0;
    check(ember_make_plan(kind, p, c, seed, seq.data(), &swap_count, adm.data(), &n_adm, swaps.data(), state.data()));
    std::vector<std::pair<uint32_t, uint32_t>> out(1ull * p * p);
    for (size_t t = 0; t < out.size(); ++t) out[t] = {seq[2 * t], seq[2 * t + 1]};
    return out;
}

}  // namespace gpu
}  // namespace ember
