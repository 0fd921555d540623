// SPDX-License-Identifier: Apache-2.0
//
// ember/pipeline.h — the reference's pipeline module (proj/src/pipeline.cpp is
// listed in proj/src/CMakeLists.txt:8 but absent): train_epoch_sync (Algorithm 1) and
// train_epoch_partitioned (Algorithm 2) over one GPU's device-resident step, as C++ over the C-ABI.
//
// A Trainer owns one GPU context, the node partitions and the relation table. With every partition
// resident (in-memory storage, or partitioned with c = p) the tables live in HBM; with c < p they live
// in pinned host memory behind the device partition buffer (c HBM slots + 2 staging
// slots, Belady eviction, prefetch, asynchronous writeback). Each epoch is one C-ABI call with no host
// synchronisation inside it; EpochStats are filled once at its end.
#pragma once

#include <chrono>
#include <cstdint>
#include <memory>
#include <vector>

#include "ember/common.h"
#include "ember/config.h"
#include "ember/gpu.hpp"
#include "ember/model.h"
#include "ember/ordering.h"
#include "ember_gpu.h"

namespace ember {

// EpochStats (epoch, mean loss, edges/sec, buffer reads/writes/stalls, max staleness).
struct EpochStats {
    std::uint64_t epoch = 0;
    double mean_loss = 0.0;
    std::uint64_t edges = 0;
    std::uint64_t batches = 0;
    double seconds = 0.0;
    double edges_per_sec = 0.0;
    std::uint64_t buffer_reads = 0, buffer_writes = 0;
    std::uint32_t buffer_stalls = 0;
    std::uint32_t max_staleness = 0;  // the device step reads every row after the previous update
};

class Trainer {
public:
    // GraphMeta subset: |V|, |R|; p comes from the config.
    Trainer(const RunConfig& cfg, std::uint64_t num_nodes, std::uint32_t num_relations) : cfg_(cfg) {
        cfg_.validate();
        const ember_model_desc md = cfg_.model_desc();
        const ember_graph_desc gd{num_nodes, num_relations, cfg_.num_partitions};
        ctx_ = std::make_unique<gpu::Context>(cfg_.device, md, gd);
        plan_ = make_plan(cfg_.ordering, cfg_.num_partitions, cfg_.capacity() < cfg_.num_partitions
                                                                  ? cfg_.capacity() : cfg_.num_partitions,
                          cfg_.order_seed);
        for (const BucketId& b : plan_.bucket_sequence) {
            seq_.push_back(b.i);
            seq_.push_back(b.j);
        }
        if (cfg_.model != ModelKind::Dot) gpu::check(ember_tables_allocate(ctx_->get(), EMBER_RELATIONS));
        if (buffered()) {
            for (std::uint32_t k = 0; k < cfg_.num_partitions; ++k) {
                const std::uint64_t n = rows(k) * cfg_.dim;
                void *t = nullptr, *a = nullptr;
                gpu::check(ember_host_alloc_pinned(n * sizeof(float), &t));
                gpu::check(ember_host_alloc_pinned(n * sizeof(float), &a));
                host_theta_.push_back(static_cast<float*>(t));
                host_acc_.push_back(static_cast<float*>(a));
            }
            buffer_ = std::make_unique<gpu::PartitionBuffer>(*ctx_, cfg_.capacity(), seq_, host_theta_, host_acc_);
        } else {
            for (std::uint32_t k = 0; k < cfg_.num_partitions; ++k)
                gpu::check(ember_tables_allocate(ctx_->get(), k));
        }
    }
    Trainer(const Trainer&) = delete;
    Trainer& operator=(const Trainer&) = delete;
    ~Trainer() {
        buffer_.reset();
        ctx_.reset();
        for (float* p : host_theta_) ember_host_free_pinned(p);
        for (float* p : host_acc_) ember_host_free_pinned(p);
    }

    gpu::Context& context() { return *ctx_; }
    const RunConfig& config() const { return cfg_; }
    const OrderingPlan& plan() const { return plan_; }
    bool buffered() const { return cfg_.capacity() < cfg_.num_partitions; }
    std::uint64_t rows(std::uint32_t part) const {
        std::uint64_t r = 0;
        gpu::check(ember_tables_get(ctx_->get(), part, nullptr, nullptr, &r));
        return r;
    }

    // init_embeddings: computed on the device; with the buffer, partition by partition
    // through a staging table into the pinned backing store (bit-identical to a resident init).
    void init_embeddings() {
        if (cfg_.model != ModelKind::Dot) ctx_->init_relations(cfg_.init_seed);
        if (!buffered()) {
            for (std::uint32_t k = 0; k < cfg_.num_partitions; ++k) ctx_->init_partition(k, cfg_.init_seed);
            return;
        }
        std::uint64_t max_rows = 0;
        for (std::uint32_t k = 0; k < cfg_.num_partitions; ++k) max_rows = std::max(max_rows, rows(k));
        DeviceArray<float> stage(*ctx_, 2 * max_rows * cfg_.dim);
        for (std::uint32_t k = 0; k < cfg_.num_partitions; ++k) {
            const std::uint64_t n = rows(k) * cfg_.dim;
            ctx_->bind_partition(k, stage.data(), stage.data() + max_rows * cfg_.dim);
            ctx_->init_partition(k, cfg_.init_seed);
            gpu::check(ember_copy_to_host(ctx_->get(), host_theta_[k], stage.data(), n * sizeof(float)));
            gpu::check(ember_copy_to_host(ctx_->get(), host_acc_[k], stage.data() + max_rows * cfg_.dim,
                                          n * sizeof(float)));
        }
    }

    // All partitions resident: train in another plan's bucket order (e.g. the order a buffered run
    // with a smaller capacity uses). A buffered trainer's order is fixed by its buffer.
    void use_plan(const OrderingPlan& plan) {
        if (buffered()) throw ConfigError("use_plan: a buffered trainer replays its buffer's plan");
        if (plan.p != cfg_.num_partitions) throw ConfigError("use_plan: plan is for another p");
        plan_ = plan;
        seq_.clear();
        for (const BucketId& b : plan_.bucket_sequence) {
            seq_.push_back(b.i);
            seq_.push_back(b.j);
        }
    }

    // theta (and acc) of partition k, or of the relation table (k = EMBER_RELATIONS), on the host,
    // in on-disk coordinate order (the tables and the backing store hold the HBM row layout).
    std::vector<float> download(std::uint32_t k, bool acc = false) {
        const std::uint64_t n = rows(k) * cfg_.dim;
        std::vector<float> out(n);
        if (buffered() && k != EMBER_RELATIONS) {
            buffer_->flush();
            const float* src = acc ? host_acc_[k] : host_theta_[k];
            std::copy(src, src + n, out.begin());
        } else {
            float *t = nullptr, *a = nullptr;
            gpu::check(ember_tables_get(ctx_->get(), k, &t, &a, nullptr));
            gpu::check(ember_copy_to_host(ctx_->get(), out.data(), acc ? a : t, n * sizeof(float)));
        }
        gpu::check(ember_rows_layout_host(static_cast<int>(cfg_.model), cfg_.dim, out.data(), rows(k), 0));
        return out;
    }

    // train_epoch_sync (Algorithm 1) / train_epoch_partitioned (Algorithm 2):
    // the plan's buckets in order, each bucket's batches (consecutive slices of its edges) in order.
    EpochStats train_epoch(const std::uint32_t* edges_dev, const std::vector<std::uint64_t>& bucket_offsets,
                           std::uint64_t epoch) {
        const std::uint32_t p = cfg_.num_partitions;
        if (bucket_offsets.size() != (std::size_t)p * p + 1) throw ConfigError("bucket_offsets must hold p*p+1 entries");
        ember_buffer_report before{};
        if (buffered()) before = buffer_->report();
        const auto t0 = std::chrono::steady_clock::now();
        ember_step_stats st = buffered() ? buffer_->train_epoch(edges_dev, bucket_offsets, epoch)
                                         : ctx_->train_epoch(edges_dev, bucket_offsets, seq_, epoch);
        if (buffered()) buffer_->flush();
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        EpochStats out;
        out.epoch = epoch;
        out.mean_loss = st.batches ? st.loss_sum / (double)st.batches : 0.0;
        out.edges = st.edges;
        out.batches = st.batches;
        out.seconds = s;
        out.edges_per_sec = s > 0 ? (double)st.edges / s : 0.0;
        if (buffered()) {
            const ember_buffer_report r = buffer_->report();
            out.buffer_reads = r.reads - before.reads;
            out.buffer_writes = r.writes - before.writes;
            out.buffer_stalls = r.stalls - before.stalls;
        }
        return out;
    }

private:
    RunConfig cfg_;
    std::unique_ptr<gpu::Context> ctx_;
    OrderingPlan plan_;
    std::vector<std::uint32_t> seq_;
    std::vector<float*> host_theta_, host_acc_;
    std::unique_ptr<gpu::PartitionBuffer> buffer_;
};

// The SPEC's free-function names.
inline EpochStats train_epoch_sync(Trainer& t, const std::uint32_t* edges_dev, const std::vector<std::uint64_t>& offsets,
                                   std::uint64_t epoch) {
    if (t.config().backend != StorageBackend::InMemory && t.buffered())
        throw ConfigError("train_epoch_sync: storage is buffered; use train_epoch_partitioned");
    return t.train_epoch(edges_dev, offsets, epoch);
}

inline EpochStats train_epoch_partitioned(Trainer& t, const std::uint32_t* edges_dev,
                                          const std::vector<std::uint64_t>& offsets, std::uint64_t epoch) {
    return t.train_epoch(edges_dev, offsets, epoch);
}

}  // namespace ember
