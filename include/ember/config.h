// SPDX-License-Identifier: Apache-2.0
//
// ember/config.h — RunConfig (the engine-cli module's config type; reference
// proj/src/CMakeLists.txt:2 lists config.cpp, absent from the reference) restricted to what the
// training step consumes, with the SPEC's validation rules ("config validation rejects every
// invariant violation listed in RunConfig before any IO") raised as ConfigError.
// The device step has no host pipeline, so the staleness bound is accepted and behaves as bound = 1
// (bound = 1 is bit-identical to the synchronous trainer).
#pragma once

#include <cstdint>
#include <string>

#include "ember/common.h"
#include "ember/model.h"
#include "ember/ordering.h"
#include "ember_gpu.h"

namespace ember {

enum class StorageBackend { InMemory, Partitioned };

struct RunConfig {
    ModelKind model = ModelKind::ComplEx;
    std::uint32_t dim = 100;
    float lr = 0.1f;
    float eps = 1e-10f;
    std::uint32_t batch_size = 50'000;  // b
    NegativeSampleSpec negatives{};     // n_t, alpha, seed, chunks
    std::uint32_t epochs = 1;
    StorageBackend backend = StorageBackend::InMemory;
    std::uint32_t num_partitions = 1;   // p
    std::uint32_t buffer_capacity = 1;  // c (partitions resident in HBM; c = p keeps all resident)
    OrderingKind ordering = OrderingKind::Elimination;
    std::uint64_t order_seed = 0;
    std::uint32_t staleness_bound = 1;
    std::uint64_t init_seed = 11;
    int device = 0;

    void validate() const {
        if (dim == 0) throw ConfigError("RunConfig: dim must be >= 1");
        if (dim % 4) throw ConfigError("RunConfig: dim must be a multiple of 4 (128-bit row accesses)");
        if (model == ModelKind::ComplEx && dim % 2) throw ConfigError("RunConfig: ComplEx requires an even dim");
        if (!(lr > 0.f)) throw ConfigError("RunConfig: lr must be > 0");
        if (!(eps > 0.f)) throw ConfigError("RunConfig: eps must be > 0 (SPEC.md:170)");
        if (batch_size == 0) throw ConfigError("RunConfig: batch_size must be >= 1");
        negatives.validate();
        if (staleness_bound < 1) throw ConfigError("RunConfig: staleness bound must be >= 1");
        if (num_partitions == 0) throw ConfigError("RunConfig: p must be >= 1");
        if (backend == StorageBackend::InMemory && num_partitions != 1)
            throw ConfigError("RunConfig: in-memory storage needs p = 1");
        if (backend == StorageBackend::Partitioned) {
            if (buffer_capacity < 2 || buffer_capacity > num_partitions)
                throw ConfigError("RunConfig: partitioned storage needs p >= c >= 2");
        }
    }

    ember_model_desc model_desc(int engine = EMBER_ENGINE_TC_BF16X3) const {
        ember_model_desc m{};
        m.kind = static_cast<std::int32_t>(model);
        m.dim = dim;
        m.lr = lr;
        m.eps = eps;
        m.batch_size = batch_size;
        m.num_negatives = negatives.n_t;
        m.alpha = negatives.alpha;
        m.num_chunks = negatives.num_chunks;
        m.neg_seed = negatives.seed;
        m.engine = engine;
        return m;
    }

    std::uint32_t capacity() const { return backend == StorageBackend::InMemory ? 1u : buffer_capacity; }
};

}  // namespace ember
