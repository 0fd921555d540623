// SPDX-License-Identifier: Apache-2.0
//
// ember/model.h — the reference's model module (ModelKind, ParameterSlice,
// NegativeSampleSpec, GradientDelta; score, sample_negatives, loss_and_grad, adagrad_step,
// init_embeddings) as C++ over the B200 C-ABI (include/ember_gpu.h). The reference lists
// proj/src/model.cpp in proj/src/CMakeLists.txt:5 but ships no model code; these are the
// declarations that file would implement, with the computation on the GPU. Header-only: link
// libember_b200.so. Errors are the reference's exception types (common.h:36-49): ConfigError for
// bad arguments (C-ABI status 1), EmberError otherwise (status 2, e.g. a non-finite score naming
// its batch).
#pragma once

#include <cmath>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "ember/common.h"
#include "ember/gpu.hpp"
#include "ember_gpu.h"

namespace ember {

// [TYPE] ModelKind: Dot, DistMult, ComplEx (d/2 complex pairs, [re | im] halves).
enum class ModelKind { Dot = EMBER_DOT, DistMult = EMBER_DISTMULT, ComplEx = EMBER_COMPLEX };

inline std::string to_string(ModelKind k) {
    switch (k) {
        case ModelKind::Dot: return "dot";
        case ModelKind::DistMult: return "distmult";
        case ModelKind::ComplEx: return "complex";
    }
    return "?";
}

inline ModelKind model_kind_from_string(const std::string& s) {
    if (s == "dot") return ModelKind::Dot;
    if (s == "distmult") return ModelKind::DistMult;
    if (s == "complex") return ModelKind::ComplEx;
    throw ConfigError("unknown model kind '" + s + "' (dot, distmult, complex)");
}

// [TYPE] NegativeSampleSpec: n_t per corruption side, degree-based fraction alpha,
// seed; num_chunks: the batch is cut into chunks that each share their own n_t negatives.
struct NegativeSampleSpec {
    std::uint32_t n_t = 1000;
    float alpha = 0.5f;
    std::uint64_t seed = 1;
    std::uint32_t num_chunks = 1;
    void validate() const {
        if (!(alpha >= 0.f && alpha <= 1.f)) throw ConfigError("NegativeSampleSpec: alpha must be in [0, 1]");
        if (num_chunks == 0) throw ConfigError("NegativeSampleSpec: num_chunks must be >= 1");
    }
};

// [OP] score of one triple: Dot = s.d; DistMult = sum s r d; ComplEx = Re(<s, r, conj(d)>).
// A pure function on host vectors (the batched scores run inside loss_and_grad on the GPU).
inline float score(ModelKind kind, const std::vector<float>& s, const std::vector<float>& r,
                   const std::vector<float>& d) {
    if (s.size() != d.size() || (kind != ModelKind::Dot && r.size() != s.size()))
        throw ConfigError("score: dimension mismatch");
    if (kind == ModelKind::ComplEx && s.size() % 2) throw ConfigError("score: ComplEx needs an even dimension");
    float f = 0.f;
    if (kind == ModelKind::Dot) {
        for (size_t k = 0; k < s.size(); ++k) f += s[k] * d[k];
    } else if (kind == ModelKind::DistMult) {
        for (size_t k = 0; k < s.size(); ++k) f += s[k] * r[k] * d[k];
    } else {
        const size_t h = s.size() / 2;
        for (size_t k = 0; k < h; ++k) {  // Re((a+ib)(c+ie)(x-iy))
            const float a = s[k], b = s[h + k], c = r[k], e = r[h + k], x = d[k], y = d[h + k];
            f += (a * c - b * e) * x + (a * e + b * c) * y;
        }
    }
    return f;
}

// Device memory owned through a context (ember_device_alloc): a typed RAII array.
template <typename T>
class DeviceArray {
public:
    DeviceArray() = default;
    DeviceArray(gpu::Context& ctx, std::size_t n) : ctx_(&ctx), n_(n) {
        void* p = nullptr;
        gpu::check(ember_device_alloc(ctx.get(), n * sizeof(T), &p));
        p_ = static_cast<T*>(p);
    }
    DeviceArray(gpu::Context& ctx, const std::vector<T>& host) : DeviceArray(ctx, host.size()) { upload(host); }
    DeviceArray(const DeviceArray&) = delete;
    DeviceArray& operator=(const DeviceArray&) = delete;
    DeviceArray(DeviceArray&& o) noexcept
        : ctx_(std::exchange(o.ctx_, nullptr)), p_(std::exchange(o.p_, nullptr)), n_(std::exchange(o.n_, 0)) {}
    DeviceArray& operator=(DeviceArray&& o) noexcept {
        if (this != &o) {
            release();
            ctx_ = std::exchange(o.ctx_, nullptr);
            p_ = std::exchange(o.p_, nullptr);
            n_ = std::exchange(o.n_, 0);
        }
        return *this;
    }
    ~DeviceArray() { release(); }

    T* data() const { return p_; }
    std::size_t size() const { return n_; }
    void upload(const std::vector<T>& host) {
        if (host.size() > n_) throw ConfigError("DeviceArray::upload: too many elements");
        gpu::check(ember_copy_to_device(ctx_->get(), p_, host.data(), host.size() * sizeof(T)));
    }
    std::vector<T> download(std::size_t count) const {
        std::vector<T> h(count);
        if (count > n_) throw ConfigError("DeviceArray::download: too many elements");
        gpu::check(ember_copy_to_host(ctx_->get(), h.data(), p_, count * sizeof(T)));
        return h;
    }
    std::vector<T> download() const { return download(n_); }

private:
    void release() {
        if (p_ && ctx_) ember_device_free(ctx_->get(), p_);
        p_ = nullptr;
    }
    gpu::Context* ctx_ = nullptr;
    T* p_ = nullptr;
    std::size_t n_ = 0;
};

// [TYPE] ParameterSlice: gathered theta rows (rows x d) and their Adagrad
// accumulators, one row per requested id, in request order.
struct ParameterSlice {
    DeviceArray<float> theta, acc;
    std::uint32_t rows = 0, dim = 0;
};

// ParameterSlice of node ids (lying in partitions i or j) or of relation ids (relations = true).
inline ParameterSlice gather(gpu::Context& ctx, const std::uint32_t* ids_dev, std::uint32_t n, std::uint32_t dim,
                             std::uint32_t i, std::uint32_t j, bool relations = false) {
    ParameterSlice s{DeviceArray<float>(ctx, (std::size_t)n * dim), DeviceArray<float>(ctx, (std::size_t)n * dim), n,
                     dim};
    ctx.gather(ids_dev, n, i, j, relations, s.theta.data(), s.acc.data());
    return s;
}

// [TYPE] GradientDelta: unique node ids (ascending) with one summed gradient row
// each, and the same for the touched relations.
struct GradientDelta {
    DeviceArray<std::uint32_t> node_ids;
    DeviceArray<float> node_rows;
    std::uint32_t n_nodes = 0;
    DeviceArray<std::uint32_t> rel_ids;
    DeviceArray<float> rel_rows;
    std::uint32_t n_rels = 0;
};

struct LossAndGrad {
    double loss = 0.0;
    DeviceArray<float> fpos;  // [nb] positive scores
    DeviceArray<float> lse;   // [2][nb] log-sum-exp per corruption side (0: destination)
    GradientDelta delta;
};

// [OP] sample_negatives: num_chunks * 2 * n_t ids [chunk][side][slot] for batch
// `batch_in_bucket` of bucket (i, j); degree-based part = endpoints of uniform bucket edges.
inline DeviceArray<std::uint32_t> sample_negatives(gpu::Context& ctx, const NegativeSampleSpec& spec,
                                                   const std::uint32_t* bucket_edges_dev, std::uint64_t bucket_n,
                                                   std::uint32_t i, std::uint32_t j, std::uint64_t epoch,
                                                   std::uint32_t bucket_step, std::uint32_t batch_in_bucket) {
    spec.validate();
    DeviceArray<std::uint32_t> out(ctx, (std::size_t)spec.num_chunks * 2 * spec.n_t);
    ctx.sample_negatives(bucket_edges_dev, bucket_n, i, j, epoch, bucket_step, batch_in_bucket, out.data());
    return out;
}

// [OP] loss_and_grad of nb positives at edges_dev (bucket (i, j)) against negs_dev:
// mean loss over the positives (both corruption sides), the positive scores, the log-sum-exps and
// the GradientDelta. No parameter changes.
inline LossAndGrad loss_and_grad(gpu::Context& ctx, std::uint32_t dim, const std::uint32_t* edges_dev,
                                 std::uint32_t nb, std::uint32_t i, std::uint32_t j, const std::uint32_t* negs_dev,
                                 std::size_t n_negs) {
    LossAndGrad out;
    out.fpos = DeviceArray<float>(ctx, nb);
    out.lse = DeviceArray<float>(ctx, 2ull * nb);
    const std::size_t cap = 2ull * nb + n_negs;
    out.delta.node_ids = DeviceArray<std::uint32_t>(ctx, cap);
    out.delta.node_rows = DeviceArray<float>(ctx, cap * dim);
    out.delta.rel_ids = DeviceArray<std::uint32_t>(ctx, nb);
    out.delta.rel_rows = DeviceArray<float>(ctx, (std::size_t)nb * dim);
    gpu::check(ember_loss_and_grad(ctx.get(), edges_dev, nb, i, j, negs_dev, out.fpos.data(), out.lse.data(),
                                   out.delta.node_ids.data(), out.delta.node_rows.data(), &out.delta.n_nodes,
                                   out.delta.rel_ids.data(), out.delta.rel_rows.data(), &out.delta.n_rels,
                                   &out.loss));
    return out;
}

// [OP] adagrad_step of a GradientDelta: node rows of bucket (i, j)'s partitions and
// the relation rows, acc += g^2; theta -= lr g / (sqrt(acc) + eps).
inline void adagrad_step(gpu::Context& ctx, const GradientDelta& delta, std::uint32_t i, std::uint32_t j) {
    if (delta.n_nodes) ctx.adagrad_apply(delta.node_ids.data(), delta.node_rows.data(), delta.n_nodes, i, j, false);
    if (delta.n_rels) ctx.adagrad_apply(delta.rel_ids.data(), delta.rel_rows.data(), delta.n_rels, i, j, true);
}

// [OP] init_embeddings: every bound partition and the relation table; global row g
// <- Rng(mix_seed(seed, g)).uniform(-1/sqrt(d), 1/sqrt(d)) x d, Adagrad state 0.
inline void init_embeddings(gpu::Context& ctx, std::uint32_t num_partitions, bool relations, std::uint64_t seed) {
    for (std::uint32_t k = 0; k < num_partitions; ++k) ctx.init_partition(k, seed);
    if (relations) ctx.init_relations(seed);
}

}  // namespace ember
