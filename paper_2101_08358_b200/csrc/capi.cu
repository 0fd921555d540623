// SPDX-License-Identifier: Apache-2.0
//
// extern "C" boundary (include/ember_gpu.h). Converts exceptions to status codes
// (ConfigError -> EMBER_EUSER, anything else -> EMBER_EINTERNAL) with a thread-local message.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <exception>
#include <functional>
#include <new>
#include <string>

#include "ember/ordering.h"
#include "engine.h"
#include "host/rounds.h"

namespace ember {
void graph_generate(int device, uint64_t V, uint32_t R, uint64_t n, uint64_t seed, float train, float valid,
                    uint32_t* edges, uint8_t* split);
void graph_bucket(int device, uint64_t V, uint32_t p, const uint32_t* in, uint64_t n, uint32_t* out,
                  uint64_t* offsets);
void graph_preprocess(int device, const uint32_t* raw, uint64_t n, uint32_t p, uint64_t seed, float train_frac,
                      float valid_frac, uint32_t* train_out, uint64_t* offsets, uint32_t* valid_out, uint32_t* test_out,
                      uint64_t* counts, uint32_t* node_tokens, uint32_t* rel_tokens, uint64_t* num_nodes,
                      uint32_t* num_rel);
double tc_selftest(int device, int mode, int K, int N, uint64_t seed);
double tc_mmabench(int device, int mode, int N, int iters, int nacc);
void launch_eval_filtered(const Engine& E, const uint32_t* test, uint32_t n_test, const uint64_t* keys, uint64_t n_keys,
                          uint32_t* ranks);
struct PartitionBuffer;
PartitionBuffer* buffer_create(Engine& E, uint32_t c, const uint32_t* seq, uint32_t steps, float* const* host_theta,
                               float* const* host_acc);
void buffer_destroy(PartitionBuffer* B);
void buffer_acquire(PartitionBuffer* B, uint32_t step, uint32_t* i, uint32_t* j);
void buffer_release(PartitionBuffer* B, uint32_t step);
void buffer_flush(PartitionBuffer* B);
void buffer_stats(PartitionBuffer* B, ember_buffer_report* out);
uint32_t buffer_decisions(PartitionBuffer* B, uint32_t* out);
Engine& buffer_engine(PartitionBuffer* B);
void launch_eval(const Engine& E, const uint32_t* test, uint32_t n_test, const uint32_t* train, uint64_t n_train,
                 uint32_t n_eval, float alpha_eval, uint32_t block, uint64_t eval_seed, uint32_t* ranks);
}  // namespace ember

using namespace ember;

struct ember_ctx {
    Engine* e;
};

struct ember_buffer {
    PartitionBuffer* b;
    ember_ctx* ctx;
};

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        g_err.clear();
        return EMBER_OK;
    } catch (const ConfigError& ex) {
        g_err = ex.what();
        return EMBER_EUSER;
    } catch (const std::bad_alloc&) {
        g_err = "host out of memory";
        return EMBER_EINTERNAL;
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return EMBER_EINTERNAL;
    } catch (...) {
        g_err = "unknown error";
        return EMBER_EINTERNAL;
    }
}

Engine& eng(ember_ctx* c) {
    if (!c || !c->e) throw ConfigError("null context");
    EMBER_CUDA(cudaSetDevice(c->e->device));
    return *c->e;
}

PartitionBuffer& buf(ember_buffer* b) {
    if (!b || !b->b) throw ConfigError("null buffer");
    eng(b->ctx);
    return *b->b;
}

void need(const void* p, const char* what) {
    if (!p) throw ConfigError(std::string(what) + " must not be NULL");
}
}  // namespace

namespace ember {
// for the other translation units behind the C-ABI (dist.cu)
Engine& engine_of(ember_ctx* c) { return eng(c); }
int guarded_status(const std::function<void()>& f) { return guarded(f); }
}  // namespace ember

namespace {
// train_epoch_partitioned (Algorithm 2): the buckets of `seq` in order, every batch
// of each; acquire/release (nullable) bracket each bucket (the partition buffer). The per-batch
// losses go to one device array read once at the end: no host synchronisation inside the epoch.
template <typename Acquire, typename Release>
void train_epoch_impl(Engine& E, const uint32_t* edges, const uint64_t* offsets, const uint32_t* seq,
                      uint64_t epoch, ember_step_stats* stats, Acquire&& acquire, Release&& release) {
    const uint32_t p = E.g.num_partitions;
    uint64_t nbatch = 0;
    for (uint64_t k = 0; k < (uint64_t)p * p; ++k) {
        if (offsets[k + 1] < offsets[k]) throw ConfigError("offsets must be non-decreasing");
        nbatch += (offsets[k + 1] - offsets[k] + E.cap_b - 1) / E.cap_b;
    }
    const uint64_t n_edges = offsets[(size_t)p * p] - offsets[0];
    NvtxRange nvtx("ember::train_epoch");
    float* losses = nullptr;
    if (stats && nbatch) EMBER_CUDA(cudaMallocAsync(&losses, nbatch * sizeof(float), E.stream));
    uint64_t slot = 0;
    for (uint32_t t = 0; t < p * p; ++t) {
        uint32_t i = seq ? seq[2 * t] : 0, j = seq ? seq[2 * t + 1] : 0;
        NvtxRange nvtx_bucket("ember::bucket");
        acquire(t, &i, &j);
        if (i >= p || j >= p) throw ConfigError("bucket out of range");
        const uint64_t lo = offsets[(size_t)i * p + j], hi = offsets[(size_t)i * p + j + 1];
        for (uint64_t b0 = 0, k = 0; lo + b0 < hi; b0 += E.cap_b, ++k) {
            const uint32_t nb = (uint32_t)std::min<uint64_t>(E.cap_b, hi - lo - b0);
            E.train_batch(edges + 3 * lo, hi - lo, b0, nb, i, j, epoch, t, (uint32_t)k, losses ? losses + slot : nullptr);
            ++slot;
        }
        release(t);
    }
    if (stats) {
        std::vector<float> h(nbatch);
        if (nbatch) {
            EMBER_CUDA(cudaMemcpyAsync(h.data(), losses, nbatch * sizeof(float), cudaMemcpyDeviceToHost, E.stream));
            EMBER_CUDA(cudaFreeAsync(losses, E.stream));
        }
        EMBER_CUDA(cudaStreamSynchronize(E.stream));
        E.check_finite();
        for (float x : h) stats->loss_sum += x;
        stats->batches += nbatch;
        stats->edges += n_edges;
    }
}
}  // namespace

extern "C" {

const char* ember_last_error(void) { return g_err.c_str(); }
int ember_version(void) { return 1; }

int ember_ctx_create(int device, const ember_model_desc* model, const ember_graph_desc* graph, void* stream,
                     ember_ctx** out) {
    return guarded([&] {
        need(model, "model");
        need(graph, "graph");
        need(out, "out");
        *out = nullptr;
        auto* c = new ember_ctx{nullptr};
        try {
            c->e = new Engine(device, *model, *graph, static_cast<cudaStream_t>(stream));
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int ember_ctx_destroy(ember_ctx* ctx) {
    return guarded([&] {
        if (!ctx) return;
        delete ctx->e;
        delete ctx;
    });
}

void* ember_ctx_stream(ember_ctx* ctx) { return ctx && ctx->e ? static_cast<void*>(ctx->e->stream) : nullptr; }

int ember_ctx_synchronize(ember_ctx* ctx) {
    return guarded([&] {
        Engine& E = eng(ctx);
        for (cudaStream_t st : {E.stream, E.side, E.io, E.io_out})
            if (st) EMBER_CUDA(cudaStreamSynchronize(st));
        E.check_finite();  // a non-finite loss since the last check is an error naming its batch
    });
}

int ember_tables_bind(ember_ctx* ctx, uint32_t part, float* theta, float* acc) {
    return guarded([&] {
        Engine& E = eng(ctx);
        if (part >= E.parts.size()) throw ConfigError("partition id out of range");
        need(theta, "theta");
        need(acc, "acc");
        if ((reinterpret_cast<uintptr_t>(theta) | reinterpret_cast<uintptr_t>(acc)) & 15)
            throw ConfigError("tables must be 16-byte aligned");
        E.parts[part].theta = theta;
        E.parts[part].acc = acc;
    });
}

int ember_relations_bind(ember_ctx* ctx, float* theta, float* acc) {
    return guarded([&] {
        Engine& E = eng(ctx);
        need(theta, "theta");
        need(acc, "acc");
        E.rel_theta = theta;
        E.rel_acc = acc;
    });
}

int ember_device_alloc(ember_ctx* ctx, size_t bytes, void** out) {
    return guarded([&] {
        Engine& E = eng(ctx);
        need(out, "out");
        *out = nullptr;
        void* p = nullptr;
        EMBER_CUDA(cudaMalloc(&p, bytes ? bytes : 16));
        E.owned.push_back(p);
        *out = p;
    });
}

int ember_device_free(ember_ctx* ctx, void* p) {
    return guarded([&] {
        Engine& E = eng(ctx);
        if (!p) return;
        auto it = std::find(E.owned.begin(), E.owned.end(), p);
        if (it == E.owned.end()) throw ConfigError("pointer was not allocated by this context");
        EMBER_CUDA(cudaStreamSynchronize(E.stream));  // (work on the context stream may still read it)
        EMBER_CUDA(cudaFree(p));
        E.owned.erase(it);
    });
}

int ember_copy_to_device(ember_ctx* ctx, void* dst_dev, const void* src_host, size_t bytes) {
    return guarded([&] {
        Engine& E = eng(ctx);
        if (!bytes) return;
        need(dst_dev, "dst_dev");
        need(src_host, "src_host");
        EMBER_CUDA(cudaMemcpyAsync(dst_dev, src_host, bytes, cudaMemcpyHostToDevice, E.stream));
        EMBER_CUDA(cudaStreamSynchronize(E.stream));
    });
}

int ember_copy_to_host(ember_ctx* ctx, void* dst_host, const void* src_dev, size_t bytes) {
    return guarded([&] {
        Engine& E = eng(ctx);
        if (!bytes) return;
        need(dst_host, "dst_host");
        need(src_dev, "src_dev");
        EMBER_CUDA(cudaMemcpyAsync(dst_host, src_dev, bytes, cudaMemcpyDeviceToHost, E.stream));
        EMBER_CUDA(cudaStreamSynchronize(E.stream));
    });
}

int ember_host_alloc_pinned(size_t bytes, void** out) {
    return guarded([&] {
        need(out, "out");
        *out = nullptr;
        EMBER_CUDA(cudaHostAlloc(out, bytes ? bytes : 16, cudaHostAllocPortable));
    });
}

int ember_host_free_pinned(void* p) {
    return guarded([&] {
        if (p) EMBER_CUDA(cudaFreeHost(p));
    });
}

int ember_tables_allocate(ember_ctx* ctx, uint32_t part) {
    return guarded([&] {
        Engine& E = eng(ctx);
        const bool rel = part == EMBER_RELATIONS;
        if (!rel && part >= E.parts.size()) throw ConfigError("partition id out of range");
        if (rel && E.m.kind == EMBER_DOT) throw ConfigError("Dot models have no relation table");
        const uint64_t rows = rel ? E.g.num_relations : E.parts[part].rows;
        float* p = nullptr;
        EMBER_CUDA(cudaMalloc(&p, 2 * rows * E.dim * sizeof(float)));
        E.owned.push_back(p);
        if (rel) {
            E.rel_theta = p;
            E.rel_acc = p + rows * E.dim;
        } else {
            E.parts[part].theta = p;
            E.parts[part].acc = p + rows * E.dim;
        }
    });
}

int ember_tables_get(ember_ctx* ctx, uint32_t part, float** theta_dev, float** acc_dev, uint64_t* rows) {
    return guarded([&] {
        Engine& E = eng(ctx);
        const bool rel = part == EMBER_RELATIONS;
        if (!rel && part >= E.parts.size()) throw ConfigError("partition id out of range");
        if (theta_dev) *theta_dev = rel ? E.rel_theta : E.parts[part].theta;
        if (acc_dev) *acc_dev = rel ? E.rel_acc : E.parts[part].acc;
        if (rows) *rows = rel ? E.g.num_relations : E.parts[part].rows;
    });
}

int ember_rows_layout(ember_ctx* ctx, float* rows_dev, uint64_t rows, int to_hbm) {
    return guarded([&] {
        Engine& E = eng(ctx);
        if (rows && !rows_dev) throw ConfigError("rows_dev is null");
        launch_rows_layout(E.stream, rows_dev, rows, nullptr, E.dim, E.m.kind, to_hbm != 0);
    });
}

int ember_rows_layout_host(int kind, uint32_t dim, float* rows, uint64_t n, int to_hbm) {
    return guarded([&] {
        if (kind < EMBER_DOT || kind > EMBER_COMPLEX) throw ConfigError("model kind must be 0, 1 or 2");
        if (dim == 0 || dim % 4) throw ConfigError("dim must be a positive multiple of 4");
        if (kind != EMBER_COMPLEX || !n) return;
        if (!rows) throw ConfigError("rows is null");
        std::vector<float> t(dim);
        for (uint64_t r = 0; r < n; ++r) {
            float* row = rows + r * dim;
            std::copy(row, row + dim, t.begin());
            for (uint32_t c = 0; c < dim; ++c) {
                const uint32_t p = hbm_pos(kind, dim, c);
                if (to_hbm) row[p] = t[c];
                else row[c] = t[p];
            }
        }
    });
}

int ember_init_partition(ember_ctx* ctx, uint32_t part, uint64_t seed) {
    return guarded([&] {
        Engine& E = eng(ctx);
        const PartView v = E.view(part);
        launch_init_rows(E.stream, v.theta, v.acc, v.first, v.rows, E.dim, E.m.kind, seed);
    });
}

int ember_init_relations(ember_ctx* ctx, uint64_t seed) {
    return guarded([&] {
        Engine& E = eng(ctx);
        if (!E.rel_theta) throw ConfigError("relation table not bound");
        launch_init_rows(E.stream, E.rel_theta, E.rel_acc, 0, E.g.num_relations, E.dim, E.m.kind, seed ^ 0x52454cULL);
    });
}

int ember_train_batch(ember_ctx* ctx, const uint32_t* bucket, uint64_t bucket_n, uint64_t batch_begin, uint32_t nb,
                      uint32_t i, uint32_t j, uint64_t epoch, uint32_t bucket_step, uint32_t batch_in_bucket,
                      float* loss_dev) {
    return guarded([&] {
        Engine& E = eng(ctx);
        need(bucket, "bucket_edges_dev");
        E.train_batch(bucket, bucket_n, batch_begin, nb, i, j, epoch, bucket_step, batch_in_bucket, loss_dev);
    });
}

namespace {
// Algorithm 2 trainEdgeBucket: all batches of one bucket; per-batch losses summed into stats.
void train_bucket(Engine& E, const uint32_t* bucket, uint64_t n, uint32_t i, uint32_t j, uint64_t epoch,
                  uint32_t bucket_step, ember_step_stats* stats) {
        double loss_sum = 0.0;
        uint64_t batches = 0;
        float* losses = nullptr;
        const uint64_t nbatch = (n + E.cap_b - 1) / E.cap_b;
        if (stats && nbatch) EMBER_CUDA(cudaMallocAsync(&losses, nbatch * sizeof(float), E.stream));
        for (uint64_t b0 = 0, k = 0; b0 < n; b0 += E.cap_b, ++k) {
            const uint32_t nb = (uint32_t)std::min<uint64_t>(E.cap_b, n - b0);
            E.train_batch(bucket, n, b0, nb, i, j, epoch, bucket_step, (uint32_t)k, losses ? losses + k : nullptr);
            ++batches;
        }
        if (stats) {
            std::vector<float> h(nbatch);
            if (nbatch) {
                EMBER_CUDA(cudaMemcpyAsync(h.data(), losses, nbatch * sizeof(float), cudaMemcpyDeviceToHost, E.stream));
                EMBER_CUDA(cudaFreeAsync(losses, E.stream));
            }
            EMBER_CUDA(cudaStreamSynchronize(E.stream));
            E.check_finite();
            for (float x : h) loss_sum += x;
            stats->loss_sum += loss_sum;
            stats->batches += batches;
            stats->edges += n;
        }
}
}  // namespace

int ember_train_bucket(ember_ctx* ctx, const uint32_t* bucket, uint64_t n, uint32_t i, uint32_t j, uint64_t epoch,
                       uint32_t bucket_step, ember_step_stats* stats) {
    return guarded([&] {
        Engine& E = eng(ctx);
        need(bucket, "bucket_edges_dev");
        train_bucket(E, bucket, n, i, j, epoch, bucket_step, stats);
    });
}

int ember_train_batch_host(ember_ctx* ctx, const uint32_t* bucket, uint64_t bucket_n, const uint32_t* host_batch,
                           uint32_t nb, uint32_t i, uint32_t j, uint64_t epoch, uint32_t bucket_step,
                           uint32_t batch_in_bucket, float* loss_host) {
    return guarded([&] {
        Engine& E = eng(ctx);
        need(bucket, "bucket_edges_dev");
        need(host_batch, "host_batch");
        E.train_batch_host(bucket, bucket_n, host_batch, nb, i, j, epoch, bucket_step, batch_in_bucket, loss_host);
    });
}

int ember_sample_negatives(ember_ctx* ctx, const uint32_t* bucket, uint64_t bucket_n, uint32_t i, uint32_t j,
                           uint64_t epoch, uint32_t bucket_step, uint32_t batch_in_bucket, uint32_t* negs_dev) {
    return guarded([&] {
        Engine& E = eng(ctx);
        need(negs_dev, "negs_dev");
        E.sample(bucket, bucket_n, i, j, epoch, bucket_step, batch_in_bucket, negs_dev);
    });
}

int ember_loss_and_grad(ember_ctx* ctx, const uint32_t* edges, uint32_t nb, uint32_t i, uint32_t j,
                        const uint32_t* negs, float* fpos, float* lse, uint32_t* node_ids, float* node_rows,
                        uint32_t* n_node, uint32_t* rel_ids, float* rel_rows, uint32_t* n_rel, double* loss) {
    return guarded([&] {
        Engine& E = eng(ctx);
        need(edges, "edges_dev");
        need(negs, "negs_dev");
        if (nb == 0 || nb > E.cap_b) throw ConfigError("batch size must be in [1, batch_size]");
        E.check_bucket(i, j);
        E.loss_target = E.s.loss;
        E.batch_tag = 1ull << 63;  // batch id 0 (a standalone batch)
        E.forward_backward(edges, nb, i, j, negs);
        launch_loss(E, nb, E.s.loss);
        if (fpos) EMBER_CUDA(cudaMemcpyAsync(fpos, E.s.fpos, nb * sizeof(float), cudaMemcpyDeviceToDevice, E.stream));
        if (lse) EMBER_CUDA(cudaMemcpyAsync(lse, E.s.lse, 2ull * nb * sizeof(float), cudaMemcpyDeviceToDevice, E.stream));
        E.reduce_and_apply(nb, i, j, false, node_ids, node_rows, rel_ids, rel_rows);
        // GradientDelta rows leave in on-disk coordinate order (counts known on the device)
        launch_rows_layout(E.stream, node_rows, E.slots(nb), E.s.nunique, E.dim, E.m.kind, false);
        launch_rows_layout(E.stream, rel_rows, E.slots(nb), E.s.nunique + 1, E.dim, E.m.kind, false);
        uint32_t counts[2] = {0, 0};
        float l = 0.f;
        EMBER_CUDA(cudaMemcpyAsync(counts, E.s.nunique, sizeof(counts), cudaMemcpyDeviceToHost, E.stream));
        EMBER_CUDA(cudaMemcpyAsync(&l, E.s.loss, sizeof(float), cudaMemcpyDeviceToHost, E.stream));
        EMBER_CUDA(cudaStreamSynchronize(E.stream));
        E.check_finite();
        if (n_node) *n_node = counts[0];
        if (n_rel) *n_rel = E.m.kind == EMBER_DOT ? 0 : counts[1];
        if (loss) *loss = l;
    });
}

int ember_adagrad_apply(ember_ctx* ctx, const uint32_t* ids, const float* rows, uint32_t n, uint32_t i, uint32_t j,
                        int relations) {
    return guarded([&] {
        Engine& E = eng(ctx);
        if (!n) return;
        need(ids, "ids_dev");
        need(rows, "rows_dev");
        uint32_t* bad = nullptr;
        EMBER_CUDA(cudaMallocAsync(&bad, sizeof(uint32_t), E.stream));
        EMBER_CUDA(cudaMemsetAsync(bad, 0, sizeof(uint32_t), E.stream));
        if (relations) {
            if (!E.rel_theta) throw ConfigError("relation table not bound");
            launch_adagrad_rows(E, ids, rows, n, E.parts[0], E.parts[0], true, bad);
        } else {
            E.check_bucket(i, j);
            launch_adagrad_rows(E, ids, rows, n, E.view(i), E.view(j), false, bad);
        }
        uint32_t nbad = 0;
        EMBER_CUDA(cudaMemcpyAsync(&nbad, bad, sizeof(uint32_t), cudaMemcpyDeviceToHost, E.stream));
        EMBER_CUDA(cudaFreeAsync(bad, E.stream));
        EMBER_CUDA(cudaStreamSynchronize(E.stream));
        if (nbad)
            throw ConfigError(std::to_string(nbad) + (relations ? " relation ids out of range (rows not updated)"
                                                              : " node ids outside partitions i and j (rows not updated)"));
    });
}

int ember_gather(ember_ctx* ctx, const uint32_t* ids, uint32_t n, uint32_t i, uint32_t j, int relations,
                 float* theta_out, float* acc_out) {
    return guarded([&] {
        Engine& E = eng(ctx);
        if (!n) return;
        need(ids, "ids_dev");
        need(theta_out, "theta_out_dev");
        uint32_t* bad = nullptr;
        EMBER_CUDA(cudaMallocAsync(&bad, sizeof(uint32_t), E.stream));
        EMBER_CUDA(cudaMemsetAsync(bad, 0, sizeof(uint32_t), E.stream));
        if (relations) {
            if (!E.rel_theta) throw ConfigError("relation table not bound");
            launch_gather_rows(E, ids, n, E.parts[0], E.parts[0], true, theta_out, acc_out, bad);
        } else {
            E.check_bucket(i, j);
            launch_gather_rows(E, ids, n, E.view(i), E.view(j), false, theta_out, acc_out, bad);
        }
        uint32_t nbad = 0;
        EMBER_CUDA(cudaMemcpyAsync(&nbad, bad, sizeof(uint32_t), cudaMemcpyDeviceToHost, E.stream));
        EMBER_CUDA(cudaFreeAsync(bad, E.stream));
        EMBER_CUDA(cudaStreamSynchronize(E.stream));
        if (nbad)
            throw ConfigError(std::to_string(nbad) + (relations ? " relation ids out of range"
                                                              : " node ids outside partitions i and j"));
    });
}

int ember_debug_scores(ember_ctx* ctx, const uint32_t* edges, uint32_t nb, uint32_t i, uint32_t j,
                       const uint32_t* negs, int side, uint32_t rows, float* out) {
    return guarded([&] {
        Engine& E = eng(ctx);
        if (side != 0 && side != 1) throw ConfigError("side must be 0 or 1");
        if (rows > nb || nb > E.cap_b) throw ConfigError("rows <= nb <= batch_size");
        E.check_bucket(i, j);
        launch_debug_scores(E, edges, nb, negs, side, rows, out, E.view(i), E.view(j));
    });
}

int ember_debug_sort_slots(ember_ctx* ctx, const uint32_t* keys, uint32_t n, uint32_t bits, uint32_t* keys_sorted,
                           uint32_t* vals_sorted, uint32_t* rank, uint8_t* uniq, uint32_t* ukeys, uint32_t* offsets,
                           uint32_t* nruns) {
    return guarded([&] {
        Engine& E = eng(ctx);
        if (n > E.cap_rows) throw ConfigError("n exceeds the context's gradient slots (3 batch_size + n_neg)");
        if (bits < 1 || bits > 32) throw ConfigError("bits must be in [1, 32]");
        if (n) need(keys, "keys_dev");
        const size_t b4 = (size_t)n * sizeof(uint32_t);
        EMBER_CUDA(cudaMemcpyAsync(E.s.keys, keys, b4, cudaMemcpyDeviceToDevice, E.stream));
        EMBER_CUDA(cudaEventRecord(E.ev_fork, E.stream));
        EMBER_CUDA(cudaStreamWaitEvent(E.side, E.ev_fork, 0));
        launch_slot_sort(E, n, bits, ~0u);
        EMBER_CUDA(cudaEventRecord(E.ev_sorted, E.side));
        EMBER_CUDA(cudaStreamWaitEvent(E.stream, E.ev_sorted, 0));
        auto out = [&](void* dst, const void* src, size_t bytes) {
            if (dst && bytes) EMBER_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, E.stream));
        };
        out(keys_sorted, E.s.keys_sorted, b4);
        out(vals_sorted, E.s.vals_sorted, b4);
        out(rank, E.s.rank, b4);
        out(uniq, E.s.uniq, n);
        out(ukeys, E.s.ukeys, b4);
        out(offsets, E.s.offsets, b4 + sizeof(uint32_t));
        out(nruns, E.s.nruns, sizeof(uint32_t));
    });
}

int ember_eval_ranks(ember_ctx* ctx, const uint32_t* test, uint32_t n_test, const uint32_t* train, uint64_t n_train,
                     uint32_t n_eval, float alpha_eval, uint32_t block, uint64_t eval_seed, uint32_t* ranks) {
    return guarded([&] {
        Engine& E = eng(ctx);
        need(test, "test_edges_dev");
        need(ranks, "ranks_dev");
        launch_eval(E, test, n_test, train, n_train, n_eval, alpha_eval, block ? block : 1, eval_seed, ranks);
    });
}

int ember_eval_ranks_filtered(ember_ctx* ctx, const uint32_t* test, uint32_t n_test, const uint64_t* keys,
                              uint64_t n_keys, uint32_t* ranks) {
    return guarded([&] {
        Engine& E = eng(ctx);
        need(test, "test_edges_dev");
        need(ranks, "ranks_dev");
        if (n_keys) need(keys, "filter_keys_dev");
        launch_eval_filtered(E, test, n_test, keys, n_keys, ranks);
    });
}

int ember_make_plan(int kind, uint32_t p, uint32_t c, uint64_t seed, uint32_t* seq, uint64_t* swap_count,
                    uint32_t* adm, uint32_t* n_adm, uint32_t* swaps, uint32_t* state) {
    return guarded([&] {
        if (kind < 0 || kind > 3) throw ConfigError("unknown ordering kind");
        const OrderingPlan plan = make_plan(static_cast<OrderingKind>(kind), p, c, seed);
        plan.validate();
        for (size_t t = 0; t < plan.bucket_sequence.size(); ++t) {
            if (seq) {
                seq[2 * t] = plan.bucket_sequence[t].i;
                seq[2 * t + 1] = plan.bucket_sequence[t].j;
            }
            if (state) state[t] = plan.bucket_state[t];
        }
        if (swap_count) *swap_count = plan.swap_count;
        if (n_adm) *n_adm = (uint32_t)plan.admission_schedule.size();
        if (adm) std::memcpy(adm, plan.admission_schedule.data(), plan.admission_schedule.size() * sizeof(uint32_t));
        if (swaps)
            for (size_t k = 0; k < plan.swap_events.size(); ++k) {
                swaps[3 * k] = plan.swap_events[k].step;
                swaps[3 * k + 1] = plan.swap_events[k].evicted;
                swaps[3 * k + 2] = plan.swap_events[k].admitted;
            }
    });
}

uint64_t ember_lower_bound_swaps(uint32_t p, uint32_t c) {
    uint64_t r = ~0ULL;
    guarded([&] { r = lower_bound_swaps(p, c); });
    return r;
}

uint64_t ember_elimination_swap_formula(uint32_t p, uint32_t c) {
    uint64_t r = ~0ULL;
    guarded([&] { r = elimination_swap_formula(p, c); });
    return r;
}

int ember_graph_generate(int device, uint64_t V, uint32_t R, uint64_t n, uint64_t seed, float train, float valid,
                         uint32_t* edges, uint8_t* split) {
    return guarded([&] {
        need(edges, "edges_out");
        graph_generate(device, V, R, n, seed, train, valid, edges, split);
    });
}

int ember_graph_bucket(int device, uint64_t V, uint32_t p, const uint32_t* in, uint64_t n, uint32_t* out,
                       uint64_t* offsets) {
    return guarded([&] {
        need(in, "edges_in");
        need(out, "edges_out");
        need(offsets, "offsets_out");
        graph_bucket(device, V, p, in, n, out, offsets);
    });
}

int ember_graph_preprocess(int device, const uint32_t* raw, uint64_t n, uint32_t p, uint64_t seed, float train_frac,
                           float valid_frac, uint32_t* train_out, uint64_t* offsets, uint32_t* valid_out,
                           uint32_t* test_out, uint64_t* counts, uint32_t* node_tokens, uint32_t* rel_tokens,
                           uint64_t* num_nodes, uint32_t* num_rel) {
    return guarded([&] {
        need(raw, "raw_dev");
        need(train_out, "train_out_dev");
        need(offsets, "offsets_host");
        need(counts, "counts_host");
        need(num_nodes, "num_nodes_host");
        need(num_rel, "num_relations_host");
        graph_preprocess(device, raw, n, p, seed, train_frac, valid_frac, train_out, offsets, valid_out, test_out,
                         counts, node_tokens, rel_tokens, num_nodes, num_rel);
    });
}

int ember_tc_selftest(int device, int mode, int K, int N, uint64_t seed, double* err) {
    return guarded([&] {
        need(err, "max_rel_err_out");
        *err = tc_selftest(device, mode, K, N, seed);
    });
}

int ember_tc_mmabench(int device, int mode, int N, int iters, double* cycles_per_mma) {
    return guarded([&] {
        need(cycles_per_mma, "cycles_per_mma");
        if (N % 16 || N < 16 || N > 256 || iters < 1) throw ConfigError("mmabench: N multiple of 16 in [16, 256]");
        *cycles_per_mma = tc_mmabench(device, mode % 16, N, iters, mode / 16 + 1);
    });
}

int ember_profile_enable(ember_ctx* ctx, int enable) {
    return guarded([&] { eng(ctx).prof_on = enable != 0; });
}

int ember_profile_read(ember_ctx* ctx, double* ms_out, uint64_t* launches_out, uint64_t* lib_calls_out) {
    return guarded([&] {
        Engine& E = eng(ctx);
        const std::vector<double> ms = E.profile_read();
        if (ms_out)
            for (size_t k = 0; k < ms.size(); ++k) ms_out[k] = ms[k];
        if (launches_out) *launches_out = E.launches;
        if (lib_calls_out) *lib_calls_out = E.lib_calls;
    });
}

int ember_buffer_create(ember_ctx* ctx, uint32_t capacity, const uint32_t* seq, uint32_t steps,
                        float* const* host_theta, float* const* host_acc, ember_buffer** out) {
    return guarded([&] {
        Engine& E = eng(ctx);
        need(seq, "seq");
        need(host_theta, "host_theta");
        need(host_acc, "host_acc");
        need(out, "out");
        *out = nullptr;
        PartitionBuffer* B = buffer_create(E, capacity, seq, steps, host_theta, host_acc);
        *out = new ember_buffer{B, ctx};
    });
}

int ember_buffer_destroy(ember_buffer* b) {
    return guarded([&] {
        if (!b) return;
        if (b->b) buffer_destroy(b->b);
        delete b;
    });
}

int ember_buffer_acquire(ember_buffer* b, uint32_t step, uint32_t* i, uint32_t* j) {
    return guarded([&] { buffer_acquire(&buf(b), step, i, j); });
}

int ember_buffer_release(ember_buffer* b, uint32_t step) {
    return guarded([&] { buffer_release(&buf(b), step); });
}

int ember_buffer_flush(ember_buffer* b) {
    return guarded([&] { buffer_flush(&buf(b)); });
}

int ember_buffer_stats(ember_buffer* b, ember_buffer_report* out) {
    return guarded([&] {
        need(out, "out");
        buffer_stats(&buf(b), out);
    });
}

int ember_buffer_decisions(ember_buffer* b, uint32_t* out, uint32_t* n) {
    return guarded([&] {
        const uint32_t k = buffer_decisions(&buf(b), out);
        if (n) *n = k;
    });
}


int ember_train_epoch_buffered(ember_ctx* ctx, ember_buffer* b, const uint32_t* edges, const uint64_t* offsets,
                               uint64_t epoch, ember_step_stats* stats) {
    return guarded([&] {
        Engine& E = eng(ctx);
        PartitionBuffer& B = buf(b);
        if (&buffer_engine(&B) != &E) throw ConfigError("buffer belongs to another context");
        need(edges, "edges_dev");
        need(offsets, "offsets_host");
        train_epoch_impl(
            E, edges, offsets, nullptr, epoch, stats, [&](uint32_t t, uint32_t* i, uint32_t* j) { buffer_acquire(&B, t, i, j); },
            [&](uint32_t t) { buffer_release(&B, t); });
    });
}

int ember_train_epoch(ember_ctx* ctx, const uint32_t* edges, const uint64_t* offsets, const uint32_t* seq,
                      uint64_t epoch, ember_step_stats* stats) {
    return guarded([&] {
        Engine& E = eng(ctx);
        need(edges, "edges_dev");
        need(offsets, "offsets_host");
        need(seq, "seq");
        for (uint32_t k = 0; k < E.g.num_partitions; ++k) E.view(k);  // every partition bound
        train_epoch_impl(E, edges, offsets, seq, epoch, stats, [](uint32_t, uint32_t*, uint32_t*) {},
                         [](uint32_t) {});
    });
}

int ember_make_rounds(uint32_t p, uint32_t world, uint32_t* order, uint32_t* round, uint32_t* rank, uint32_t* holder,
                      uint32_t* n_rounds) {
    return guarded([&] {
        const RoundSchedule S = make_rounds(p, world);
        if (order) std::memcpy(order, S.order.data(), S.order.size() * sizeof(uint32_t));
        if (round) std::memcpy(round, S.round.data(), S.round.size() * sizeof(uint32_t));
        if (rank) std::memcpy(rank, S.rank.data(), S.rank.size() * sizeof(uint32_t));
        if (holder) std::memcpy(holder, S.holder.data(), S.holder.size() * sizeof(uint32_t));
        if (n_rounds) *n_rounds = S.rounds;
    });
}

int ember_make_rounds_overlap(uint32_t p, uint32_t world, uint32_t* order, uint32_t* round, uint32_t* rank,
                              uint8_t* early, uint32_t* holder, uint32_t* n_rounds) {
    return guarded([&] {
        const RoundSchedule S = make_rounds_overlap(p, world);
        if (order) std::memcpy(order, S.order.data(), S.order.size() * sizeof(uint32_t));
        if (round) std::memcpy(round, S.round.data(), S.round.size() * sizeof(uint32_t));
        if (rank) std::memcpy(rank, S.rank.data(), S.rank.size() * sizeof(uint32_t));
        if (early) std::memcpy(early, S.early.data(), S.early.size());
        if (holder) std::memcpy(holder, S.holder.data(), S.holder.size() * sizeof(uint32_t));
        if (n_rounds) *n_rounds = S.rounds;
    });
}

int ember_relations_external(ember_ctx* ctx, float* grad) {
    return guarded([&] {
        Engine& E = eng(ctx);
        if (grad && (reinterpret_cast<uintptr_t>(grad) & 15)) throw ConfigError("grad_dev must be 16-byte aligned");
        E.rel_ext = grad;
    });
}

int ember_relations_apply_dense(ember_ctx* ctx, const float* grad) {
    return guarded([&] {
        Engine& E = eng(ctx);
        need(grad, "grad_dev");
        E.apply_relations_dense(grad);
    });
}

int ember_overflow_rows(ember_ctx* ctx, uint64_t* total) {
    return guarded([&] {
        need(total, "total");
        *total = tc_overflow_rows(eng(ctx));
    });
}

int ember_comm_init(ember_ctx* ctx, const void* id, int rank, int world) {
    return guarded([&] {
        Engine& E = eng(ctx);
        need(id, "nccl_unique_id");
        E.comm_init(id, rank, world);
    });
}

int ember_comm_barrier(ember_ctx* ctx) {
    return guarded([&] {
        Engine& E = eng(ctx);
        EMBER_CUDA(cudaStreamSynchronize(E.stream));
    });
}

int ember_partition_copy(ember_ctx* ctx, float* dst_theta, float* dst_acc, int dst_device, const float* src_theta,
                         const float* src_acc, int src_device, uint64_t rows) {
    return guarded([&] {
        Engine& E = eng(ctx);
        const size_t bytes = (size_t)rows * E.dim * sizeof(float);
        if (dst_device == src_device) {
            EMBER_CUDA(cudaMemcpyAsync(dst_theta, src_theta, bytes, cudaMemcpyDeviceToDevice, E.stream));
            EMBER_CUDA(cudaMemcpyAsync(dst_acc, src_acc, bytes, cudaMemcpyDeviceToDevice, E.stream));
        } else {
            EMBER_CUDA(cudaMemcpyPeerAsync(dst_theta, dst_device, src_theta, src_device, bytes, E.stream));
            EMBER_CUDA(cudaMemcpyPeerAsync(dst_acc, dst_device, src_acc, src_device, bytes, E.stream));
        }
    });
}

}  // extern "C"
