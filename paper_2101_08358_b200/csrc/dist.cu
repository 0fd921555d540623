// SPDX-License-Identifier: Apache-2.0
//
// train_epoch_partitioned over G GPUs on the device (Algorithm 2,
// PAPER.md:164-188): one process per GPU, the round loop in host C++ (host/dist_driver.cpp), and
// this rank's work on its GPU:
//   * step: Engine::step (the full training step; with world > 1 the relation gradient is summed
//     densely, all-reduced by NCCL on the step stream and applied by the dense Adagrad, so the
//     relation replicas stay bit-identical), or Engine::idle_step when the rank is out of batches;
//   * handoff: one NCCL group of ncclSend/ncclRecv of whole partitions (theta then acc) on a
//     separate copy stream and a second communicator, issued at the schedule's handoff point (with
//     the overlapped schedule: after the departing pair's buckets, so the copy runs while the
//     staying pair trains); the step stream waits for it only before the next round;
//   * tables: `slots` device slots of the largest partition (theta + acc), as many as the rank
//     holds plus the most it receives in one handoff; a partition lives in one slot at a time and
//     is bound into the Engine while it is held.
// The C callback form (ember_dist_run) runs the same loop with the caller's rank ops: the CPU
// tests drive it with the oracle and gloo.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <functional>
#include <memory>
#include <vector>

#include "engine.h"
#include "host/dist_driver.h"
#include "host/rounds.h"

namespace ember {

Engine& engine_of(ember_ctx* ctx);                   // capi.cu
int guarded_status(const std::function<void()>& f);  // capi.cu: exceptions -> status codes

namespace {

uint64_t part_rows(const ember_graph_desc& g, uint32_t k) {
    const uint64_t q = g.num_nodes / g.num_partitions, r = g.num_nodes % g.num_partitions;
    return q + (k < r ? 1 : 0);
}

struct DistGpu final : RankOps {
    Engine& E;
    uint32_t rank, world, p;
    const uint32_t* edges = nullptr;
    void* p2p = nullptr;  // handoff communicator (world > 1)
    cudaStream_t copy = nullptr;
    cudaEvent_t ev_compute = nullptr, ev_copied = nullptr;
    uint64_t max_rows = 0, slot_floats = 0;
    std::vector<float*> slot_base;  // slot -> theta (acc follows at + max_rows * dim)
    std::vector<int> slot_of, pending;  // partition -> slot held / slot receiving (-1: none)
    std::vector<uint32_t> free_slots;
    uint64_t sent_bytes = 0;

    DistGpu(Engine& e, uint32_t r, uint32_t w, uint32_t parts) : E(e), rank(r), world(w), p(parts) {}

    ~DistGpu() override {
        if (copy) cudaStreamSynchronize(copy);
        for (uint32_t k = 0; k < p && k < E.parts.size(); ++k)
            if (slot_of[k] >= 0) E.parts[k].theta = E.parts[k].acc = nullptr;
        for (float* b : slot_base) cudaFree(b);
        if (ev_compute) cudaEventDestroy(ev_compute);
        if (ev_copied) cudaEventDestroy(ev_copied);
        if (copy) cudaStreamDestroy(copy);
        nccl_comm_destroy(p2p);
    }

    float* th(int slot) const { return slot_base[slot]; }
    float* ac(int slot) const { return slot_base[slot] + max_rows * E.dim; }

    void bind(uint32_t x, int slot) {
        slot_of[x] = slot;
        E.parts[x].theta = th(slot);
        E.parts[x].acc = ac(slot);
    }

    void step(const BatchRef* b, uint64_t epoch) override {
        if (b)
            E.train_batch(edges + 3 * b->lo, b->hi - b->lo, b->begin, b->nb, b->i, b->j, epoch, b->bucket_step,
                          b->batch_in_bucket, nullptr);
        else
            E.idle_step();
    }

    void send_recv(uint32_t, const std::vector<Move>& mv) override {
        EMBER_CUDA(cudaEventRecord(ev_compute, E.stream));  // the departing partitions' last steps
        EMBER_CUDA(cudaStreamWaitEvent(copy, ev_compute, 0));
        std::vector<std::pair<uint32_t, int>> incoming, outgoing;
        for (const Move& m : mv) {
            if (m.dst == rank) {
                if (free_slots.empty()) throw EmberError("dist: no free partition slot for an arriving partition");
                incoming.emplace_back(m.part, (int)free_slots.back());
                free_slots.pop_back();
            } else if (m.src == rank) {
                if (slot_of[m.part] < 0) throw EmberError("dist: sending a partition this rank does not hold");
                outgoing.emplace_back(m.part, slot_of[m.part]);
            }
        }
        nccl_group(true);
        for (const Move& m : mv) {
            const uint64_t n = part_rows(E.g, m.part) * E.dim;
            if (m.src == rank) {
                const int s = slot_of[m.part];
                nccl_send_f32(th(s), n, (int)m.dst, p2p, copy);
                nccl_send_f32(ac(s), n, (int)m.dst, p2p, copy);
                sent_bytes += 2 * n * sizeof(float);
            } else if (m.dst == rank) {
                int s = -1;
                for (auto& in : incoming)
                    if (in.first == m.part) s = in.second;
                nccl_recv_f32(th(s), n, (int)m.src, p2p, copy);
                nccl_recv_f32(ac(s), n, (int)m.src, p2p, copy);
            }
        }
        nccl_group(false);
        EMBER_CUDA(cudaEventRecord(ev_copied, copy));
        for (auto& in : incoming) pending[in.first] = in.second;
        // departing slots: reusable by later receives (ordered after this group on the copy stream)
        for (auto& out : outgoing) {
            slot_of[out.first] = -1;
            E.parts[out.first].theta = E.parts[out.first].acc = nullptr;
            free_slots.push_back((uint32_t)out.second);
        }
    }

    void acquire(uint32_t, const std::vector<uint32_t>& arrived) override {
        bool waited = false;
        for (uint32_t x : arrived) {
            if (pending[x] < 0) continue;
            if (!waited) EMBER_CUDA(cudaStreamWaitEvent(E.stream, ev_copied, 0));
            waited = true;
            bind(x, pending[x]);
            pending[x] = -1;
        }
    }
};

}  // namespace

struct DistHandle {
    std::unique_ptr<DistDriver> drv;
    std::unique_ptr<DistGpu> ops;
    DistReport last{};
};

}  // namespace ember

using namespace ember;

struct ember_dist : DistHandle {};

namespace {

template <typename F>
int dguard(F&& f) {
    return guarded_status(std::function<void()>(f));
}

RoundSchedule schedule_for(uint32_t p, uint32_t world, int overlap) {
    return overlap ? make_rounds_overlap(p, world) : make_rounds(p, world);
}

void fill_report(const DistReport& r, ember_dist_report* out) {
    if (!out) return;
    out->steps = r.steps;
    out->batches = r.batches;
    out->edges = r.edges;
    out->handoffs = r.handoffs;
    out->moved_partitions = r.moved_partitions;
    out->early_handoffs = r.early_handoffs;
}

// C callbacks as RankOps
struct CallbackOps final : RankOps {
    const ember_rank_ops* o;
    explicit CallbackOps(const ember_rank_ops* ops) : o(ops) {}
    static void ok(int rc, const char* what) {
        if (rc) throw EmberError(std::string("rank op ") + what + " failed (" + std::to_string(rc) + ")");
    }
    void step(const BatchRef* b, uint64_t epoch) override {
        if (!b) return ok(o->step(o->user, nullptr, epoch), "step");
        ember_batch_ref r{b->bucket_step, b->i, b->j, b->batch_in_bucket, b->lo, b->hi, b->begin, b->nb, 0};
        ok(o->step(o->user, &r, epoch), "step");
    }
    void send_recv(uint32_t round, const std::vector<Move>& mv) override {
        std::vector<uint32_t> flat;
        for (const Move& m : mv) flat.insert(flat.end(), {m.part, m.src, m.dst});
        ok(o->send_recv(o->user, round, flat.data(), (uint32_t)mv.size()), "send_recv");
    }
    void acquire(uint32_t round, const std::vector<uint32_t>& arrived) override {
        if (o->acquire) ok(o->acquire(o->user, round, arrived.data(), (uint32_t)arrived.size()), "acquire");
    }
};

}  // namespace

extern "C" {

int ember_dist_plan(uint32_t p, uint32_t world, uint32_t rank, int overlap, const uint64_t* offsets,
                    uint32_t batch_size, uint32_t* steps_per_round, uint32_t* handoff_step, uint64_t* total_steps) {
    return dguard([&] {
        DistDriver d(schedule_for(p, world, overlap), offsets, batch_size, rank);
        for (uint32_t r = 0; r < d.rounds(); ++r) {
            if (steps_per_round) steps_per_round[r] = d.steps_in_round(r);
            if (handoff_step) handoff_step[r] = d.handoff_step(r);
        }
        if (total_steps) *total_steps = d.total_steps();
    });
}

int ember_dist_run(uint32_t p, uint32_t world, uint32_t rank, int overlap, const uint64_t* offsets,
                   uint32_t batch_size, uint64_t epoch, uint64_t first_step, uint64_t n_steps,
                   const ember_rank_ops* ops, ember_dist_report* out) {
    return dguard([&] {
        if (!ops || !ops->step || !ops->send_recv) throw ConfigError("rank ops: step and send_recv are required");
        DistDriver d(schedule_for(p, world, overlap), offsets, batch_size, rank);
        CallbackOps cb(ops);
        fill_report(d.run(cb, epoch, first_step, n_steps), out);
    });
}

int ember_dist_create(ember_ctx* ctx, uint32_t rank, uint32_t world, int overlap, const void* nccl_id_steps,
                      const void* nccl_id_handoff, const uint32_t* edges_dev, const uint64_t* offsets_host,
                      ember_dist** out) {
    return dguard([&] {
        Engine& E = engine_of(ctx);
        if (!out) throw ConfigError("out is null");
        if (!edges_dev) throw ConfigError("edges_dev is null");
        const uint32_t p = E.g.num_partitions;
        if (world > 1 && (!nccl_id_steps || !nccl_id_handoff)) throw ConfigError("world > 1 needs two NCCL unique ids");
        auto h = std::make_unique<ember_dist>();
        h->drv = std::make_unique<DistDriver>(schedule_for(p, world, overlap), offsets_host, E.m.batch_size, rank);
        const RoundSchedule& S = h->drv->schedule();
        auto ops = std::make_unique<DistGpu>(E, rank, world, p);
        ops->edges = edges_dev;
        ops->slot_of.assign(p, -1);
        ops->pending.assign(p, -1);
        // slots: the most partitions this rank holds in a round + the most it receives in one handoff
        uint32_t need = 0;
        for (uint32_t r = 0; r < S.rounds; ++r) {
            uint32_t held = 0, in = 0;
            for (uint32_t x = 0; x < p; ++x) held += S.holder[(size_t)r * p + x] == rank;
            for (const Move& m : h->drv->moves(r)) in += m.dst == rank;
            need = std::max(need, held + in);
        }
        for (uint32_t k = 0; k < p; ++k) ops->max_rows = std::max(ops->max_rows, part_rows(E.g, k));
        EMBER_CUDA(cudaSetDevice(E.device));
        for (uint32_t s = 0; s < need; ++s) {
            float* b = nullptr;
            EMBER_CUDA(cudaMalloc(&b, 2 * ops->max_rows * E.dim * sizeof(float)));
            ops->slot_base.push_back(b);
        }
        for (uint32_t s = need; s-- > 0;) ops->free_slots.push_back(s);
        for (uint32_t x = 0; x < p; ++x)  // round 0: bind the partitions this rank starts with
            if (S.holder[x] == rank) {
                ops->bind(x, (int)ops->free_slots.back());
                ops->free_slots.pop_back();
            }
        EMBER_CUDA(cudaStreamCreateWithFlags(&ops->copy, cudaStreamNonBlocking));
        EMBER_CUDA(cudaEventCreateWithFlags(&ops->ev_compute, cudaEventDisableTiming));
        EMBER_CUDA(cudaEventCreateWithFlags(&ops->ev_copied, cudaEventDisableTiming));
        if (world > 1) {
            E.comm_init(nccl_id_steps, (int)rank, (int)world);  // relation all-reduce on the step stream
            ops->p2p = nccl_comm_create(nccl_id_handoff, (int)rank, (int)world);
        }
        h->ops = std::move(ops);
        *out = h.release();
    });
}

int ember_dist_destroy(ember_dist* d) {
    return dguard([&] { delete d; });
}

int ember_dist_init_embeddings(ember_dist* d, uint64_t seed) {
    return dguard([&] {
        if (!d) throw ConfigError("dist is null");
        Engine& E = d->ops->E;
        for (uint32_t x = 0; x < d->ops->p; ++x)
            if (d->ops->slot_of[x] >= 0) {
                const PartView v = E.parts[x];
                launch_init_rows(E.stream, v.theta, v.acc, v.first, v.rows, E.dim, E.m.kind, seed);
            }
        if (E.rel_theta)
            launch_init_rows(E.stream, E.rel_theta, E.rel_acc, 0, E.g.num_relations, E.dim, E.m.kind,
                             seed ^ 0x52454cULL);
    });
}

int ember_dist_train_epoch(ember_dist* d, uint64_t epoch, uint64_t first_step, uint64_t n_steps,
                           ember_dist_report* out) {
    return dguard([&] {
        if (!d) throw ConfigError("dist is null");
        NvtxRange nvtx("ember::dist_epoch");
        d->last = d->drv->run(*d->ops, epoch, first_step, n_steps);
        fill_report(d->last, out);
        if (out) out->handoff_bytes = d->ops->sent_bytes;
    });
}

int ember_dist_tables(ember_dist* d, uint32_t part, float** theta_dev, float** acc_dev) {
    return dguard([&] {
        if (!d) throw ConfigError("dist is null");
        if (part >= d->ops->p) throw ConfigError("partition id out of range");
        const int s = d->ops->slot_of[part];
        if (theta_dev) *theta_dev = s >= 0 ? d->ops->th(s) : nullptr;
        if (acc_dev) *acc_dev = s >= 0 ? d->ops->ac(s) : nullptr;
    });
}

int ember_nccl_unique_id(void* out128) {
    return dguard([&] {
        if (!out128) throw ConfigError("out is null");
        nccl_unique_id(out128);
    });
}

int ember_dist_loss(ember_dist* d, float* loss_host) {
    return dguard([&] {
        if (!d || !loss_host) throw ConfigError("dist / loss_host is null");
        Engine& E = d->ops->E;
        EMBER_CUDA(cudaMemcpyAsync(loss_host, E.s.loss, sizeof(float), cudaMemcpyDeviceToHost, E.stream));
        EMBER_CUDA(cudaStreamSynchronize(E.stream));
    });
}

int ember_dist_synchronize(ember_dist* d) {
    return dguard([&] {
        if (!d) throw ConfigError("dist is null");
        EMBER_CUDA(cudaStreamSynchronize(d->ops->copy));
        EMBER_CUDA(cudaStreamSynchronize(d->ops->E.stream));
        d->ops->E.check_finite();
    });
}

}  // extern "C"
