// SPDX-License-Identifier: Apache-2.0
//
// Device partition buffer (SPEC.md:296-357 [MODULE] buffer; §4.2, Algorithm 2).
//
// HBM is the buffer, pinned host memory is the backing store. The buffer holds c resident
// partition slots plus exactly 2 staging slots ("c resident blocks plus exactly 2
// staging blocks"), each a [rows_max x dim] theta block followed by its acc block. The
// OrderingPlan is known in advance, so every decision is made up front by the buffer's own
// Belady replay (furthest next use, ties to the lower id) and turned into a
// static copy schedule on two copy streams:
//
//   writeback k  (D2H, wb stream):   evictee y_k, once the compute stream has released y_k's
//                                    last use before its eviction step (dead from then on);
//   load k       (H2D, load stream): admission x_k into the slot freed by writeback k-2 (the
//                                    two staging slots for k = 0, 1), after that writeback and
//                                    after any earlier writeback of x_k itself (host RAW);
//   compute at the eviction step t_k waits on load k.
//
// Loads are issued as soon as their dependencies are issued, so each prefetch runs ahead of
// the computation while at most c + 2 slots exist. The epoch's initial
// fill is waited for per partition at its first use, and the epoch-end flush of each final
// resident starts right after its last use, so both overlap the computation as well. All copies and waits
// are stream-ordered; the host blocks only in flush() and stats(). Stall time = compute waiting
// on a load, measured on the device (event on the compute stream before the wait vs the load's
// completion event).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "engine.h"

namespace ember {

struct PartitionBuffer {
    Engine* E = nullptr;
    uint32_t p = 0, c = 0, steps = 0;
    std::vector<uint32_t> seq;  // 2 per step
    std::vector<float*> host_theta, host_acc;
    uint64_t rows_max = 0;
    size_t slot_bytes = 0;        // theta + acc of one slot
    std::vector<char*> slot;      // c + 2 device slots
    cudaStream_t load_st = nullptr, wb_st = nullptr;

    struct Swap {
        uint32_t step, evicted, admitted;
        uint32_t last_use;   // evictee's last use before `step`
        int prev_wb;         // earlier swap this epoch that wrote `admitted` back (-1: none)
        uint32_t slot;       // slot the admission is loaded into
        uint32_t freed;      // slot the evictee occupied
    };
    std::vector<uint32_t> fill;            // first c admissions, in order (slot m <- fill[m])
    std::vector<Swap> swaps;
    std::vector<std::vector<uint32_t>> wb_at;  // step -> swaps whose evictee is released there
    std::vector<std::vector<uint32_t>> flush_at;  // step -> final residents whose last use it is
    std::vector<int> final_slot;                  // partition -> slot at epoch end (-1: not resident)

    // per-epoch progress
    uint32_t cursor = 0;
    size_t wb_issued = 0, load_issued = 0;
    bool in_epoch = false;
    std::vector<int> slot_of;  // partition -> slot while resident (plan state), -1 otherwise
    std::vector<uint8_t> wb_ready;  // swap -> its writeback has been issued
    std::vector<uint8_t> waited;    // swap -> the compute stream waited on its load, stall not yet read
    std::vector<uint8_t> fill_pending;  // partition -> compute has not yet waited for its fill load
    std::vector<cudaEvent_t> ev_release, ev_wb, ev_load, ev_need, ev_fill, ev_fillm;

    uint64_t reads = 0, writes = 0, bytes_read = 0, bytes_written = 0, epochs = 0;
    double stall_ms = 0.0;
    uint32_t stalls = 0;

    uint64_t part_rows(uint32_t k) const { return partition_size(E->g.num_nodes, p, k); }
    float* theta_of(uint32_t s) const { return reinterpret_cast<float*>(slot[s]); }
    float* acc_of(uint32_t s) const { return reinterpret_cast<float*>(slot[s] + slot_bytes / 2); }

    void plan_schedule() {
        std::vector<std::vector<uint32_t>> uses(p);
        for (uint32_t t = 0; t < steps; ++t) {
            const uint32_t i = seq[2 * t], j = seq[2 * t + 1];
            uses[i].push_back(t);
            if (j != i) uses[j].push_back(t);
        }
        auto next_use = [&](uint32_t x, uint32_t t) -> uint64_t {
            auto it = std::lower_bound(uses[x].begin(), uses[x].end(), t);
            return it == uses[x].end() ? ~0ULL : *it;
        };
        std::vector<uint8_t> resident(p, 0);
        std::vector<int> last_wb(p, -1), where(p, -1);
        fill.clear();
        swaps.clear();
        wb_at.assign(steps, {});
        for (uint32_t t = 0; t < steps; ++t) {
            const uint32_t i = seq[2 * t], j = seq[2 * t + 1];
            for (uint32_t need : {i, j}) {
                if (resident[need]) continue;
                if (fill.size() < c) {
                    where[need] = (int)fill.size();
                    fill.push_back(need);
                    resident[need] = 1;
                    continue;
                }
                bool found = false;
                uint32_t victim = 0;
                uint64_t furthest = 0;
                for (uint32_t x = 0; x < p; ++x) {  // ascending ids: ties go to the lower id
                    if (!resident[x] || x == i || x == j) continue;
                    const uint64_t nu = next_use(x, t);
                    if (!found || nu > furthest) {
                        found = true;
                        victim = x;
                        furthest = nu;
                    }
                }
                if (!found) throw ConfigError("buffer: no evictable partition (capacity too small)");
                const size_t k = swaps.size();
                Swap s;
                s.step = t;
                s.evicted = victim;
                s.admitted = need;
                auto it = std::lower_bound(uses[victim].begin(), uses[victim].end(), t);
                if (it == uses[victim].begin()) throw EmberError("buffer: evictee never used");
                s.last_use = *(it - 1);
                s.prev_wb = last_wb[need];
                s.freed = (uint32_t)where[victim];
                s.slot = k < 2 ? c + (uint32_t)k : swaps[k - 2].freed;
                swaps.push_back(s);
                wb_at[s.last_use].push_back((uint32_t)k);
                last_wb[victim] = (int)k;
                resident[victim] = 0;
                where[victim] = -1;
                resident[need] = 1;
                where[need] = (int)s.slot;
            }
        }
        // epoch-end flush: each final resident is written back right after its last use
        flush_at.assign(steps, {});
        final_slot = where;
        for (uint32_t x = 0; x < p; ++x)
            if (where[x] >= 0) flush_at[uses[x].back()].push_back(x);
    }

    void bind(uint32_t part, int s) {
        PartView& v = E->parts[part];
        v.theta = s >= 0 ? theta_of((uint32_t)s) : nullptr;
        v.acc = s >= 0 ? acc_of((uint32_t)s) : nullptr;
    }

    void copy_in(uint32_t part, uint32_t s, cudaStream_t st) {
        const size_t b = (size_t)part_rows(part) * E->dim * sizeof(float);
        EMBER_CUDA(cudaMemcpyAsync(theta_of(s), host_theta[part], b, cudaMemcpyHostToDevice, st));
        EMBER_CUDA(cudaMemcpyAsync(acc_of(s), host_acc[part], b, cudaMemcpyHostToDevice, st));
        ++reads;
        bytes_read += 2 * b;
    }

    void copy_out(uint32_t part, uint32_t s, cudaStream_t st) {
        const size_t b = (size_t)part_rows(part) * E->dim * sizeof(float);
        EMBER_CUDA(cudaMemcpyAsync(host_theta[part], theta_of(s), b, cudaMemcpyDeviceToHost, st));
        EMBER_CUDA(cudaMemcpyAsync(host_acc[part], acc_of(s), b, cudaMemcpyDeviceToHost, st));
        ++writes;
        bytes_written += 2 * b;
    }

    // Issues every load whose dependencies (writeback k-2, the previous writeback of the same
    // partition) have been issued, in admission order.
    void pump_loads() {
        while (load_issued < swaps.size()) {
            const size_t k = load_issued;
            const Swap& s = swaps[k];
            if (k >= 2 && !wb_ready[k - 2]) break;
            if (s.prev_wb >= 0 && !wb_ready[(size_t)s.prev_wb]) break;
            if (k >= 2) EMBER_CUDA(cudaStreamWaitEvent(load_st, ev_wb[k - 2], 0));
            if (s.prev_wb >= 0) EMBER_CUDA(cudaStreamWaitEvent(load_st, ev_wb[(size_t)s.prev_wb], 0));
            copy_in(s.admitted, s.slot, load_st);
            EMBER_CUDA(cudaEventRecord(ev_load[k], load_st));
            ++load_issued;
        }
    }

    void begin_epoch() {
        collect();  // the previous epoch's stall events are reused below
        cursor = 0;
        wb_issued = load_issued = 0;
        wb_ready.assign(swaps.size(), 0);
        waited.assign(swaps.size(), 0);
        slot_of.assign(p, -1);
        for (uint32_t k = 0; k < p; ++k) bind(k, -1);
        // The initial fill on the load stream, each partition with its own completion event (the
        // compute stream waits per partition at its first use). The loads wait for the previous
        // epoch's flush (host read-after-write, slot write-after-read) or, in the first epoch,
        // for the work enqueued before (init).
        if (epochs == 0) {
            EMBER_CUDA(cudaEventRecord(ev_fill[0], E->stream));
            EMBER_CUDA(cudaStreamWaitEvent(load_st, ev_fill[0], 0));
        } else {
            EMBER_CUDA(cudaStreamWaitEvent(load_st, ev_fill[3], 0));
        }
        fill_pending.assign(p, 0);
        for (uint32_t m = 0; m < fill.size(); ++m) {
            copy_in(fill[m], m, load_st);
            EMBER_CUDA(cudaEventRecord(ev_fillm[m], load_st));
            slot_of[fill[m]] = (int)m;
            fill_pending[fill[m]] = 1;
            bind(fill[m], (int)m);
        }
        pump_loads();
        in_epoch = true;
    }

    // Algorithm 2 "acquire": the bucket at `step` becomes resident on the compute stream.
    void acquire(uint32_t step, uint32_t* i_out, uint32_t* j_out) {
        if (step >= steps) throw ConfigError("buffer: step out of range");
        if (!in_epoch) {
            if (step != 0) throw ConfigError("buffer: an epoch starts at step 0");
            begin_epoch();
        }
        if (step != cursor) throw ConfigError("buffer: buckets must be acquired in plan order");
        // swaps at this step, in order: the compute stream waits for the admission's load
        for (size_t k = 0; k < swaps.size(); ++k) {
            const Swap& s = swaps[k];
            if (s.step != step) continue;
            pump_loads();
            if (k >= load_issued) throw EmberError("buffer: load not issuable (schedule bug)");
            EMBER_CUDA(cudaEventRecord(ev_need[k], E->stream));
            EMBER_CUDA(cudaStreamWaitEvent(E->stream, ev_load[k], 0));
            waited[k] = 1;
            bind(s.evicted, -1);
            slot_of[s.evicted] = -1;
            bind(s.admitted, (int)s.slot);
            slot_of[s.admitted] = (int)s.slot;
        }
        const uint32_t i = seq[2 * step], j = seq[2 * step + 1];
        if (slot_of[i] < 0 || slot_of[j] < 0) throw EmberError("buffer: bucket partition not resident");
        for (uint32_t x : {i, j})
            if (fill_pending[x]) {
                EMBER_CUDA(cudaStreamWaitEvent(E->stream, ev_fillm[(uint32_t)slot_of[x]], 0));
                fill_pending[x] = 0;
            }
        if (i_out) *i_out = i;
        if (j_out) *j_out = j;
    }

    // Algorithm 2 "release": the compute stream is done with the bucket; evictees whose last use
    // this was start their writeback, and loads waiting on those writebacks are issued.
    void release(uint32_t step) {
        if (!in_epoch || step != cursor) throw ConfigError("buffer: release out of order");
        EMBER_CUDA(cudaEventRecord(ev_release[step], E->stream));
        for (uint32_t k : wb_at[step]) {
            const Swap& s = swaps[k];
            EMBER_CUDA(cudaStreamWaitEvent(wb_st, ev_release[step], 0));
            copy_out(s.evicted, s.freed, wb_st);
            EMBER_CUDA(cudaEventRecord(ev_wb[k], wb_st));
            wb_ready[k] = 1;
        }
        for (uint32_t x : flush_at[step]) {  // epoch-end writeback of a final resident, overlapped
            EMBER_CUDA(cudaStreamWaitEvent(wb_st, ev_release[step], 0));
            copy_out(x, (uint32_t)final_slot[x], wb_st);
        }
        pump_loads();
        ++cursor;
        if (cursor == steps) end_epoch();
    }

    // Epoch end: every resident (dirty) partition has been written back after its last use
    // (SPEC.md:326, :334); the next epoch's loads wait for these writes, the compute stream does not.
    void end_epoch() {
        EMBER_CUDA(cudaEventRecord(ev_fill[3], wb_st));
        for (uint32_t x = 0; x < p; ++x) bind(x, -1);
        in_epoch = false;
        ++epochs;
    }

    void collect() {
        bool any = false;
        for (uint8_t w : waited) any |= w != 0;
        if (!any) return;
        EMBER_CUDA(cudaStreamSynchronize(E->stream));
        EMBER_CUDA(cudaStreamSynchronize(load_st));
        for (size_t k = 0; k < waited.size(); ++k) {
            if (!waited[k]) continue;
            waited[k] = 0;
            float ms = 0.f;
            EMBER_CUDA(cudaEventElapsedTime(&ms, ev_need[k], ev_load[k]));
            if (ms > 0.f) {
                stall_ms += ms;
                ++stalls;
            }
        }
    }

    // The context stream (and the host) wait until every writeback has landed in host memory.
    void flush() {
        if (in_epoch) throw ConfigError("buffer: flush in the middle of an epoch");
        if (epochs) EMBER_CUDA(cudaStreamWaitEvent(E->stream, ev_fill[3], 0));
        EMBER_CUDA(cudaStreamSynchronize(E->stream));
    }

    ~PartitionBuffer() {
        cudaSetDevice(E->device);
        cudaStreamSynchronize(E->stream);
        if (load_st) cudaStreamSynchronize(load_st);
        if (wb_st) cudaStreamSynchronize(wb_st);
        if (in_epoch)
            for (uint32_t x = 0; x < p; ++x) bind(x, -1);
        for (auto* v : {&ev_release, &ev_wb, &ev_load, &ev_need, &ev_fill, &ev_fillm})
            for (cudaEvent_t e : *v) cudaEventDestroy(e);
        for (char* s : slot) cudaFree(s);
        if (load_st) cudaStreamDestroy(load_st);
        if (wb_st) cudaStreamDestroy(wb_st);
    }
};

PartitionBuffer* buffer_create(Engine& E, uint32_t c, const uint32_t* seq, uint32_t steps, float* const* host_theta,
                               float* const* host_acc) {
    const uint32_t p = E.g.num_partitions;
    if (c < 1 || c > p) throw ConfigError("buffer: capacity must be in [1, p]");
    if (c < 2 && p > 1) throw ConfigError("buffer: capacity must be >= 2 when p > 1");
    if (steps != p * p) throw ConfigError("buffer: the plan must hold p*p buckets");
    std::vector<uint8_t> seen((size_t)p * p, 0);
    for (uint32_t t = 0; t < steps; ++t) {
        const uint32_t i = seq[2 * t], j = seq[2 * t + 1];
        if (i >= p || j >= p || seen[(size_t)i * p + j]++) throw ConfigError("buffer: plan is not a permutation of buckets");
    }
    auto* B = new PartitionBuffer();
    B->E = &E;
    try {
        B->p = p;
        B->c = c;
        B->steps = steps;
        B->seq.assign(seq, seq + 2 * (size_t)steps);
        B->host_theta.assign(host_theta, host_theta + p);
        B->host_acc.assign(host_acc, host_acc + p);
        for (uint32_t k = 0; k < p; ++k)
            if (!B->host_theta[k] || !B->host_acc[k]) throw ConfigError("buffer: every partition needs host theta and acc");
        for (uint32_t k = 0; k < p; ++k) B->rows_max = std::max(B->rows_max, B->part_rows(k));
        B->slot_bytes = 2 * ((B->rows_max * E.dim * sizeof(float) + 255) / 256 * 256);
        B->plan_schedule();
        const uint32_t nslots = c + (p > c ? 2 : 0);
        B->slot.assign(nslots, nullptr);
        for (uint32_t s = 0; s < nslots; ++s) EMBER_CUDA(cudaMalloc(&B->slot[s], B->slot_bytes));
        EMBER_CUDA(cudaStreamCreateWithFlags(&B->load_st, cudaStreamNonBlocking));
        EMBER_CUDA(cudaStreamCreateWithFlags(&B->wb_st, cudaStreamNonBlocking));
        auto mk = [](std::vector<cudaEvent_t>& v, size_t n, bool timing) {
            v.assign(n, nullptr);
            for (auto& e : v) EMBER_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
        };
        mk(B->ev_release, steps, false);
        mk(B->ev_wb, B->swaps.size(), false);
        mk(B->ev_load, B->swaps.size(), true);
        mk(B->ev_need, B->swaps.size(), true);
        mk(B->ev_fill, 4, false);
        mk(B->ev_fillm, c, false);
    } catch (...) {
        delete B;
        throw;
    }
    return B;
}

void buffer_destroy(PartitionBuffer* B) { delete B; }
void buffer_acquire(PartitionBuffer* B, uint32_t step, uint32_t* i, uint32_t* j) { B->acquire(step, i, j); }
void buffer_release(PartitionBuffer* B, uint32_t step) { B->release(step); }
void buffer_flush(PartitionBuffer* B) { B->flush(); }
Engine& buffer_engine(PartitionBuffer* B) { return *B->E; }

void buffer_stats(PartitionBuffer* B, ember_buffer_report* out) {
    B->collect();
    out->reads = B->reads;
    out->writes = B->writes;
    out->bytes_read = B->bytes_read;
    out->bytes_written = B->bytes_written;
    out->swaps_per_epoch = B->swaps.size();
    out->epochs = B->epochs;
    out->stalls = B->stalls;
    out->stall_ms = B->stall_ms;
    out->slots = (uint32_t)B->slot.size();
    out->slot_bytes = B->slot_bytes;
}

uint32_t buffer_decisions(PartitionBuffer* B, uint32_t* out) {
    if (out)
        for (size_t k = 0; k < B->swaps.size(); ++k) {
            out[3 * k] = B->swaps[k].step;
            out[3 * k + 1] = B->swaps[k].evicted;
            out[3 * k + 2] = B->swaps[k].admitted;
        }
    return (uint32_t)B->swaps.size();
}

}  // namespace ember
