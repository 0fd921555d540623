// SPDX-License-Identifier: Apache-2.0
//
// Engine: the device-resident training step (Algorithm 1, PAPER.md:84-99 / SPEC.md:376-384
// train_epoch_sync semantics, bound = 1). Per batch:
//   step stream:   sample + slot keys -+-> gather+adjust -> contraction (scores, LSE, dA, dN) -> chain rule
//                                      |                              (join) ^           -> loss
//   helper stream:                     +-> (key, slot) sort -> runs -------+
//   then one segmented sum over the sorted gradient rows -> Adagrad (relations and nodes;
//   relations synchronously, after an NCCL all-reduce when world > 1).
// The helper stream only overlaps work that the step stream would otherwise serialise; the
// result is identical to a single-stream order. Stage 2/4 transfers of the paper's pipeline
// vanish: parameters stay in HBM.
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "engine.h"

namespace ember {

namespace {

template <typename T>
T* dalloc(size_t n) {
    if (n == 0) n = 1;
    void* p = nullptr;
    EMBER_CUDA(cudaMalloc(&p, n * sizeof(T)));
    return static_cast<T*>(p);
}

uint32_t bits_for(uint64_t n) {
    uint32_t b = 1;
    while (b < 32 && (1ULL << b) < n) ++b;
    return b;
}

// ---- NCCL, loaded at run time so single-GPU use never needs the library -----------------
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*destroy)(ncclComm_t) = nullptr;
    const char* (*err)(ncclResult_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*unique_id)(ncclUniqueId*) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::mutex mu;  // contexts may be created from several host threads
    std::lock_guard<std::mutex> lock(mu);
    if (!api.h) {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names)
            if ((api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!api.h) throw EmberError("NCCL not loadable (libnccl.so.2): " + std::string(dlerror()));
        api.init_rank = reinterpret_cast<decltype(api.init_rank)>(dlsym(api.h, "ncclCommInitRank"));
        api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(api.h, "ncclAllReduce"));
        api.destroy = reinterpret_cast<decltype(api.destroy)>(dlsym(api.h, "ncclCommDestroy"));
        api.err = reinterpret_cast<decltype(api.err)>(dlsym(api.h, "ncclGetErrorString"));
        api.send = reinterpret_cast<decltype(api.send)>(dlsym(api.h, "ncclSend"));
        api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(api.h, "ncclRecv"));
        api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(api.h, "ncclGroupStart"));
        api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(api.h, "ncclGroupEnd"));
        api.unique_id = reinterpret_cast<decltype(api.unique_id)>(dlsym(api.h, "ncclGetUniqueId"));
        if (!api.init_rank || !api.all_reduce || !api.destroy || !api.send || !api.recv || !api.group_start ||
            !api.group_end || !api.unique_id)
            throw EmberError("NCCL symbols missing");
    }
    return api;
}

__global__ void k_adagrad_dense(float* th, float* ac, const float* g, uint64_t n, float lr, float eps) {
    griddep_wait();
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float gi = g[i];
    if (gi == 0.f) return;  // untouched row elements: Adagrad is the identity for g == 0
    const float a = __fadd_rn(ac[i], __fmul_rn(gi, gi));
    ac[i] = a;
    th[i] = __fsub_rn(th[i], __fdiv_rn(__fmul_rn(lr, gi), __fadd_rn(__fsqrt_rn(a), eps)));
}

bool getenv_flag(const char* name) {
    const char* v = getenv(name);
    return v && v[0] == '1';
}

// A/B switch: EMBER_NO_DIRECT=1 sends every gradient row through the segmented reduction.
bool getenv_direct() {
    const char* v = getenv("EMBER_NO_DIRECT");
    return !(v && v[0] == '1');
}

}  // namespace

void nccl_check(int r, const char* what) {
    if (r != ncclSuccess)
        throw EmberError(std::string(what) + " failed: " + (nccl().err ? nccl().err((ncclResult_t)r) : "?"));
}

void* nccl_comm_create(const void* unique_id, int rank, int world) {
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    ncclComm_t comm = nullptr;
    nccl_check(nccl().init_rank(&comm, world, id, rank), "ncclCommInitRank");
    return comm;
}

void nccl_unique_id(void* out) {
    ncclUniqueId id;
    nccl_check(nccl().unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
}

void nccl_comm_destroy(void* comm) {
    if (comm) nccl().destroy(static_cast<ncclComm_t>(comm));
}

void nccl_group(bool start) { nccl_check(start ? nccl().group_start() : nccl().group_end(), "ncclGroupStart/End"); }

void nccl_send_f32(const float* buf, size_t n, int peer, void* comm, cudaStream_t st) {
    nccl_check(nccl().send(buf, n, ncclFloat32, peer, static_cast<ncclComm_t>(comm), st), "ncclSend");
}

void nccl_recv_f32(float* buf, size_t n, int peer, void* comm, cudaStream_t st) {
    nccl_check(nccl().recv(buf, n, ncclFloat32, peer, static_cast<ncclComm_t>(comm), st), "ncclRecv");
}

bool pdl_enabled() {
    static const bool on = [] {
        const char* v = getenv("EMBER_PDL");
        return !(v && v[0] == '0');
    }();
    return on;
}

Engine::Engine(int dev, const ember_model_desc& md, const ember_graph_desc& gd, cudaStream_t st)
    : device(dev), m(md), g(gd) {
    if (m.kind < EMBER_DOT || m.kind > EMBER_COMPLEX) throw ConfigError("model kind must be 0 (Dot), 1 (DistMult), 2 (ComplEx)");
    if (m.dim == 0 || m.dim % 4 != 0) throw ConfigError("dim must be a positive multiple of 4");
    if (m.dim > 1792) throw ConfigError("dim must be <= 1792 (long-segment reduction stages 32 rows in shared memory)");
    if (m.batch_size == 0) throw ConfigError("batch_size must be >= 1");
    if (!(m.alpha >= 0.f && m.alpha <= 1.f)) throw ConfigError("alpha must be in [0, 1]");
    if (!(m.eps > 0.f)) throw ConfigError("eps must be > 0 (SPEC.md:170)");
    if (g.num_partitions == 0 || g.num_nodes < g.num_partitions) throw ConfigError("need 1 <= p <= |V|");
    if (g.num_nodes > 0xffffffffULL) throw ConfigError("node ids are u32");
    if (m.kind != EMBER_DOT && g.num_relations == 0) throw ConfigError("DistMult/ComplEx need relations");
    if (m.engine != EMBER_ENGINE_TC_BF16X3 && m.engine != EMBER_ENGINE_SIMT_FP32) throw ConfigError("unknown engine");
    if (m.engine == EMBER_ENGINE_SIMT_FP32 && !getenv_flag("EMBER_TEST_ENGINES"))
        throw ConfigError("the SIMT fp32 engine is the tests' reference engine (set EMBER_TEST_ENGINES=1)");
    dim = m.dim;
    nt = m.num_negatives;
    chunks = m.num_chunks ? m.num_chunks : 1;
    if (chunks > m.batch_size) throw ConfigError("num_chunks must be <= batch_size");
    cap_b = m.batch_size;
    n_neg = chunks * 2 * nt;
    cap_rows = 3 * cap_b + n_neg;

    EMBER_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop;
    EMBER_CUDA(cudaGetDeviceProperties(&prop, device));
    sm_count = prop.multiProcessorCount;
    if (st) {
        stream = st;
    } else {
        // The step stream gets the highest priority: when the helper stream's sort blocks and the
        // step's kernels compete for SMs, the block scheduler dispatches the step's blocks first.
        int least = 0, greatest = 0;
        EMBER_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        const char* pr = getenv("EMBER_STREAM_PRIORITY");
        EMBER_CUDA(cudaStreamCreateWithPriority(&stream, cudaStreamNonBlocking, pr && atoi(pr) == 0 ? least : greatest));
        own_stream = true;
    }
    if (getenv("EMBER_SERIAL_SORT")) {  // A/B switch: sort on the step stream (no overlap)
        side = stream;
    } else if (const char* sp = getenv("EMBER_SIDE_PRIORITY")) {  // A/B: 1 = the greatest priority
        int least = 0, greatest = 0;
        EMBER_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        EMBER_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, atoi(sp) ? greatest : least));
    } else {
        EMBER_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    }
    EMBER_CUDA(cudaStreamCreateWithFlags(&io, cudaStreamNonBlocking));
    EMBER_CUDA(cudaStreamCreateWithFlags(&io_out, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
        EMBER_CUDA(cudaEventCreateWithFlags(&ev_staged[k], cudaEventDisableTiming));
        EMBER_CUDA(cudaEventCreateWithFlags(&ev_consumed[k], cudaEventDisableTiming));
        EMBER_CUDA(cudaEventCreateWithFlags(&ev_loss_read[k], cudaEventDisableTiming));
    }
    EMBER_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
    EMBER_CUDA(cudaEventCreateWithFlags(&ev_sorted, cudaEventDisableTiming));
    EMBER_CUDA(cudaStreamCreateWithFlags(&comm, cudaStreamNonBlocking));
    EMBER_CUDA(cudaEventCreateWithFlags(&ev_rel_grad, cudaEventDisableTiming));
    EMBER_CUDA(cudaEventCreateWithFlags(&ev_rel_done, cudaEventDisableTiming));
    if (const char* e = getenv("EMBER_DENSE_RELATIONS")) force_dense = atoi(e) != 0;
    sample_on_step = getenv("EMBER_SAMPLE_ON_STEP") && atoi(getenv("EMBER_SAMPLE_ON_STEP")) != 0;
    seg_walk = getenv("EMBER_SEG_WALK") && atoi(getenv("EMBER_SEG_WALK")) != 0;
    parts.assign(g.num_partitions, PartView{nullptr, nullptr, 0, 0});
    for (uint32_t k = 0; k < g.num_partitions; ++k) {
        parts[k].first = partition_offset(g.num_nodes, g.num_partitions, k);
        parts[k].rows = partition_size(g.num_nodes, g.num_partitions, k);
    }
    if (tc_engine() && !tc_engine_supported(*this))
        throw ConfigError("tensor-core engine needs a CC 10.0 device (B200) and num_chunks == 1");
    const bool wide_path = tc_engine() && (dim > 128 || chunks > 1);

    const uint64_t b = cap_b, d = dim;
    s.negs = dalloc<uint32_t>(n_neg);
    s.batch = dalloc<uint32_t>(2 * 3 * (uint64_t)b);
    s.A = dalloc<float>(2 * b * d);
    s.N = dalloc<float>((uint64_t)n_neg * d);
    s.fpos = dalloc<float>(b);
    s.lse = dalloc<float>(2 * b);
    s.g0 = dalloc<float>(2 * b);
    s.dA = dalloc<float>(2 * (uint64_t)std::max<uint64_t>(b, (uint64_t)pad_rows(cap_b)) * d);
    s.grows = dalloc<float>((uint64_t)cap_rows * d);
    s.loss = dalloc<float>(4);  // [0]: steps; [1 + k]: host-batch steps of staging slot k
    // one per k_loss block, or one per warp of the fused chain rule (<= 3 x 8 warps per SM)
    s.loss_part = reinterpret_cast<float*>(dalloc<double>(std::max<uint64_t>(b / 512 + 2, 24ull * sm_count + 32)));
    s.loss_done = dalloc<uint32_t>(1);
    EMBER_CUDA(cudaMemset(s.loss_done, 0, sizeof(uint32_t)));
    s.bad_batch = dalloc<unsigned long long>(1);
    EMBER_CUDA(cudaMemset(s.bad_batch, 0, sizeof(unsigned long long)));
    s.keys = dalloc<uint32_t>(cap_rows);
    s.keys_sorted = dalloc<uint32_t>(cap_rows);
    s.vals_sorted = dalloc<uint32_t>(cap_rows);
    s.rank = dalloc<uint32_t>(cap_rows);
    s.uniq = dalloc<uint8_t>(cap_rows);
    s.ukeys = dalloc<uint32_t>(cap_rows);
    s.offsets = dalloc<uint32_t>(cap_rows + 1);  // offsets[nruns] = n closes the last run
    // (runs past nruns are never read by the step; zeroed once so whole-buffer copies are defined)
    EMBER_CUDA(cudaMemset(s.ukeys, 0, (size_t)cap_rows * sizeof(uint32_t)));
    EMBER_CUDA(cudaMemset(s.offsets, 0, (size_t)(cap_rows + 1) * sizeof(uint32_t)));
    for (int k = 0; k < 2; ++k) {
        s.sort_keys[k] = dalloc<uint32_t>(cap_rows);
        s.sort_vals[k] = dalloc<uint32_t>(cap_rows);
    }
    s.sort_hist = dalloc<uint32_t>(slot_sort_scratch_words(cap_rows));
    s.sort_status = dalloc<unsigned long long>(slot_sort_tiles(cap_rows));
    s.sort_ctr = dalloc<uint32_t>(1);
    s.nsplit = dalloc<uint32_t>(1);
    s.nruns = dalloc<uint32_t>(1);
    s.nunique = dalloc<uint32_t>(2);
    // at most cap_rows / LONG_SEG long segments, each with <= len / LONG_CHUNK + 1 chunks
    const uint32_t max_long = cap_rows / EMBER_LONG_SEG + 1;
    const uint32_t max_chunks = cap_rows / EMBER_LONG_CHUNK + max_long;
    s.longs = dalloc<uint32_t>(3 + 3 * max_long);
    s.seg_act = dalloc<uint32_t>(cap_rows);
    s.long_owner = dalloc<uint32_t>(max_chunks);
    s.long_partial = dalloc<float>((uint64_t)max_chunks * d);

    EMBER_CUDA(cudaMemset(s.nunique, 0, 2 * sizeof(uint32_t)));
    EMBER_CUDA(cudaMemset(s.longs, 0, 3 * sizeof(uint32_t)));
    if (m.engine == EMBER_ENGINE_SIMT_FP32) {
        s.S = dalloc<float>(2 * b * (uint64_t)(nt ? nt : 1));
        s.dN_part = dalloc<float>((uint64_t)dsplit * n_neg * d);
    }
    if (tc_engine() && !wide_path) {  // packed operand geometry: dim padded to 16, rows to 128- and 96-row tiles
        KP = (int)((dim + 15) / 16 * 16);
        CB = KP / 8;
        b_cap = pad_rows(cap_b);
        n_pad = pad_rows(nt);
        s.Apk = dalloc<uint16_t>((size_t)2 * 2 * CB * b_cap * 8);
        s.Npk = dalloc<uint16_t>((size_t)2 * 2 * CB * n_pad * 8);
    }
    if (tc_engine()) {
        if (wide_path) wide_setup(*this);
        else tc_setup(*this);
    }
    EMBER_CUDA(cudaStreamSynchronize(stream));
}

Engine::~Engine() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    if (side && side != stream) cudaStreamSynchronize(side);
    tc_release(*this);
    wide_release(*this);
    void* ptrs[] = {s.batch, s.A,         s.N,      s.Apk,       s.Npk,     s.fpos,       s.lse,    s.g0,
                    s.S,     s.dA,        s.dN_part, s.grows,    s.loss,    s.loss_part,  s.loss_done,  s.bad_batch,
                    s.nunique, s.long_partial, s.rel_dense, s.negs, s.keys, s.keys_sorted, s.vals_sorted,
                    s.rank, s.ukeys, s.offsets, s.nruns, s.longs, s.long_owner, s.uniq, s.sort_keys[0],
                    s.sort_keys[1], s.sort_vals[0], s.sort_vals[1], s.sort_hist, s.sort_status, s.sort_ctr, s.nsplit,
                    s.seg_act};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    for (void* p : owned) cudaFree(p);
    cudaGetLastError();
    if (nccl_comm) {
        try {
            nccl().destroy(static_cast<ncclComm_t>(nccl_comm));
        } catch (...) {
        }
    }
    if (io) cudaStreamSynchronize(io);
    if (io_out) cudaStreamSynchronize(io_out);
    for (int k = 0; k < 2; ++k) {
        if (ev_staged[k]) cudaEventDestroy(ev_staged[k]);
        if (ev_consumed[k]) cudaEventDestroy(ev_consumed[k]);
        if (ev_loss_read[k]) cudaEventDestroy(ev_loss_read[k]);
    }
    if (io) cudaStreamDestroy(io);
    if (io_out) cudaStreamDestroy(io_out);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_sorted) cudaEventDestroy(ev_sorted);
    if (ev_rel_grad) cudaEventDestroy(ev_rel_grad);
    if (ev_rel_done) cudaEventDestroy(ev_rel_done);
    if (comm) {
        cudaStreamSynchronize(comm);
        cudaStreamDestroy(comm);
    }
    if (side && side != stream) cudaStreamDestroy(side);
    if (own_stream) cudaStreamDestroy(stream);
}

PartView Engine::view(uint32_t part) const {
    if (part >= parts.size()) throw ConfigError("partition id out of range");
    const PartView& v = parts[part];
    if (!v.theta || !v.acc) throw ConfigError("partition " + std::to_string(part) + " has no bound tables");
    return v;
}

void Engine::check_bucket(uint32_t i, uint32_t j) const {
    view(i);
    view(j);
    if (m.kind != EMBER_DOT && (!rel_theta || !rel_acc)) throw ConfigError("relation table not bound");
}

KeySpace Engine::keyspace(uint32_t i, uint32_t j) const {
    KeySpace ks;
    ks.lo = view(std::min(i, j));
    ks.hi = view(std::max(i, j));
    ks.node_range = ks.lo.rows + (i != j ? ks.hi.rows : 0);
    const uint64_t n_keys = ks.node_range + (m.kind != EMBER_DOT ? g.num_relations : 0);
    ks.bits = bits_for(n_keys);
    return ks;
}

void Engine::sample(const uint32_t* bucket, uint64_t bucket_n, uint32_t i, uint32_t j, uint64_t epoch,
                    uint32_t bucket_step, uint32_t batch_in_bucket, uint32_t* negs_out) {
    const uint64_t base = mix_seed(mix_seed(m.neg_seed, epoch, bucket_step), batch_in_bucket);
    launch_sample(*this, negs_out, base, bucket, bucket_n, view(i), view(j));
}

void Engine::sort_keys(const uint32_t* edges, uint32_t nb, uint32_t i, uint32_t j, const uint32_t* negs) {
    const KeySpace ks = keyspace(i, j);
    launch_keys(*this, edges, nb, negs, ks);
    sort_slots(nb, ks);
}

void Engine::sort_slots(uint32_t nb, const KeySpace& ks, uint32_t direct) {
    const uint32_t n = slots(nb);
    launch_slot_sort(*this, slots(nb), ks.bits, (uint32_t)ks.node_range);
    launch_long_plan(*this, slots(nb), ks.node_range, direct);
    EMBER_CUDA(cudaEventRecord(ev_sorted, side));
    sorted_pending = true;
}

void Engine::join_sorted() {
    if (!sorted_pending) return;
    EMBER_CUDA(cudaStreamWaitEvent(stream, ev_sorted, 0));
    sorted_pending = false;
}

void Engine::forward_backward(const uint32_t* edges, uint32_t nb, uint32_t i, uint32_t j, const uint32_t* negs,
                              bool presorted) {
    const PartView pi = view(i), pj = view(j);
    dn_pending = false;  // (set by this step's contraction, consumed by its chain rule)
    if (!presorted) {  // helper stream, overlapped with the gathers and the contraction
        EMBER_CUDA(cudaEventRecord(ev_fork, stream));
        EMBER_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
        sort_keys(edges, nb, i, j, negs);
    }
    mark(PHASE_GATHER);
    const bool fused = tc_engine() && !wide;  // d <= 128: the gather packs the bf16 operands itself
    if (!wide) launch_gather_adjust(*this, edges, nb, pi, pj, fused, negs);  // (wide: in launch_contract_wide)
    launch_gather_negatives(*this, negs, pi, pj, fused);
    mark(PHASE_CONTRACT);
    if (wide)
        launch_contract_wide(*this, nb, edges, pi, pj);  // joins the sort before scattering dN rows
    else if (tc_engine())
        launch_contract_tc(*this, nb);  // joins the sort before scattering dN rows
    else
        launch_contract_simt(*this, nb);
    mark(PHASE_CHAIN);
    join_sorted();
    launch_chain_rule(*this, edges, nb, pi, pj);
}

void Engine::reduce_and_apply(uint32_t nb, uint32_t i, uint32_t j, bool apply, uint32_t* node_ids_out,
                              float* node_rows_out, uint32_t* rel_ids_out, float* rel_rows_out) {
    const KeySpace ks = keyspace(i, j);
    // Relations: in place (1 GPU), or summed into a dense [R][dim] buffer that is all-reduced
    // (internal NCCL comm) or handed to the caller (rel_ext: external reduction, then
    // ember_relations_apply_dense) before the relation Adagrad.
    const bool ext = rel_ext != nullptr;
    const bool dense = apply && m.kind != EMBER_DOT && (world > 1 || ext || force_dense);
    float* buf = ext ? rel_ext : s.rel_dense;
    if (dense && !ext) {
        // The relation keys are reduced, summed across ranks and applied (dense Adagrad) on `comm`
        // while the node keys (most of the reduction) are reduced on the step stream; the step
        // stream joins before anything reads relations again.
        if (!s.rel_dense) s.rel_dense = dalloc<float>((uint64_t)g.num_relations * dim);
        EMBER_CUDA(cudaEventRecord(ev_rel_grad, stream));
        EMBER_CUDA(cudaStreamWaitEvent(comm, ev_rel_grad, 0));
        EMBER_CUDA(cudaMemsetAsync(s.rel_dense, 0, (size_t)g.num_relations * dim * sizeof(float), comm));
        launch_segments(*this, slots(nb), ks, apply, true, nullptr, nullptr, nullptr, nullptr, 1, comm);
        allreduce_relations(comm);
        apply_relations_dense(s.rel_dense, comm);
        EMBER_CUDA(cudaEventRecord(ev_rel_done, comm));
        launch_segments(*this, slots(nb), ks, apply, true, node_ids_out, node_rows_out, rel_ids_out, rel_rows_out, 2);
        EMBER_CUDA(cudaStreamWaitEvent(stream, ev_rel_done, 0));
        return;
    }
    if (dense) EMBER_CUDA(cudaMemsetAsync(buf, 0, (size_t)g.num_relations * dim * sizeof(float), stream));
    launch_segments(*this, slots(nb), ks, apply, dense, node_ids_out, node_rows_out, rel_ids_out, rel_rows_out);
}

void Engine::idle_step() {
    // a lockstep step without a batch (multi-GPU): this rank's relation gradient is zero, but the
    // all-reduce is a collective and the dense Adagrad applies the other ranks' sum
    if (m.kind == EMBER_DOT || world <= 1) return;
    EMBER_CUDA(cudaMemsetAsync(s.rel_dense, 0, (size_t)g.num_relations * dim * sizeof(float), stream));
    allreduce_relations(stream);
    apply_relations_dense(s.rel_dense);
}

void Engine::apply_relations_dense(const float* grad, cudaStream_t st) {
    if (m.kind == EMBER_DOT) return;
    if (!rel_theta || !rel_acc) throw ConfigError("relation table not bound");
    const uint64_t rn = (uint64_t)g.num_relations * dim;
    launch_pdl(k_adagrad_dense, dim3((unsigned)((rn + 255) / 256)), dim3(256), 0, st ? st : stream, rel_theta, rel_acc,
               grad, rn, m.lr, m.eps);
    EMBER_LAUNCHED(*this);
}

void Engine::mark(int phase) {
    if (!prof_on) return;
    cudaEvent_t ev;
    EMBER_CUDA(cudaEventCreate(&ev));
    EMBER_CUDA(cudaEventRecord(ev, stream));
    prof_events.emplace_back(phase, ev);
}

void Engine::train_batch_host(const uint32_t* bucket, uint64_t bucket_n, const uint32_t* host_batch, uint32_t nb,
                              uint32_t i, uint32_t j, uint64_t epoch, uint32_t bucket_step, uint32_t batch_in_bucket,
                              float* loss_host) {
    if (nb == 0 || nb > cap_b) throw ConfigError("batch size must be in [1, batch_size]");
    const int k = (int)(host_steps++ & 1);
    uint32_t* slot = s.batch + (uint64_t)k * 3 * cap_b;
    // the copy waits only for the step two calls back (the last reader of this slot), so it
    // overlaps the previous step; the step waits for its copy
    if (host_steps > 2) EMBER_CUDA(cudaStreamWaitEvent(io, ev_consumed[k], 0));
    EMBER_CUDA(cudaMemcpyAsync(slot, host_batch, (size_t)nb * 12, cudaMemcpyHostToDevice, io));
    EMBER_CUDA(cudaEventRecord(ev_staged[k], io));
    EMBER_CUDA(cudaStreamWaitEvent(stream, ev_staged[k], 0));
    // the loss lands in slot k's own word and is read back on io_out, off the step stream (whose
    // kernels then chain with programmatic launches); the word is rewritten two steps later, after
    // that read (ev_loss_read)
    float* loss_dev = s.loss + 1 + k;
    if (host_steps > 2) EMBER_CUDA(cudaStreamWaitEvent(stream, ev_loss_read[k], 0));
    step(slot, nb, bucket, bucket_n, i, j, epoch, bucket_step, batch_in_bucket, loss_dev, ev_staged[k]);
    EMBER_CUDA(cudaEventRecord(ev_consumed[k], stream));
    EMBER_CUDA(cudaStreamWaitEvent(io_out, ev_consumed[k], 0));
    if (loss_host) EMBER_CUDA(cudaMemcpyAsync(loss_host, loss_dev, sizeof(float), cudaMemcpyDeviceToHost, io_out));
    EMBER_CUDA(cudaEventRecord(ev_loss_read[k], io_out));
}

void Engine::train_batch(const uint32_t* bucket, uint64_t bucket_n, uint64_t batch_begin, uint32_t nb, uint32_t i,
                         uint32_t j, uint64_t epoch, uint32_t bucket_step, uint32_t batch_in_bucket, float* loss_out) {
    if (batch_begin + nb > bucket_n) throw ConfigError("batch exceeds bucket");
    step(bucket + 3 * batch_begin, nb, bucket, bucket_n, i, j, epoch, bucket_step, batch_in_bucket, loss_out);
}

void Engine::check_finite() {
    unsigned long long tag = 0;
    EMBER_CUDA(cudaStreamSynchronize(stream));
    EMBER_CUDA(cudaMemcpy(&tag, s.bad_batch, sizeof(tag), cudaMemcpyDeviceToHost));
    if (!tag) return;
    EMBER_CUDA(cudaMemset(s.bad_batch, 0, sizeof(tag)));
    throw EmberError("non-finite loss in batch (epoch " + std::to_string((tag >> 40) & 0xFFFFF) + ", bucket step " +
                     std::to_string((tag >> 20) & 0xFFFFF) + ", batch " + std::to_string(tag & 0xFFFFF) + ")");
}

void Engine::step(const uint32_t* edges, uint32_t nb, const uint32_t* bucket, uint64_t bucket_n, uint32_t i,
                  uint32_t j, uint64_t epoch, uint32_t bucket_step, uint32_t batch_in_bucket, float* loss_out,
                  cudaEvent_t edges_ready) {
    if (nb == 0 || nb > cap_b) throw ConfigError("batch size must be in [1, batch_size]");
    check_bucket(i, j);
    NvtxRange nvtx("ember::step");
    // Sampling and the gradient-slot keys: one kernel on the step stream (ordered after the caller's
    // work that produced the batch and the bucket). Only the (key, slot) sort forks onto the helper
    // stream, where it overlaps the gathers and the contraction; the step stream joins it before the
    // first gradient scatter. edges_ready: the batch is staged by another stream (host batches).
    if (edges_ready) EMBER_CUDA(cudaStreamWaitEvent(stream, edges_ready, 0));
    const KeySpace ks = keyspace(i, j);
    mark(PHASE_SAMPLE);
    const uint64_t base = mix_seed(mix_seed(m.neg_seed, epoch, bucket_step), batch_in_bucket);
    direct_hi = getenv_direct() ? 2 * nb : 0;
    // EMBER_HOST_INLINE=1 (A/B): also for host-staged batches, where it measured slower (0.3229 vs
    // 0.3031 ms per step of the host-buffer path: the staging waits then sit right before the gather)
    static const int host_inline = getenv("EMBER_HOST_INLINE") ? atoi(getenv("EMBER_HOST_INLINE")) : 0;
    if (tc_engine() && !wide && !sample_on_step && (!edges_ready || host_inline)) {
        // The packed gather draws the shared negatives itself (same counter-based stream), so the
        // sampling + keys kernel runs on the helper stream beside it, forked here: after the caller's
        // work on the step stream and the previous step's updates.
        EMBER_CUDA(cudaEventRecord(ev_fork, stream));
        EMBER_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
        launch_sample_keys(*this, edges, nb, base, bucket, bucket_n, view(i), view(j), ks, side);
        neg_inline.on = 1;
        neg_inline.base = base;
        neg_inline.bucket = bucket;
        neg_inline.bucket_n = bucket_n;
    } else {
        launch_sample_keys(*this, edges, nb, base, bucket, bucket_n, view(i), view(j), ks);
        EMBER_CUDA(cudaEventRecord(ev_fork, stream));
        EMBER_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
    }
    sort_slots(nb, ks, direct_hi);
    loss_target = loss_out ? loss_out : s.loss;
    batch_tag = (1ull << 63) | ((epoch & 0xFFFFFull) << 40) | ((uint64_t)(bucket_step & 0xFFFFFu) << 20) |
                (batch_in_bucket & 0xFFFFFu);
    forward_backward(edges, nb, i, j, s.negs, true);
    neg_inline.on = 0;
    launch_loss(*this, nb, loss_out ? loss_out : s.loss);
    mark(PHASE_REDUCE);
    reduce_and_apply(nb, i, j, true, nullptr, nullptr, nullptr, nullptr);
    direct_hi = 0;
    mark(PHASE_END);
}

std::vector<double> Engine::profile_read() {
    std::vector<double> ms(PHASE_END + 1, 0.0);
    EMBER_CUDA(cudaStreamSynchronize(stream));
    for (size_t k = 0; k + 1 < prof_events.size(); ++k) {
        if (prof_events[k].first == PHASE_END) continue;
        float t = 0.f;
        EMBER_CUDA(cudaEventElapsedTime(&t, prof_events[k].second, prof_events[k + 1].second));
        ms[prof_events[k].first] += t;
    }
    for (auto& pe : prof_events) cudaEventDestroy(pe.second);
    prof_events.clear();
    return ms;
}

void Engine::comm_init(const void* unique_id, int r, int w) {
    if (w < 1 || r < 0 || r >= w) throw ConfigError("bad rank/world");
    rank = r;
    world = w;
    if (w == 1) return;
    ncclUniqueId id;
    std::memcpy(&id, unique_id, sizeof(id));
    ncclComm_t comm = nullptr;
    EMBER_CUDA(cudaSetDevice(device));
    ncclResult_t res = nccl().init_rank(&comm, w, id, r);
    if (res != ncclSuccess) throw EmberError(std::string("ncclCommInitRank failed: ") + (nccl().err ? nccl().err(res) : "?"));
    nccl_comm = comm;
    if (m.kind != EMBER_DOT && !s.rel_dense) s.rel_dense = dalloc<float>((uint64_t)g.num_relations * dim);
}

void Engine::allreduce_relations(cudaStream_t st) {
    if (!nccl_comm) return;
    const uint64_t rn = (uint64_t)g.num_relations * dim;
    ncclResult_t r = nccl().all_reduce(s.rel_dense, s.rel_dense, rn, ncclFloat32, ncclSum, static_cast<ncclComm_t>(nccl_comm), st);
    if (r != ncclSuccess) throw EmberError(std::string("ncclAllReduce failed: ") + (nccl().err ? nccl().err(r) : "?"));
}

}  // namespace ember
