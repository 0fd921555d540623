// SPDX-License-Identifier: Apache-2.0
//
// Engine: one GPU's training context behind the C-ABI (include/ember_gpu.h).
// Owns the step's device scratch, sized once for the configured batch; borrows the
// partition tables. All work is ordered on one CUDA stream (the single compute worker of
// SPEC.md:372); internally the key sort forks onto a helper stream and joins back.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "ember/common.h"
#include "ember_gpu.h"

namespace ember {

// Segmented reduction: keys with more than EMBER_LONG_SEG gradient rows take the chunked path
// (EMBER_LONG_CHUNK-row chunk partials, kernels_step.cu).
#define EMBER_LONG_SEG 16
#define EMBER_LONG_CHUNK 32

#define EMBER_CUDA(call)                                                                        \
    do {                                                                                        \
        cudaError_t e_ = (call);                                                                \
        if (e_ != cudaSuccess)                                                                  \
            throw ::ember::EmberError(std::string("CUDA error ") + cudaGetErrorString(e_) + " at " + \
                                      __FILE__ + ":" + std::to_string(__LINE__) + ": " #call);  \
    } while (0)

// After each of our kernel launches: surface launch errors, count the launch.
#define EMBER_LAUNCHED(E)                      \
    do {                                       \
        EMBER_CUDA(cudaGetLastError());        \
        ++(E).launches;                        \
    } while (0)

// HBM row layout. Dot/DistMult rows are stored in coordinate order. A ComplEx row, [re | im]
// halves of h = d/2 on disk, is stored with its halves interleaved by pairs:
// on-disk coordinate re k sits at 4(k/2) + k%2 and im k at 4(k/2) + 2 + k%2, so the 16 bytes at
// float offset 4q hold the complex coordinates {re 2q, re 2q+1, im 2q, im 2q+1} (one aligned
// 128-bit access per lane, d % 4 == 0). Every product of the step is a dot product over a row's
// coordinates, so kernels work on HBM order throughout; only init, the ParameterSlice /
// GradientDelta entry points and the storage boundary map coordinates (ember_rows_layout).
__host__ __device__ inline uint32_t hbm_pos(int kind, uint32_t d, uint32_t c) {
    if (kind != EMBER_COMPLEX) return c;
    const uint32_t h = d / 2, im = c >= h ? 1u : 0u, k = c - im * h;
    return 4 * (k >> 1) + 2 * im + (k & 1);
}

// A node id -> row pointer view of one partition: row(id) = base + (id - first) * dim.
struct PartView {
    float* theta;
    float* acc;
    uint64_t first;
    uint64_t rows;
};

// Gradient-row keys of one batch of bucket (i, j). Node ids live in partitions lo = min(i, j)
// and hi = max(i, j); key = id - first_lo for the lo partition, rows_lo + (id - first_hi) for
// the hi one (so ascending keys = ascending global ids), relation r -> node_range + r. With
// p = 16 this is a 24-bit key: three 8-bit radix passes.
struct KeySpace {
    PartView lo, hi;
    uint64_t node_range;
    uint32_t bits;
};

// Gradient-row production index ("slot") of one batch: [0, nb) source rows, [nb, 2nb)
// destination rows, [2nb, 2nb + n_neg) negative rows, [2nb + n_neg, 3nb + n_neg) relation rows.
// rank[slot] = the slot's position after sorting by (key, slot); producers write each gradient
// row straight to grows[rank[slot]], so every key's rows are contiguous and in slot order.
//
// Scratch layouts (row-major, dim-wide rows unless noted):
//   negs   [chunks][2][nt]             sampled negative ids (side 0 = dst corruption)
//   A      [2][b][dim]                 adjusted vectors, fp32 (SIMT engine / debug scores)
//   N      [chunks*2*nt][dim]          negative rows, fp32 (SIMT engine / debug scores)
//   Apk    [2][2CB][b_cap][8] bf16     adjusted vectors split hi|lo (tensor-core engine)
//   Npk    [2][2CB][n_pad][8] bf16     negative rows split hi|lo (tensor-core engine)
//   fpos   [b]; lse, g0 [2][b]; dA [2][b][dim]
//   grows  [3b + n_neg][dim]           gradient rows in sorted (key, slot) order
struct Scratch {
    uint32_t* negs = nullptr;
    uint32_t* batch = nullptr;  // staging for host batches: 2 x [b][3] (double-buffered)
    float* A = nullptr;
    float* N = nullptr;
    uint16_t* Apk = nullptr;
    uint16_t* Npk = nullptr;
    float* fpos = nullptr;
    float* lse = nullptr;
    float* g0 = nullptr;
    float* S = nullptr;       // SIMT engine: [2][b][nt] scores -> P/b
    float* dA = nullptr;
    float* dN_part = nullptr; // SIMT engine split-K partials
    float* grows = nullptr;
    float* loss = nullptr;       // [1]
    float* loss_part = nullptr;  // per-block partial sums of the loss reduction
    uint32_t* loss_done = nullptr;
    unsigned long long* bad_batch = nullptr;  // first batch whose loss was non-finite (sticky, 0 = none)
    uint32_t* keys = nullptr;
    uint32_t* keys_sorted = nullptr;
    uint32_t* vals_sorted = nullptr;
    uint32_t* rank = nullptr;
    uint8_t* uniq = nullptr;      // slot -> its key occurs once among the batch's slots
    uint32_t* ukeys = nullptr;
    uint32_t* offsets = nullptr;  // [runs + 1]: offsets[nruns] = n
    uint32_t* nruns = nullptr;    // [1] unique keys (RLE)
    uint32_t* nunique = nullptr;  // [2] unique node keys, unique relation keys
    uint32_t* longs = nullptr;        // [2 + 3 * cap]: long segments, chunk slots, then (u, base, nch)
    uint32_t* long_owner = nullptr;   // chunk slot -> long segment
    uint32_t* seg_act = nullptr;      // runs with segment-kernel work (k_long_plan; count in longs[2])
    float* long_partial = nullptr;    // chunk slot -> partial row

    // slot sort (sort.cu): ping-pong key/value buffers, per-tile digit histograms, run-scan state
    uint32_t* sort_keys[2] = {nullptr, nullptr};
    uint32_t* sort_vals[2] = {nullptr, nullptr};
    uint32_t* sort_hist = nullptr;
    unsigned long long* sort_status = nullptr;
    uint32_t* sort_ctr = nullptr;
    uint32_t* nsplit = nullptr;  // [1] first run of a relation key (~0u: none), written by the sort
    float* rel_dense = nullptr;  // [R][dim] relation gradient summed over ranks (world > 1)
};

// The fixed-order sum of the dN partials over chunks, row (side, n) -> gradient slot slot0 + side nt + n
// at its sorted position: k_dn_reduce, or the prologue of the pipelined chain rule (pending in
// Engine::dn until then). nsides: 2, or 2 x num_chunks (tc_wide.cu).
struct DnReduce {
    const float4* part = nullptr;  // column-blocked [chunk][nsides][d/4][n_pad]
    int chunks = 0, nt = 0, n_pad = 0, d = 0, nsides = 0;
    uint32_t slot0 = 0;
    uint32_t* flags = nullptr;  // the overflow list consumed by the fixup: counted and reset here
    unsigned long long* flags_total = nullptr;
};

// One (side, column block, negative) item of a DnReduce; t < nsides * (d/4) * nt.
__device__ __forceinline__ void dn_reduce_item(const DnReduce& r, int64_t t, const uint32_t* __restrict__ rank,
                                               float* __restrict__ out) {
    const int d4 = r.d / 4;
    const int n = (int)(t % r.nt);
    const int c4 = (int)((t / r.nt) % d4);
    const int side = (int)(t / ((int64_t)r.nt * d4));
    const float4* p = r.part + ((size_t)side * d4 + c4) * r.n_pad + n;
    const size_t cstride = (size_t)r.nsides * d4 * r.n_pad;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int c = 0;
    for (; c + 4 <= r.chunks; c += 4) {  // 4 loads in flight, added in chunk order
        float4 x[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) x[i] = __ldg(p + (size_t)(c + i) * cstride);
#pragma unroll
        for (int i = 0; i < 4; ++i) acc.x += x[i].x, acc.y += x[i].y, acc.z += x[i].z, acc.w += x[i].w;
    }
    for (; c < r.chunks; ++c) {
        const float4 x = __ldg(p + (size_t)c * cstride);
        acc.x += x.x, acc.y += x.y, acc.z += x.z, acc.w += x.w;
    }
    const uint32_t pos = rank[r.slot0 + side * r.nt + n];
    reinterpret_cast<float4*>(out + (size_t)pos * r.d)[c4] = acc;
}

struct TcState;    // tensor-core engine state (tc_score.cu, d <= 128)
struct WideState;  // tensor-core engine state for d > 128 (tc_wide.cu)

struct Engine {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;  // key sort runs here, overlapped with gather + contraction
    cudaEvent_t ev_fork = nullptr, ev_sorted = nullptr;
    // relation gradients summed across ranks (world > 1): the relation keys are reduced first, their
    // all-reduce + dense Adagrad run on `comm` while the node keys are reduced on the step stream
    cudaStream_t comm = nullptr;
    cudaEvent_t ev_rel_grad = nullptr, ev_rel_done = nullptr;
    bool force_dense = false;  // EMBER_DENSE_RELATIONS=1: that path at world 1 (tests: bit-identical)
    // A/B switches read per context (tests: bit-identical either way): EMBER_SAMPLE_ON_STEP=1 samples
    // on the step stream before the gather; EMBER_SEG_WALK=1 the segment kernel visits every run
    bool sample_on_step = false, seg_walk = false;
    // host-batch path: positives copied on `io` into one of two staging slots, overlapping the
    // previous step; ev_staged[k]: copy into slot k done; ev_consumed[k]: the step reading slot k done
    cudaStream_t io = nullptr, io_out = nullptr;  // host->device batches / device->host losses
    cudaEvent_t ev_staged[2] = {nullptr, nullptr}, ev_consumed[2] = {nullptr, nullptr};
    cudaEvent_t ev_loss_read[2] = {nullptr, nullptr};  // the loss of the step using slot k has been read back
    uint64_t host_steps = 0;
    bool own_stream = false;
    bool sorted_pending = false;
    ember_model_desc m{};
    ember_graph_desc g{};
    uint32_t dim = 0;
    uint32_t nt = 0;
    uint32_t chunks = 1;
    uint32_t cap_b = 0;
    uint32_t n_neg = 0;     // chunks * 2 * nt
    uint32_t cap_rows = 0;  // 3 * cap_b + n_neg gradient slots
    uint32_t dsplit = 16;   // split-K factor for dN in the SIMT engine
    std::vector<PartView> parts;
    std::vector<void*> owned;  // device memory allocated through the context (ember_device_alloc, tables)
    float* rel_theta = nullptr;
    float* rel_acc = nullptr;
    Scratch s;
    TcState* tc = nullptr;
    WideState* wide = nullptr;  // d > 128: the three-pass tcgen05 GEMM path (tc_wide.cu)
    // packed-operand geometry (tensor-core engine)
    int KP = 0, CB = 0, b_cap = 0, n_pad = 0;
    int sm_count = 148;
    // multi-GPU
    void* nccl_comm = nullptr;
    int rank = 0, world = 1;
    float* rel_ext = nullptr;  // caller-owned [R][dim] relation-gradient buffer (external reduction)
    // Training steps apply Adagrad to source/destination rows whose key occurs once in the batch
    // right in the chain rule (slots < direct_hi = 2nb); 0: every row goes through the segmented
    // reduction.
    uint32_t direct_hi = 0;
    mutable uint32_t plan_direct = 0;
    // this step's negatives drawn by the packed gather itself (sampling + keys on the helper stream)
    struct {
        int on = 0;
        uint64_t base = 0, bucket_n = 0;
        const uint32_t* bucket = nullptr;
    } neg_inline;  // direct threshold the last k_long_plan's run list was built for
    // where the step's loss goes; the tensor-core chain rule reduces it there itself (loss_fused)
    float* loss_target = nullptr;
    // batch id of the step being enqueued ("non-finite score -> error carrying batch id")
    unsigned long long batch_tag = 0;
    void check_finite();  // throws EmberError (status 2) naming the first non-finite batch since the last check
    mutable bool loss_fused = false;
    // the contraction's dN reduction, left to the chain rule's prologue (launch_chain_rule)
    mutable DnReduce dn{};
    mutable bool dn_pending = false;
    // profiling: CUDA events at phase boundaries on the step stream + our own kernel launches
    bool prof_on = false;
    std::vector<std::pair<int, cudaEvent_t>> prof_events;
    mutable uint64_t launches = 0;
    mutable uint64_t lib_calls = 0;  // library kernel calls on the step (none since the hand-written slot sort)
    void mark(int phase);

    Engine(int device, const ember_model_desc& m, const ember_graph_desc& g, cudaStream_t stream);
    ~Engine();

    PartView view(uint32_t part) const;
    void check_bucket(uint32_t i, uint32_t j) const;
    KeySpace keyspace(uint32_t i, uint32_t j) const;
    bool tc_engine() const { return m.engine == EMBER_ENGINE_TC_BF16X3; }
    uint32_t slots(uint32_t nb) const { return 2 * nb + n_neg + (m.kind != EMBER_DOT ? nb : 0); }
    // Rows of a packed operand holding n rows: whole 128-row resident tiles and whole 96-row
    // streamed tiles of the tensor-core engine (zero / -inf padded).
    static int pad_rows(uint32_t n) {
        const uint32_t a = (n + 127) / 128 * 128, b = (n + 95) / 96 * 96;
        return (int)((std::max(a, b) + 31) / 32 * 32);
    }

    // pipeline stages
    void sample(const uint32_t* bucket, uint64_t bucket_n, uint32_t i, uint32_t j, uint64_t epoch,
                uint32_t bucket_step, uint32_t batch_in_bucket, uint32_t* negs_out);
    // Keys of the batch's gradient slots, sorted on the helper stream (forked by the caller).
    void sort_keys(const uint32_t* edges, uint32_t nb, uint32_t i, uint32_t j, const uint32_t* negs);
    // direct: the chain rule applies node keys occurring once with slot < direct (k_long_plan leaves
    // them out of the segment kernel's run list)
    void sort_slots(uint32_t nb, const KeySpace& ks, uint32_t direct = 0);  // (key, slot) sort of s.keys on the helper stream
    void join_sorted();  // the step stream waits for sort_keys' results
    // Computes loss and gradient rows for one batch into grows (sorted order).
    void forward_backward(const uint32_t* edges, uint32_t nb, uint32_t i, uint32_t j, const uint32_t* negs,
                          bool presorted = false);
    // Segmented sum of the sorted gradient rows, then Adagrad (or export of the deltas).
    void reduce_and_apply(uint32_t nb, uint32_t i, uint32_t j, bool apply, uint32_t* node_ids_out,
                          float* node_rows_out, uint32_t* rel_ids_out, float* rel_rows_out);
    void train_batch(const uint32_t* bucket, uint64_t bucket_n, uint64_t batch_begin, uint32_t nb, uint32_t i,
                     uint32_t j, uint64_t epoch, uint32_t bucket_step, uint32_t batch_in_bucket, float* loss_out);
    // The same step with the positives in host memory (double-buffered asynchronous copy).
    void train_batch_host(const uint32_t* bucket, uint64_t bucket_n, const uint32_t* host_batch, uint32_t nb,
                          uint32_t i, uint32_t j, uint64_t epoch, uint32_t bucket_step, uint32_t batch_in_bucket,
                          float* loss_host);
    // One Algorithm-1 step on nb positives at `edges` (device) of bucket (i, j).
    // edges_ready (nullable): an event the helper stream must wait for before reading `edges`.
    void step(const uint32_t* edges, uint32_t nb, const uint32_t* bucket, uint64_t bucket_n, uint32_t i, uint32_t j,
              uint64_t epoch, uint32_t bucket_step, uint32_t batch_in_bucket, float* loss_out,
              cudaEvent_t edges_ready = nullptr);
    void allreduce_relations(cudaStream_t st);
    void idle_step();  // lockstep step without a batch (world > 1): zero relation gradient, all-reduce, Adagrad
    void apply_relations_dense(const float* grad, cudaStream_t st = nullptr);  // dense relation Adagrad (zero rows are no-ops)
    void comm_init(const void* nccl_unique_id, int rank, int world);
    std::vector<double> profile_read();  // ms per phase summed over marked batches
};

void dn_reduce_run(const Engine& E, const DnReduce& r);  // k_dn_reduce on the step stream (tc_score.cu)

enum Phase { PHASE_SAMPLE = 0, PHASE_GATHER = 1, PHASE_CONTRACT = 2, PHASE_CHAIN = 3, PHASE_REDUCE = 4, PHASE_END = 5 };

// NVTX range for the scope (host-side enqueue of a step / bucket / epoch; visible in Nsight timelines,
// near-free without a tool attached).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// Programmatic dependent launch (PDL) on the step stream: a kernel's CTAs may be scheduled while
// the previous kernel drains; every kernel launched this way starts (after its own set-up) with
// griddep_wait(), which returns once the previous grid has completed and its writes are visible.
// EMBER_PDL=0 launches them as ordinary stream-ordered kernels (A/B).
__device__ __forceinline__ void griddep_wait() {
#if defined(__CUDA_ARCH__)
    asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
}
// The dependent grid (launched with PDL) may be scheduled once every CTA of this grid has executed
// this (or exited); its griddep_wait() still waits for this grid's completion.
__device__ __forceinline__ void griddep_launch() {
#if defined(__CUDA_ARCH__)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
bool pdl_enabled();
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    EMBER_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// kernel launchers (kernels_step.cu, gemm_simt.cu, tc_score.cu, graph.cu)
void launch_sample(const Engine& E, uint32_t* out, uint64_t base_seed, const uint32_t* bucket, uint64_t bucket_n,
                   const PartView& src, const PartView& dst);
void launch_sample_on(const Engine& E, cudaStream_t st, uint32_t* out, uint64_t base_seed, const uint32_t* bucket,
                      uint64_t bucket_n, const PartView& src, const PartView& dst);
// packed: write the tensor-core engine's bf16 hi|lo operands (Apk/Npk), else fp32 A / N.
void launch_gather_adjust(const Engine& E, const uint32_t* edges, uint32_t nb, const PartView& pi, const PartView& pj,
                          bool packed, const uint32_t* negs);
void launch_gather_negatives(const Engine& E, const uint32_t* negs, const PartView& pi, const PartView& pj, bool packed);
// the wide tensor-core path's packed gather (tc_wide.cu layout: cap rows, chunk q at q CP, cr rows per chunk)
void launch_gather_pack_wide(const Engine& E, const uint32_t* edges, uint32_t nb, const PartView& pi, const PartView& pj,
                             uint16_t* Apk, uint32_t CBA, uint32_t cap, uint32_t CP, uint32_t cr);
void launch_keys(const Engine& E, const uint32_t* edges, uint32_t nb, const uint32_t* negs, const KeySpace& ks);
// the training step's sample_negatives + gradient-slot keys, one kernel on the step stream
void launch_sample_keys(const Engine& E, const uint32_t* edges, uint32_t nb, uint64_t base, const uint32_t* bucket,
                        uint64_t bucket_n, const PartView& src, const PartView& dst, const KeySpace& ks, cudaStream_t st = nullptr);
// the (key, slot) sort of s.keys and its runs, on the helper stream (sort.cu)
void launch_slot_sort(const Engine& E, uint32_t n, uint32_t bits, uint32_t split_key);
size_t slot_sort_scratch_words(uint32_t cap);
uint32_t slot_sort_tiles(uint32_t cap);
void launch_contract_simt(Engine& E, uint32_t nb);
void launch_contract_tc(Engine& E, uint32_t nb);
void launch_chain_rule(const Engine& E, const uint32_t* edges, uint32_t nb, const PartView& pi, const PartView& pj);
void launch_loss(const Engine& E, uint32_t nb, float* loss_out);
// the long-segment chunk plan (keys with > EMBER_LONG_SEG rows) on the helper stream after the sort
void launch_long_plan(const Engine& E, uint32_t n_slots, uint64_t node_range, uint32_t direct);
// part: 0 every key, 1 relation keys only, 2 node keys only (the split: s.nsplit)
void launch_segments(const Engine& E, uint32_t n_slots, const KeySpace& ks, bool apply, bool rel_dense,
                     uint32_t* node_ids_out, float* node_rows_out, uint32_t* rel_ids_out, float* rel_rows_out,
                     int part = 0, cudaStream_t st = nullptr);
void launch_adagrad_rows(const Engine& E, const uint32_t* ids, const float* rows, uint32_t n, const PartView& pi,
                         const PartView& pj, bool relations,
                         uint32_t* bad);
void launch_gather_rows(const Engine& E, const uint32_t* ids, uint32_t n, const PartView& pi, const PartView& pj,
                        bool relations, float* th_out, float* ac_out, uint32_t* bad);
void launch_init_rows(cudaStream_t st, float* theta, float* acc, uint64_t first_row, uint64_t rows, uint32_t dim,
                      int kind, uint64_t seed);
// rows between on-disk coordinate order and the HBM layout, in place (no-op unless ComplEx);
// n_dev (nullable): row count read on the device, n its upper bound
void launch_rows_layout(cudaStream_t st, float* rows, uint64_t n, const uint32_t* n_dev, uint32_t dim, int kind,
                        bool to_hbm);
void launch_debug_scores(const Engine& E, const uint32_t* edges, uint32_t nb, const uint32_t* negs, int side,
                         uint32_t rows, float* out, const PartView& pi, const PartView& pj);
void launch_eval_ranks(const Engine& E, const uint32_t* test, uint32_t n_test, const uint32_t* negs, uint32_t n_eval,
                       uint32_t block, uint32_t* ranks);
// NCCL (loaded at run time, engine.cu): communicators and point-to-point copies for the multi-GPU
// driver (dist.cu); errors throw EmberError
void* nccl_comm_create(const void* unique_id, int rank, int world);
void nccl_unique_id(void* out128);
void nccl_comm_destroy(void* comm);
void nccl_group(bool start);
void nccl_send_f32(const float* buf, size_t n, int peer, void* comm, cudaStream_t st);
void nccl_recv_f32(float* buf, size_t n, int peer, void* comm, cudaStream_t st);
bool tc_engine_supported(const Engine& E);
void tc_setup(Engine& E);
void tc_release(Engine& E);
uint64_t tc_overflow_rows(Engine& E);
bool wide_supported(const Engine& E);
void wide_setup(Engine& E);
void wide_release(Engine& E);
uint64_t wide_overflow_rows(Engine& E);
void launch_contract_wide(Engine& E, uint32_t nb, const uint32_t* edges, const PartView& pi, const PartView& pj);

}  // namespace ember
