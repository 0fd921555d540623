// SPDX-License-Identifier: Apache-2.0
//
// Engine: one GPU's training context behind the C-ABI (include/ember_gpu.h).
// Owns the step's device scratch, sized once for the configured batch; borrows the
// partition tables. All work goes to one CUDA stream (the single compute worker of
// SPEC.md:372).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "ember/common.h"
#include "ember_gpu.h"

namespace ember {

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

// A node id -> row pointer view of one partition: row(id) = base + (id - first) * dim.
struct PartView {
    float* theta;
    float* acc;
    uint64_t first;
    uint64_t rows;
};

// Scratch for one step. Layouts (row-major, dim-wide rows unless noted):
//   negs   [chunks][2][nt]             sampled negative ids (side 0 = dst corruption)
//   A      [2][b][dim]                 adjusted vectors (side 0: adj_dst, side 1: adj_src)
//   fpos   [b]                         positive scores
//   lse,g0 [2][b]                      log-sum-exp per row, dL/dfpos per side
//   N      [chunks*2*nt][dim]          gathered negative rows
//   S      [2][b][nt]                  scores, overwritten by P/b (SIMT engine only)
//   dA     [2][b][dim]
//   grows  [2b + chunks*2*nt][dim]     node gradient rows: src rows, dst rows, negative rows (= dN)
//   rrows  [b][dim]                    relation gradient rows
struct Scratch {
    uint32_t* negs = nullptr;
    uint32_t* batch = nullptr;  // staging for host batches [b][3]
    float* A = nullptr;
    float* fpos = nullptr;
    float* lse = nullptr;
    float* g0 = nullptr;
    float* N = nullptr;
    float* S = nullptr;
    float* dA = nullptr;
    float* dN_part = nullptr;
    float* grows = nullptr;
    float* rrows = nullptr;
    float* row_loss = nullptr;
    float* loss = nullptr;      // [1]
    uint32_t* keys = nullptr;
    uint32_t* keys_sorted = nullptr;
    uint32_t* vals = nullptr;
    uint32_t* vals_sorted = nullptr;
    uint32_t* ukeys = nullptr;
    uint32_t* counts = nullptr;
    uint32_t* offsets = nullptr;
    uint32_t* nunique = nullptr;  // [2]: nodes, relations
    void* cub_tmp = nullptr;
    size_t cub_bytes = 0;
    // bf16 hi/lo operand tiles for the tensor-core engine
    uint16_t* Atc = nullptr;
    uint16_t* Ntc = nullptr;
    uint16_t* NTtc = nullptr;
    float* dN_tc = nullptr;
    float* rel_dense = nullptr;  // [R][dim] relation gradient summed over ranks (world > 1)
    uint32_t* cc = nullptr;      // chunks per unique id (segmented reduction)
    uint32_t* coff = nullptr;    // exclusive scan of cc
    float* partial = nullptr;    // [2b + negs][dim] per-chunk partial sums
};

struct TcState;  // tensor-core engine state (tc_score.cu)

struct Engine {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    ember_model_desc m{};
    ember_graph_desc g{};
    uint32_t dim = 0;
    uint32_t nt = 0;
    uint32_t chunks = 1;
    uint32_t cap_b = 0;
    uint32_t n_neg = 0;     // chunks * 2 * nt
    uint32_t dsplit = 16;   // split-K factor for dN in the SIMT engine
    uint32_t key_bits = 32;
    std::vector<PartView> parts;
    float* rel_theta = nullptr;
    float* rel_acc = nullptr;
    Scratch s;
    TcState* tc = nullptr;
    int sm_count = 148;
    // multi-GPU
    void* nccl_comm = nullptr;
    int rank = 0, world = 1;
    // profiling: CUDA events at phase boundaries on the step stream + our own kernel launches
    bool prof_on = false;
    std::vector<std::pair<int, cudaEvent_t>> prof_events;
    mutable uint64_t launches = 0;
    mutable uint64_t lib_calls = 0;  // CUB device-wide calls (library kernels, counted separately)
    void mark(int phase);

    Engine(int device, const ember_model_desc& m, const ember_graph_desc& g, cudaStream_t stream);
    ~Engine();

    PartView view(uint32_t part) const;
    void check_bucket(uint32_t i, uint32_t j) const;

    // pipeline stages
    void sample(const uint32_t* bucket, uint64_t bucket_n, uint32_t i, uint32_t j, uint64_t epoch,
                uint32_t bucket_step, uint32_t batch_in_bucket, uint32_t* negs_out);
    // Computes loss and node/relation gradient rows for one batch into scratch (grows, rrows).
    void forward_backward(const uint32_t* edges, uint32_t nb, uint32_t i, uint32_t j, const uint32_t* negs);
    // Dedupe + segmented sum of the gradient rows, then Adagrad (or export the deltas).
    void reduce_and_apply(const uint32_t* edges, uint32_t nb, uint32_t i, uint32_t j, const uint32_t* negs,
                          bool apply, uint32_t* node_ids_out, float* node_rows_out, uint32_t* rel_ids_out,
                          float* rel_rows_out);
    void train_batch(const uint32_t* bucket, uint64_t bucket_n, uint64_t batch_begin, uint32_t nb, uint32_t i,
                     uint32_t j, uint64_t epoch, uint32_t bucket_step, uint32_t batch_in_bucket, float* loss_out);
    // One Algorithm-1 step on nb positives at `edges` (device) of bucket (i, j).
    void step(const uint32_t* edges, uint32_t nb, const uint32_t* bucket, uint64_t bucket_n, uint32_t i, uint32_t j,
              uint64_t epoch, uint32_t bucket_step, uint32_t batch_in_bucket, float* loss_out);
    void allreduce_relations(uint32_t nb);
    void comm_init(const void* nccl_unique_id, int rank, int world);
    std::vector<double> profile_read();  // ms per phase summed over marked batches
};

enum Phase { PHASE_SAMPLE = 0, PHASE_GATHER = 1, PHASE_CONTRACT = 2, PHASE_CHAIN = 3, PHASE_REDUCE = 4, PHASE_END = 5 };

// kernel launchers (kernels_step.cu, gemm_simt.cu, tc_score.cu, graph.cu)
void launch_sample(const Engine& E, uint32_t* out, uint64_t base_seed, const uint32_t* bucket, uint64_t bucket_n,
                   const PartView& src, const PartView& dst);
void launch_gather_adjust(const Engine& E, const uint32_t* edges, uint32_t nb, const PartView& pi, const PartView& pj);
void launch_gather_negatives(const Engine& E, const uint32_t* negs, const PartView& pi, const PartView& pj);
void launch_contract_simt(Engine& E, uint32_t nb);
void launch_contract_tc(Engine& E, uint32_t nb);
void launch_chain_rule(const Engine& E, const uint32_t* edges, uint32_t nb, const PartView& pi, const PartView& pj);
void launch_loss(const Engine& E, uint32_t nb, float* loss_out);
void launch_adagrad_segments(const Engine& E, const uint32_t* ukeys, const uint32_t* offsets, const uint32_t* counts,
                             const uint32_t* nunique, const uint32_t* vals_sorted, const float* rows, uint32_t max_u,
                             const PartView& pi, const PartView& pj, bool relations, uint32_t* ids_out,
                             float* rows_out, bool apply);
void launch_adagrad_rows(const Engine& E, const uint32_t* ids, const float* rows, uint32_t n, const PartView& pi,
                         const PartView& pj, bool relations);
void launch_init_rows(cudaStream_t st, float* theta, float* acc, uint64_t first_row, uint64_t rows, uint32_t dim,
                      uint64_t seed);
void launch_debug_scores(const Engine& E, const uint32_t* edges, uint32_t nb, const uint32_t* negs, int side,
                         uint32_t rows, float* out, const PartView& pi, const PartView& pj);
void launch_eval_ranks(const Engine& E, const uint32_t* test, uint32_t n_test, const uint32_t* negs, uint32_t n_eval,
                       uint32_t block, uint32_t* ranks);
bool tc_engine_supported(const Engine& E);
void tc_setup(Engine& E);
void tc_release(Engine& E);

}  // namespace ember
