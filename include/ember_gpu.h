/* SPDX-License-Identifier: Apache-2.0
 *
 * ember_gpu.h — the C-ABI drop-in boundary of the B200-native minibatch training step.
 *
 * The reference (proj/, namespace ember) declares its trainer only as SPEC operations;
 * proj/src/model.cpp and pipeline.cpp are listed in proj/src/CMakeLists.txt:5,8 but absent.
 * Each entry point below names the SPEC/paper operation it replaces. Plain C types only:
 * device pointers are `T*` into memory on the context's device, host pointers are marked.
 * Every call returns EMBER_OK (0), EMBER_EUSER (1: bad config/arguments, the reference's
 * ConfigError) or EMBER_EINTERNAL (2: CUDA/IO failure, non-finite score);
 * a non-finite batch loss is recorded on the device without a host sync and
 * reported by the next synchronising call (ember_ctx_synchronize, ember_train_bucket/epoch with
 * stats, ember_loss_and_grad) as status 2 with "non-finite loss in batch (epoch e, bucket step
 * s, batch k)";
 * ember_last_error() returns the thread-local message (SPEC.md:552 exit codes).
 * No exceptions cross this boundary. One context per GPU, not thread-safe, all work is
 * enqueued on the context's stream ("the model computation stage only uses a
 * single worker").
 */
#ifndef EMBER_GPU_H
#define EMBER_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EMBER_OK 0
#define EMBER_EUSER 1
#define EMBER_EINTERNAL 2

/* ModelKind */
#define EMBER_DOT 0
#define EMBER_DISTMULT 1
#define EMBER_COMPLEX 2

/* Contraction engine for the shared-negative scores.
 * TC_BF16X3: tcgen05 tensor cores, operands split hi+lo in bf16 (3 products, fp32 accumulate),
 *            ~2^-16 relative per product — inside the 1e-4 parity tolerance. Any d (d <= 128 with
 *            one negative set per batch: the fused kernels of tc_score.cu; d > 128 or chunked
 *            negatives: the three-pass kernels of tc_wide.cu). The product engine.
 * SIMT_FP32: CUDA-core fp32 tiles, the tests' reference engine: rejected unless the environment
 *            sets EMBER_TEST_ENGINES=1. */
#define EMBER_ENGINE_SIMT_FP32 0
#define EMBER_ENGINE_TC_BF16X3 1

/* OrderingKind (reference ordering.h:14) */
#define EMBER_ORDER_ELIMINATION 0
#define EMBER_ORDER_HILBERT 1
#define EMBER_ORDER_HILBERT_SYMMETRIC 2
#define EMBER_ORDER_RANDOM 3

typedef struct ember_ctx ember_ctx;

/* Hyper-parameters of the step: SPEC RunConfig subset + NegativeSampleSpec
 * (SPEC.md:129-132). num_chunks: the batch is cut into num_chunks contiguous chunks, each scored
 * against its own n_t shared negatives per corruption side (1 = whole batch shares). */
typedef struct {
    int32_t kind;
    uint32_t dim;
    float lr;
    float eps;
    uint32_t batch_size;    /* b: max edges per step */
    uint32_t num_negatives; /* n_t per chunk per side */
    float alpha;            /* degree-based fraction */
    uint32_t num_chunks;
    uint64_t neg_seed;
    int32_t engine;         /* EMBER_ENGINE_* */
    uint32_t reserved;
} ember_model_desc;

/* GraphMeta subset. Partition k owns global rows
 * [k*floor(V/p) + min(k, V%p), +floor(V/p) + (k < V%p)). */
typedef struct {
    uint64_t num_nodes;
    uint32_t num_relations;
    uint32_t num_partitions;
} ember_graph_desc;

typedef struct {
    double loss_sum;        /* sum of per-batch mean losses */
    uint64_t batches;
    uint64_t edges;
    uint64_t unique_nodes;  /* node rows updated (sum over batches), filled when stats requested */
    uint64_t unique_rels;
} ember_step_stats;

/* ---- lifecycle -------------------------------------------------------------------------- */
/* stream: a cudaStream_t to enqueue on (NULL -> the context creates its own). */
int ember_ctx_create(int device, const ember_model_desc* model, const ember_graph_desc* graph, void* stream,
                     ember_ctx** out);
int ember_ctx_destroy(ember_ctx* ctx);
void* ember_ctx_stream(ember_ctx* ctx);
/* Waits for all work of the context (its stream and its internal copy / helper streams). */
int ember_ctx_synchronize(ember_ctx* ctx);
const char* ember_last_error(void);
int ember_version(void);

/* ---- device memory through the context (for C/C++ callers without a CUDA runtime of their own)
 * ember_device_alloc: `bytes` of device memory on the context's device, owned by the context (freed
 * by ember_device_free or ember_ctx_destroy). The copies are ordered on the context stream and
 * return when done (host memory may be pageable). Pinned host memory (for the partition buffer's
 * backing store and asynchronous host batches): ember_host_alloc_pinned / ember_host_free_pinned. */
int ember_device_alloc(ember_ctx* ctx, size_t bytes, void** out);
int ember_device_free(ember_ctx* ctx, void* dev_ptr);
int ember_copy_to_device(ember_ctx* ctx, void* dst_dev, const void* src_host, size_t bytes);
int ember_copy_to_host(ember_ctx* ctx, void* dst_host, const void* src_dev, size_t bytes);
int ember_host_alloc_pinned(size_t bytes, void** out);
int ember_host_free_pinned(void* host_ptr);

/* ---- parameter storage (PartitionBlock; ParameterSlice SPEC.md:125) ------------
 * Caller-owned device memory, borrowed: theta and acc are [rows x dim] f32 row-major for the
 * partition's rows in the HBM row layout. For Dot/DistMult that is the on-disk node_part_<k>.bin
 * layout. A ComplEx row ([re | im] halves of h = dim/2 on disk) holds
 * its halves interleaved by pairs: re k at 4(k/2) + k%2, im k at 4(k/2) + 2 + k%2, so each
 * aligned 16 bytes are {re 2q, re 2q+1, im 2q, im 2q+1}. ember_rows_layout converts rows in place
 * (to_hbm = 1: on-disk -> HBM; 0: back) on the context stream, ember_rows_layout_host on the host;
 * both are no-ops unless the model is ComplEx. The per-op entry points that take or return rows
 * (ember_gather, ember_adagrad_apply, ember_loss_and_grad) use the on-disk coordinate order. */
int ember_rows_layout(ember_ctx* ctx, float* rows_dev, uint64_t rows, int to_hbm);
int ember_rows_layout_host(int kind, uint32_t dim, float* rows, uint64_t n, int to_hbm);
int ember_tables_bind(ember_ctx* ctx, uint32_t part, float* theta_dev, float* acc_dev);
int ember_relations_bind(ember_ctx* ctx, float* theta_dev, float* acc_dev);
/* Context-owned tables: allocates theta and acc of partition `part` (EMBER_RELATIONS: the relation
 * table) on the device and binds them; ember_tables_get returns the bound pointers and row count. */
#define EMBER_RELATIONS 0xffffffffu
int ember_tables_allocate(ember_ctx* ctx, uint32_t part);
int ember_tables_get(ember_ctx* ctx, uint32_t part, float** theta_dev, float** acc_dev, uint64_t* rows);
/* init_embeddings for one bound partition / the relation table:
 * global row g <- Rng(mix_seed(seed, g)).uniform(-1/sqrt(d), 1/sqrt(d)) x d; acc <- 0.
 * Relations use seed ^ 0x52454c (row = relation id). */
int ember_init_partition(ember_ctx* ctx, uint32_t part, uint64_t seed);
int ember_init_relations(ember_ctx* ctx, uint64_t seed);

/* ---- the training step (Algorithm 1; Stage 1+3+5 of Fig. 4) --------------
 * One batch = edges [batch_begin, batch_begin+nb) of bucket (i, j) whose edges live at
 * bucket_edges_dev (bucket_n EdgeTriples, device). Negatives are drawn from the bucket
 * (degree part) and partitions j (dst side) / i (src side). Relations and nodes are updated
 * in place with Adagrad before the call's work completes on the stream.
 * loss_dev (nullable): device float receiving this batch's mean loss. */
int ember_train_batch(ember_ctx* ctx, const uint32_t* bucket_edges_dev, uint64_t bucket_n, uint64_t batch_begin,
                      uint32_t nb, uint32_t i, uint32_t j, uint64_t epoch, uint32_t bucket_step,
                      uint32_t batch_in_bucket, float* loss_dev);
/* trainEdgeBucket (Algorithm 2): all batches of one bucket, in order.
 * stats (host, nullable) is filled after a stream sync when non-NULL. */
int ember_train_bucket(ember_ctx* ctx, const uint32_t* bucket_edges_dev, uint64_t bucket_n, uint32_t i, uint32_t j,
                       uint64_t epoch, uint32_t bucket_step, ember_step_stats* stats);
/* train_epoch_partitioned with every partition bound (HBM-resident): all buckets
 * of seq (2*p*p u32: the plan's bucket sequence) in order, each bucket's batches in order,
 * bucket_step = position in seq. edges_dev: bucketed edges, offsets_host: p*p+1 u64. stats
 * (nullable) is filled after one synchronisation at the end of the epoch. */
int ember_train_epoch(ember_ctx* ctx, const uint32_t* edges_dev, const uint64_t* offsets_host, const uint32_t* seq,
                      uint64_t epoch, ember_step_stats* stats);
/* Same step with the nb positives in HOST memory (pinned recommended), copied in asynchronously on
 * an internal copy stream (double-buffered: the copy overlaps the previous step). The degree-based
 * sampler still reads the bucket (bucket_edges_dev), which stays device-resident. loss_host
 * (nullable; pinned for an asynchronous copy) receives the loss asynchronously: it is valid after
 * ember_ctx_synchronize. The caller keeps host_batch alive until then as well. */
int ember_train_batch_host(ember_ctx* ctx, const uint32_t* bucket_edges_dev, uint64_t bucket_n,
                           const uint32_t* host_batch, uint32_t nb, uint32_t i, uint32_t j, uint64_t epoch,
                           uint32_t bucket_step, uint32_t batch_in_bucket, float* loss_host);

/* ---- per-op entry points (SPEC model ops), for parity tests ------------------------------ */
/* sample_negatives: negs_dev receives num_chunks*2*n_t ids [chunk][side][slot]. */
int ember_sample_negatives(ember_ctx* ctx, const uint32_t* bucket_edges_dev, uint64_t bucket_n, uint32_t i, uint32_t j,
                           uint64_t epoch, uint32_t bucket_step, uint32_t batch_in_bucket, uint32_t* negs_dev);
/* loss_and_grad: no parameter update. Outputs (device, nullable): fpos[nb],
 * lse[2*nb]; node GradientDelta: unique ids ascending + summed rows (capacity 2nb + negs);
 * relation GradientDelta likewise (capacity nb). Counts and loss are written to host. */
int ember_loss_and_grad(ember_ctx* ctx, const uint32_t* edges_dev, uint32_t nb, uint32_t i, uint32_t j,
                        const uint32_t* negs_dev, float* fpos_dev, float* lse_dev, uint32_t* node_ids_dev,
                        float* node_rows_dev, uint32_t* n_node_host, uint32_t* rel_ids_dev, float* rel_rows_dev,
                        uint32_t* n_rel_host, double* loss_host);
/* ParameterSlice gather (getGpuParameters): exactly one row per id,
 * in id order. Node ids (global) must lie in partition i or j; relations != 0: relation ids.
 * theta_out_dev: n x dim f32; acc_out_dev (nullable) likewise. Synchronises the stream (status 1
 * and nothing written for the offending rows when an id is out of range). */
int ember_gather(ember_ctx* ctx, const uint32_t* ids_dev, uint32_t n, uint32_t i, uint32_t j, int relations,
                 float* theta_out_dev, float* acc_out_dev);
/* adagrad_step on n rows of bucket (i, j)'s node tables (relations != 0: the
 * relation table). ids/rows device. Synchronises the stream; ids outside partitions i and j (or
 * outside [0, R)) are not written and make the call return status 1. */
int ember_adagrad_apply(ember_ctx* ctx, const uint32_t* ids_dev, const float* rows_dev, uint32_t n, uint32_t i,
                        uint32_t j, int relations);
/* Scores S[r][k] = f(edge r, negative k) for the first `rows` edges of a batch against chunk 0's
 * side-`side` negatives (debug/parity; out_dev: rows x n_t). */
int ember_debug_scores(ember_ctx* ctx, const uint32_t* edges_dev, uint32_t nb, uint32_t i, uint32_t j,
                       const uint32_t* negs_dev, int side, uint32_t rows, float* out_dev);
/* The step's (key, slot) sort on n <= 3 batch_size + n_neg keys of `bits` bits (debug/parity):
 * keys_sorted / vals_sorted (n), rank (n: slot -> sorted position), uniq (n bytes: the slot's key
 * occurs once), ukeys (n), offsets (n + 1: run u = [offsets[u], offsets[u + 1])), nruns (1); all
 * device buffers, written on the context stream. */
int ember_debug_sort_slots(ember_ctx* ctx, const uint32_t* keys_dev, uint32_t n, uint32_t bits, uint32_t* keys_sorted_dev,
                           uint32_t* vals_sorted_dev, uint32_t* rank_dev, uint8_t* uniq_dev, uint32_t* ukeys_dev,
                           uint32_t* offsets_dev, uint32_t* nruns_dev);

/* ---- link-prediction eval, unfiltered sampled negatives ------------------ */
int ember_eval_ranks(ember_ctx* ctx, const uint32_t* test_edges_dev, uint32_t n_test, const uint32_t* train_edges_dev,
                     uint64_t n_train, uint32_t n_eval_neg, float alpha_eval, uint32_t block, uint64_t eval_seed,
                     uint32_t* ranks_dev);

/* Filtered protocol (FB15k-type configs): all nodes are
 * candidates, candidates forming a known triple are skipped; filter_keys_dev: n_keys u64 sorted
 * ascending, key = s<<40 | r<<24 | t. ranks_dev: 2*n_test (dst corruption ranks, then src). */
int ember_eval_ranks_filtered(ember_ctx* ctx, const uint32_t* test_edges_dev, uint32_t n_test,
                              const uint64_t* filter_keys_dev, uint64_t n_keys, uint32_t* ranks_dev);

/* ---- ordering (reference ordering.h, bit-identical) -------------------------------------- */
int ember_make_plan(int kind, uint32_t p, uint32_t c, uint64_t seed, uint32_t* seq_out /* 2*p*p */,
                    uint64_t* swap_count, uint32_t* admissions_out /* c + 2*p*p */, uint32_t* n_admissions,
                    uint32_t* swaps_out /* 3 per swap, <= 2*p*p swaps */, uint32_t* bucket_state_out /* p*p */);
uint64_t ember_lower_bound_swaps(uint32_t p, uint32_t c);
uint64_t ember_elimination_swap_formula(uint32_t p, uint32_t c);

/* ---- synthetic graphs (test/bench data; SURVEY §8(d) generator) ---------------------------
 * Edge e of a graph with `seed`: power-law sources, Zipf relations, community-planted
 * destinations. Generated on the device (device != -1) or host (device == -1) into
 * edges_out (n x 3 u32, same memory space). split_out (nullable, n bytes): 0 train, 1 valid,
 * 2 test with the given fractions. */
int ember_graph_generate(int device, uint64_t num_nodes, uint32_t num_relations, uint64_t n_edges, uint64_t seed,
                         float train_frac, float valid_frac, uint32_t* edges_out, uint8_t* split_out);
/* bucket_edges: stable counting sort of n edges by (part(src), part(dst)).
 * offsets_out: p*p+1 u64. device == -1 -> host arrays. */
int ember_graph_bucket(int device, uint64_t num_nodes, uint32_t p, const uint32_t* edges_in, uint64_t n,
                       uint32_t* edges_out, uint64_t* offsets_out);

/* Graph-store preprocessing on the device (ingest + partition_nodes + bucket_edges).
 * raw_dev: n edges of (src, rel, dst) tokens (arbitrary u32 values, device). Node / relation
 * tokens are mapped to dense ids (rank among the sorted unique tokens); the nodes are then
 * relabeled by a seeded random permutation, so each partition (contiguous row range) is a random
 * node subset; the edges are shuffled (seeded) and split: first floor(train_frac*n) train, next
 * floor(valid_frac*n) valid, rest test. Train is bucketed (stable) into train_out_dev with
 * offsets_host (p*p+1); valid/test (nullable) keep the shuffled order. counts_host[3]: split sizes.
 * node_tokens_dev (nullable, capacity 2n): token of each relabeled node id; rel_tokens_dev
 * (nullable, capacity n): token of each relation id. Exactly restated by the CPU oracle. */
int ember_graph_preprocess(int device, const uint32_t* raw_dev, uint64_t n, uint32_t p, uint64_t seed,
                           float train_frac, float valid_frac, uint32_t* train_out_dev, uint64_t* offsets_host,
                           uint32_t* valid_out_dev, uint32_t* test_out_dev, uint64_t* counts_host,
                           uint32_t* node_tokens_dev, uint32_t* rel_tokens_dev, uint64_t* num_nodes_host,
                           uint32_t* num_relations_host);

/* ---- measurement ----------------------------------------------------------------------------
 * enable != 0: record CUDA events on the context stream at step phase boundaries.
 * ms_out[6]: summed ms per phase {sample, gather, contraction, chain+loss, reduce+adagrad, -}
 * since the last read; launches_out: our kernels launched since context creation; lib_calls_out:
 * CUB device-wide calls (library kernels) since creation. Synchronises the stream. */
int ember_profile_enable(ember_ctx* ctx, int enable);
int ember_profile_read(ember_ctx* ctx, double* ms_out, uint64_t* launches_out, uint64_t* lib_calls_out);
/* Rows (batch row x side) whose log-sum-exp left the tensor-core engine's safe range and were
 * recomputed exactly (fp32, CUDA cores), summed since context creation (0 for the SIMT engine).
 * Synchronises the context stream. */
int ember_overflow_rows(ember_ctx* ctx, uint64_t* total);
/* Self-test of the tcgen05 building blocks on `device` (one 128 x N x K bf16 product vs a double
 * host product); max_rel_err_out = max|err| / max|ref|. mode: see csrc/tc_selftest.cu. */
int ember_tc_selftest(int device, int mode, int K, int N, uint64_t seed, double* max_rel_err_out);
/* Microbenchmark: cycles per back-to-back tcgen05.mma (M=128, K=16, bf16, N columns) issued by one
 * thread. mode %16: 0 SS, 1 TS (A in TMEM), 2 TS with MN-major B, 3 SS with MN-major B; mode / 16 + 1
 * independent accumulators are cycled round-robin (N * count <= 256 columns). */
int ember_tc_mmabench(int device, int mode, int N, int iters, double* cycles_per_mma);

/* ---- device partition buffer (§4.2, Algorithm 2) ------------------
 * HBM holds `capacity` resident partition slots + 2 staging slots; pinned host memory is the
 * backing store (host_theta[k], host_acc[k]: partition k's [rows_k x dim] f32 arrays, pinned
 * for asynchronous copies). The buffer replays one epoch's bucket sequence (seq: 2*steps ids,
 * steps = p*p, from ember_make_plan) with Belady eviction (furthest next use, ties to the
 * lower id), prefetching each admission on a copy stream and writing evicted partitions back
 * asynchronously; misses per epoch == the plan's swap_count. While the buffer is attached it
 * binds the context's partition tables itself (ember_tables_bind must not be used). */
typedef struct ember_buffer ember_buffer;
typedef struct {
    uint64_t reads;          /* partition loads (initial fill + admissions) */
    uint64_t writes;         /* partition writebacks (evictions + epoch-end flush) */
    uint64_t bytes_read;
    uint64_t bytes_written;
    uint64_t swaps_per_epoch;
    uint64_t epochs;         /* completed epochs */
    uint32_t stalls;         /* admissions the compute stream had to wait for */
    uint32_t slots;          /* device slots allocated (capacity + 2 when capacity < p) */
    double stall_ms;         /* device time the compute stream waited on loads */
    uint64_t slot_bytes;
} ember_buffer_report;

int ember_buffer_create(ember_ctx* ctx, uint32_t capacity, const uint32_t* seq, uint32_t steps,
                        float* const* host_theta, float* const* host_acc, ember_buffer** out);
int ember_buffer_destroy(ember_buffer* buf);
/* acquire_pair: bucket seq[step] becomes resident for work enqueued after this call
 * on the context stream; steps are acquired in plan order, an epoch starts at step 0.
 * i_out/j_out (nullable) receive the bucket. */
int ember_buffer_acquire(ember_buffer* buf, uint32_t step, uint32_t* i_out, uint32_t* j_out);
/* The bucket's work has been enqueued: evictees whose last use this was start writing back.
 * Releasing the last step ends the epoch (all residents are written back). */
int ember_buffer_release(ember_buffer* buf, uint32_t step);
/* Between epochs: the context stream and the host wait until every writeback has landed in host memory. */
int ember_buffer_flush(ember_buffer* buf);
int ember_buffer_stats(ember_buffer* buf, ember_buffer_report* out);
/* The eviction decisions of one epoch: 3 u32 per swap (step, evicted, admitted); *n = swaps. */
int ember_buffer_decisions(ember_buffer* buf, uint32_t* out, uint32_t* n);
/* train_epoch_partitioned (Algorithm 2) through the buffer: every bucket of
 * the plan in order (acquire -> all batches of the bucket -> release). edges_dev: bucketed
 * edges (device), offsets_host: p*p+1 u64 bucket offsets (host). stats nullable. */
int ember_train_epoch_buffered(ember_ctx* ctx, ember_buffer* buf, const uint32_t* edges_dev,
                               const uint64_t* offsets_host, uint64_t epoch, ember_step_stats* stats);

/* ---- multi-GPU------------------------------------------------------------ */
/* Conflict-free round schedule (csrc/host/rounds.cpp): circle-method perfect
 * matchings of the p partitions, p/(2*world) pairs per GPU per round, buckets (a,b),(b,a) per
 * pair and the self-buckets in round 0. p even and world | p/2 (or p == world == 1).
 * order/round/rank: p*p u32 each — bucket id i*p+j in global schedule order, its round, its
 * GPU. holder: rounds*p u32 — GPU holding partition x in round r. *n_rounds = p-1 (1 if p==1).
 * The global position of a bucket is its bucket_step for the sampler seeds. */
int ember_make_rounds(uint32_t p, uint32_t world, uint32_t* order, uint32_t* round, uint32_t* rank, uint32_t* holder,
                      uint32_t* n_rounds);
/* Overlapped round schedule (csrc/host/rounds.cpp make_rounds_overlap): p a power of two >= 4 and
 * world | p/4. Rounds use the matchings {x, x ^ v_r} over GF(2)^k; every GPU holds whole cosets
 * x + span{v_{r-1}, v_r}, trains the pair that leaves it after the round first (early = 1) and the
 * pair that stays second, so the departing partitions' handoff overlaps the staying pair's
 * buckets. Same outputs as ember_make_rounds plus early: p*p u8. */
int ember_make_rounds_overlap(uint32_t p, uint32_t world, uint32_t* order, uint32_t* round, uint32_t* rank,
                              uint8_t* early, uint32_t* holder, uint32_t* n_rounds);
/* ---- multi-GPU driver (host/dist_driver.cpp, dist.cu): train_epoch_partitioned over `world` GPUs,
 * one process per GPU (Algorithm 2). Every rank runs the rounds of
 * the schedule (overlap = 0: ember_make_rounds; 1: ember_make_rounds_overlap) in lockstep: a step
 * is the rank's next batch (or an idle step when it has none left) followed, for models with
 * relations, by the NCCL all-reduce of the dense relation gradient and the relation Adagrad; after
 * a round the partitions that change holder move as one NCCL send/recv group on a copy stream and a
 * second communicator, issued at the same lockstep step on every rank: with overlap = 1 right after
 * the departing pair's buckets, so the copy runs under the staying pair's steps. The driver owns
 * the partition tables (slots of the largest partition: held + the most received per handoff).
 * nccl_id_steps / nccl_id_handoff: two ncclUniqueId (128 bytes each) shared by the ranks (ignored
 * at world 1). edges_dev: the bucketed edges; offsets_host: p*p+1 bucket offsets; batches of
 * model.batch_size. */
typedef struct ember_dist ember_dist;
typedef struct {
    uint64_t steps, batches, edges, handoffs, moved_partitions;
    uint64_t early_handoffs; /* handoffs issued before their round's last step (overlapped) */
    uint64_t handoff_bytes;  /* bytes this rank sent (ember_dist_train_epoch, cumulative) */
} ember_dist_report;
int ember_dist_create(ember_ctx* ctx, uint32_t rank, uint32_t world, int overlap, const void* nccl_id_steps,
                      const void* nccl_id_handoff, const uint32_t* edges_dev, const uint64_t* offsets_host,
                      ember_dist** out);
int ember_dist_destroy(ember_dist* d);
/* init_embeddings of the partitions this rank starts with + the relation replica. */
int ember_dist_init_embeddings(ember_dist* d, uint64_t seed);
/* Lockstep steps [first_step, first_step + n_steps) of the epoch (n_steps = UINT64_MAX: to the
 * end); no host synchronisation inside. */
int ember_dist_train_epoch(ember_dist* d, uint64_t epoch, uint64_t first_step, uint64_t n_steps,
                           ember_dist_report* out);
/* Where a partition this rank holds now lives (NULL when it is elsewhere). */
int ember_dist_tables(ember_dist* d, uint32_t part, float** theta_dev, float** acc_dev);
/* Waits for the step and copy streams; reports a non-finite batch loss (status 2). */
int ember_dist_synchronize(ember_dist* d);
/* The last step's mean batch loss, read back on the step stream (synchronous). */
int ember_dist_loss(ember_dist* d, float* loss_host);
/* A fresh ncclUniqueId (128 bytes) for ember_dist_create / ember_comm_init (rank 0 makes it, the
 * caller shares it). Loads NCCL at run time. */
int ember_nccl_unique_id(void* out128);
/* The lockstep plan: steps per round, the step after which each round's handoff is issued (0: none),
 * total steps (nullable outputs; arrays of p-1 entries, 1 if p == 1). */
int ember_dist_plan(uint32_t p, uint32_t world, uint32_t rank, int overlap, const uint64_t* offsets,
                    uint32_t batch_size, uint32_t* steps_per_round, uint32_t* handoff_step, uint64_t* total_steps);
/* The same round loop over caller-supplied rank operations (e.g. a CPU backend and a host
 * transport): step(batch or NULL for an idle step), send_recv(round, moves as (part, src, dst)
 * triples, n) at the handoff point, acquire(round, arrived parts, n) before a round's first step
 * (nullable). A nonzero return aborts with status 2. */
typedef struct {
    uint32_t bucket_step, i, j, batch_in_bucket;
    uint64_t lo, hi, begin; /* bucket edges [lo, hi); batch [lo + begin, lo + begin + nb) */
    uint32_t nb, pad;
} ember_batch_ref;
typedef struct {
    void* user;
    int (*step)(void* user, const ember_batch_ref* batch, uint64_t epoch);
    int (*send_recv)(void* user, uint32_t round, const uint32_t* moves, uint32_t n_moves);
    int (*acquire)(void* user, uint32_t round, const uint32_t* parts, uint32_t n);
} ember_rank_ops;
int ember_dist_run(uint32_t p, uint32_t world, uint32_t rank, int overlap, const uint64_t* offsets,
                   uint32_t batch_size, uint64_t epoch, uint64_t first_step, uint64_t n_steps,
                   const ember_rank_ops* ops, ember_dist_report* out);

/* External relation reduction: with grad_dev != NULL every training step zeroes grad_dev
 * ([R x dim] f32, device) and writes the batch's summed relation gradients into it instead of
 * updating the relation table; the caller reduces it across ranks (e.g. an NCCL all-reduce on the
 * context stream) and applies it with ember_relations_apply_dense (the relation Adagrad of
 * SPEC.md:166 over all rows; rows with zero gradient are unchanged). NULL: in-place updates. */
int ember_relations_external(ember_ctx* ctx, float* grad_dev);
int ember_relations_apply_dense(ember_ctx* ctx, const float* grad_dev);
/* nccl_unique_id: 128 bytes (ncclUniqueId) shared by all ranks. NCCL is loaded at run time. */
int ember_comm_init(ember_ctx* ctx, const void* nccl_unique_id, int rank, int world);
/* Sum the relation gradients across ranks before the relation Adagrad (on by default once
 * comm is initialised). */
int ember_comm_barrier(ember_ctx* ctx);
/* Copy a partition's theta+acc (rows x dim each) device->device, possibly across GPUs
 * (P2P over NVLink via cudaMemcpyPeerAsync on the context stream). */
int ember_partition_copy(ember_ctx* ctx, float* dst_theta, float* dst_acc, int dst_device, const float* src_theta,
                         const float* src_acc, int src_device, uint64_t rows);

#ifdef __cplusplus
}
#endif
#endif /* EMBER_GPU_H */
