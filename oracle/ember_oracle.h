/* CPU oracle for the Gaius/Marius minibatch training step (arXiv 2101.08358).
 *
 * TEST INFRASTRUCTURE ONLY. This is the checker: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it. The product
 * (paper_2101_08358_b200/) never links or calls it.
 *
 * Parity status: the reference ships NO code for this path (proj/src/model.cpp,
 * pipeline.cpp, eval.cpp are listed in proj/src/CMakeLists.txt:1-10 but absent),
 * so this file restates the SPEC contracts and paper equations. It is pinned by
 * (a) the reference's own RNG (common.h:51-117), checked bit-for-bit against
 *     oracle/_ref/libember_ref.so built from the reference sources,
 * (b) every SPEC worked example for the model/eval ops,
 * (c) central finite differences.
 * The float arithmetic of score/loss/gradient itself is "parity unpinned" by
 * executable reference code (none exists); see DESIGN.md §Oracle.
 */
#ifndef EMBER_ORACLE_H
#define EMBER_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_DOT = 0, ORC_DISTMULT = 1, ORC_COMPLEX = 2 };

typedef struct {
    int32_t kind;           /* ModelKind */
    uint32_t dim;           /* d */
    float lr;               /* Adagrad learning rate */
    float eps;              /* Adagrad eps */
    uint32_t num_negatives; /* n_t per chunk per corruption side */
    float alpha;            /* degree-based fraction alpha */
    uint32_t num_chunks;    /* negatives are shared per chunk of the batch (1 = whole batch) */
    uint32_t pad_;
    uint64_t neg_seed;      /* seed of the negative-sampling stream */
} orc_model;

/* RNG, common.h:51-117 */
uint64_t orc_splitmix64(uint64_t x);
uint64_t orc_mix_seed(uint64_t base, uint64_t salt);
uint64_t orc_mix_seed3(uint64_t base, uint64_t a, uint64_t b);
void orc_rng_next(uint64_t seed, uint32_t k, uint64_t* out);
void orc_rng_uniform_below(uint64_t seed, uint64_t n, uint32_t k, uint64_t* out);
void orc_rng_uniform(uint64_t seed, float lo, float hi, uint32_t k, float* out);

/* Partition geometry: uniform split, sizes differ by at most one. */
uint64_t orc_part_offset(uint64_t num_nodes, uint32_t p, uint32_t k);
uint64_t orc_part_size(uint64_t num_nodes, uint32_t p, uint32_t k);

/* score(kind, s, r, d). */
float orc_score(int32_t kind, uint32_t dim, const float* s, const float* r, const float* d);

/* init_embeddings: row g gets Rng(mix_seed(seed, g)).uniform(-a, a) x dim, a = 1/sqrt(d). */
void orc_init_rows(uint64_t seed, uint32_t dim, uint64_t row_begin, uint64_t rows, float* theta);

/* sample_negatives. out: num_chunks * 2 * n_t ids laid out
 * [chunk][side][slot], side 0 = destination corruption (pool = dst partition), side 1 = source
 * corruption (pool = src partition). Degree part = endpoint of a uniform edge of the bucket. */
void orc_sample_negatives(const orc_model* m, uint64_t epoch, uint32_t bucket_step, uint32_t batch_in_bucket,
                          const uint32_t* bucket_edges, uint64_t bucket_n, uint64_t src_off, uint64_t src_size,
                          uint64_t dst_off, uint64_t dst_size, uint32_t* out);

/* loss_and_grad on one batch. Tables are global-id indexed [rows x dim].
 * Outputs (all caller-allocated, may be NULL except the counters):
 *   fpos[nb], lse[2*nb] (side-major), node_ids/node_rows: unique touched node ids ascending and the
 *   summed gradient rows (capacity 2*nb + 2*chunks*n_t), rel_ids/rel_rows likewise (capacity nb).
 * Returns the batch loss (mean over positives, both sides summed). Non-finite score -> returns NaN. */
double orc_loss_and_grad(const orc_model* m, const uint32_t* edges, uint32_t nb, const uint32_t* negs,
                         const float* node_theta, const float* rel_theta, float* fpos, float* lse,
                         uint32_t* node_ids, float* node_rows, uint32_t* n_node, uint32_t* rel_ids, float* rel_rows,
                         uint32_t* n_rel);

/* adagrad_step: per element acc += g^2; theta -= lr*g/(sqrt(acc)+eps). */
void orc_adagrad_apply(uint32_t dim, float lr, float eps, const uint32_t* ids, const float* rows, uint32_t n,
                       float* theta, float* acc);

/* One synchronous step = Algorithm 1: sample -> loss_and_grad -> adagrad on nodes and
 * relations. Returns loss. */
double orc_train_batch(const orc_model* m, uint64_t epoch, uint32_t bucket_step, uint32_t batch_in_bucket,
                       const uint32_t* bucket_edges, uint64_t bucket_n, uint64_t batch_begin, uint32_t nb,
                       uint64_t src_off, uint64_t src_size, uint64_t dst_off, uint64_t dst_size, float* node_theta,
                       float* node_acc, float* rel_theta, float* rel_acc);

/* eval. rank = 1 + #{neg : score(neg) >= score(pos)} (pessimistic ties).
 * Unfiltered: every test edge in a block of `block` edges is ranked against that block's shared
 * negatives (same sampler, stream keyed by eval_seed). Filtered: candidates are all nodes; any
 * corruption that forms a triple in `filter_keys` (sorted packed (s<<40|r<<24|d), V<2^24, R<2^16)
 * is skipped; the positive itself never counts. ranks_out: 2*n_test (side-major). */
void orc_eval_ranks(int32_t kind, uint32_t dim, const float* node_theta, const float* rel_theta, uint64_t num_nodes,
                    const uint32_t* test_edges, uint32_t n_test, int filtered, const uint64_t* filter_keys,
                    uint64_t n_filter, const uint32_t* train_edges, uint64_t n_train, uint32_t n_eval_neg,
                    float alpha_eval, uint32_t block, uint64_t eval_seed, uint32_t* ranks_out);

/* aggregate: out[0] = MRR, out[1..nk] = Hits@k. */
void orc_aggregate(const uint32_t* ranks, uint64_t n, const uint32_t* ks, uint32_t nk, double* out);

/* graph-store preprocessing, the semantics ember_graph_preprocess pins:
 * dense ids = rank among sorted unique tokens; node relabel = position in the order of dense
 * ids by (mix_seed(mix_seed(seed, 0x9e47), v), v); edge shuffle = order of edge indices by
 * (mix_seed(mix_seed(seed, 0x5917), e), e); split floor(train*n) / floor(valid*n) / rest;
 * train bucketed by (part(src), part(dst)), stable. Outputs as in the C-ABI (host arrays). */
void orc_preprocess(const uint32_t* raw, uint64_t n, uint32_t p, uint64_t seed, float train_frac, float valid_frac,
                    uint32_t* train_out, uint64_t* offsets, uint32_t* valid_out, uint32_t* test_out, uint64_t* counts,
                    uint32_t* node_tokens, uint32_t* rel_tokens, uint64_t* num_nodes, uint32_t* num_rel);

/* The benchmark graph generator (the definition ember_graph_generate implements):
 * edges first .. first+n-1 of the graph (V, R, seed) into edges (n x 3), split bytes (nullable). */
void orc_graph_generate(uint64_t V, uint32_t R, uint64_t first, uint64_t n, uint64_t seed, float train_frac,
                        float valid_frac, uint32_t* edges, uint8_t* split);
/* bucket_edges: the edges with split byte `which` (split NULL: all), stably sorted by
 * (part(src), part(dst)); offsets: p*p+1. Returns the number of selected edges. */
uint64_t orc_graph_bucket(uint64_t V, uint32_t p, const uint32_t* edges, const uint8_t* split, uint8_t which,
                          uint64_t n, uint32_t* out, uint64_t* offsets);
/* The CPU trainer's step on a batch of bucket (i, j) with partitions i and j in host memory
 * ([rows x dim] theta/acc each, global rows first_i.. / first_j..; i == j: pass the same partition
 * twice): sample -> dedupe -> gather the parameter slice -> loss_and_grad -> Adagrad in place.
 * Returns the batch loss; *n_unique_out (nullable) = unique node rows of the batch. */
double orc_train_batch_parts(const orc_model* m, uint64_t epoch, uint32_t bucket_step, uint32_t batch_in_bucket,
                             const uint32_t* bucket_edges, uint64_t bucket_n, uint64_t batch_begin, uint32_t nb,
                             uint64_t first_i, uint64_t rows_i, float* theta_i, float* acc_i, uint64_t first_j,
                             uint64_t rows_j, float* theta_j, float* acc_j, float* rel_theta, float* rel_acc,
                             uint32_t* n_unique_out);

int orc_num_threads(void);
void orc_set_num_threads(int n);  /* OpenMP team size of later calls (bench: 1-thread leg) */

#ifdef __cplusplus
}
#endif
#endif
