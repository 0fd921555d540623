// SPDX-License-Identifier: Apache-2.0
//
// Synthetic graphs with planted structure and edge bucketing.
// Test/bench data plumbing, not the hot path. Edge e is a pure function of (seed, e):
//   src rank ~ power law w(r) ∝ (r+1)^-0.9 (inverse CDF of the continuous law),
//   relation ~ Zipf(1) over [0, R) (R == 1: single relation, social graph),
//   with prob 0.9 the destination is drawn (same power law) inside community pi_r(comm(src)),
//   comm(rank) = rank mod K and pi_r an affine bijection of Z_K; otherwise globally.
//   Ranks map to node ids through a keyed Feistel permutation (no tables needed).
#include <cub/cub.cuh>

#include <cmath>
#include <vector>

#include "engine.h"

namespace ember {
namespace {

struct Gen {
    uint64_t V;
    uint32_t R;
    uint32_t K;      // communities, power of two
    uint64_t seed;
    uint32_t half;   // Feistel half width in bits
    float train, valid;
    double node_pow_hi;  // (V+1)^0.1 - 1
};

EMBER_HD double u01(uint64_t h) { return static_cast<double>(h >> 11) * 0x1.0p-53; }

EMBER_HD uint64_t powerlaw(double u, uint64_t n) {
    const double a = pow(static_cast<double>(n) + 1.0, 0.1) - 1.0;
    const double x = pow(1.0 + u * a, 10.0);
    uint64_t r = x < 1.0 ? 0 : static_cast<uint64_t>(x) - 1;
    return r >= n ? n - 1 : r;
}

EMBER_HD uint32_t zipf_rel(double u, uint32_t R) {
    const double x = exp(u * log(static_cast<double>(R) + 1.0));
    uint32_t r = x < 1.0 ? 0 : static_cast<uint32_t>(x) - 1;
    return r >= R ? R - 1 : r;
}

EMBER_HD uint64_t feistel(uint64_t x, const Gen& g) {
    const uint64_t mask = (1ULL << g.half) - 1;
    do {
        uint64_t l = x >> g.half, r = x & mask;
        for (uint32_t round = 0; round < 4; ++round) {
            const uint64_t f = splitmix64(r ^ mix_seed(g.seed, 0xfe15ULL + round)) & mask;
            const uint64_t nl = r;
            r = l ^ f;
            l = nl;
        }
        x = (l << g.half) | r;
    } while (x >= g.V);  // cycle-walk back into [0, V)
    return x;
}

EMBER_HD void gen_edge(const Gen& g, uint64_t e, uint32_t* out3, uint8_t* split) {
    const uint64_t h = mix_seed(g.seed, e);
    const uint64_t src_rank = powerlaw(u01(splitmix64(h + 1)), g.V);
    const uint32_t rel = g.R <= 1 ? 0u : zipf_rel(u01(splitmix64(h + 2)), g.R);
    uint64_t dst_rank;
    if (u01(splitmix64(h + 3)) < 0.9) {
        const uint64_t c = src_rank & (g.K - 1);
        uint64_t c2 = c;
        if (g.R > 1) {
            const uint64_t hr = mix_seed(g.seed ^ 0x7e1aULL, rel);
            const uint64_t a = 2 * (hr % (g.K / 2 > 0 ? g.K / 2 : 1)) + 1;
            c2 = (a * c + (splitmix64(hr) & (g.K - 1))) & (g.K - 1);
        }
        const uint64_t members = (g.V - c2 + g.K - 1) / g.K;
        dst_rank = c2 + g.K * powerlaw(u01(splitmix64(h + 4)), members);
    } else {
        dst_rank = powerlaw(u01(splitmix64(h + 4)), g.V);
    }
    out3[0] = static_cast<uint32_t>(feistel(src_rank, g));
    out3[1] = rel;
    out3[2] = static_cast<uint32_t>(feistel(dst_rank, g));
    if (split) {
        const double us = u01(splitmix64(h + 5));
        *split = us < g.train ? 0 : (us < static_cast<double>(g.train) + g.valid ? 1 : 2);
    }
}

Gen make_gen(uint64_t V, uint32_t R, uint64_t seed, float train, float valid) {
    Gen g{};
    g.V = V;
    g.R = R;
    uint32_t K = 1;
    while (K < 1024 && static_cast<uint64_t>(K) * 8 <= V) K <<= 1;
    g.K = K;
    g.seed = seed;
    uint32_t bits = 1;
    while ((1ULL << bits) < V) ++bits;
    g.half = (bits + 1) / 2;
    g.train = train;
    g.valid = valid;
    return g;
}

__global__ void k_gen(Gen g, uint64_t first, uint64_t n, uint32_t* edges, uint8_t* split) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    gen_edge(g, first + e, edges + 3 * e, split ? split + e : nullptr);
}

EMBER_HD uint32_t part_of(uint64_t id, uint64_t V, uint32_t p) {
    const uint64_t q = V / p, r = V % p;
    const uint64_t big = r * (q + 1);
    return id < big ? static_cast<uint32_t>(id / (q + 1)) : static_cast<uint32_t>(r + (id - big) / q);
}

__global__ void k_bucket_keys(const uint32_t* edges, uint64_t n, uint64_t V, uint32_t p, uint32_t* keys,
                              uint32_t* vals) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    keys[e] = part_of(edges[3 * e], V, p) * p + part_of(edges[3 * e + 2], V, p);
    vals[e] = static_cast<uint32_t>(e);
}

__global__ void k_permute_edges(const uint32_t* in, const uint32_t* order, uint64_t n, uint32_t* out) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    const uint64_t s = order[e];
    out[3 * e] = in[3 * s];
    out[3 * e + 1] = in[3 * s + 1];
    out[3 * e + 2] = in[3 * s + 2];
}

__global__ void k_bucket_offsets(const uint32_t* keys_sorted, uint64_t n, uint32_t nb, uint64_t* offsets) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > nb) return;
    uint64_t lo = 0, hi = n;  // first index with key >= b
    while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (keys_sorted[mid] < b) lo = mid + 1;
        else hi = mid;
    }
    offsets[b] = lo;
}

}  // namespace

void graph_generate(int device, uint64_t V, uint32_t R, uint64_t n, uint64_t seed, float train, float valid,
                    uint32_t* edges, uint8_t* split) {
    if (V == 0 || V > 0xffffffffULL) throw ConfigError("num_nodes must be in [1, 2^32)");
    if (R == 0) R = 1;
    const Gen g = make_gen(V, R, seed, train, valid);
    if (device < 0) {
#pragma omp parallel for schedule(static)
        for (int64_t e = 0; e < static_cast<int64_t>(n); ++e) gen_edge(g, e, edges + 3 * e, split ? split + e : nullptr);
        return;
    }
    EMBER_CUDA(cudaSetDevice(device));
    const uint64_t step = 1ULL << 30;
    for (uint64_t b = 0; b < n; b += step) {
        const uint64_t m = std::min(step, n - b);
        k_gen<<<(unsigned)((m + 255) / 256), 256>>>(g, b, m, edges + 3 * b, split ? split + b : nullptr);
        EMBER_CUDA(cudaGetLastError());
    }
    EMBER_CUDA(cudaDeviceSynchronize());
}

void graph_bucket(int device, uint64_t V, uint32_t p, const uint32_t* in, uint64_t n, uint32_t* out,
                  uint64_t* offsets) {
    if (p == 0 || p > 4096) throw ConfigError("bucket: 1 <= p <= 4096");
    const uint32_t nbk = p * p;
    if (device < 0) {
        std::vector<uint64_t> cnt(nbk + 1, 0);
        std::vector<uint32_t> key(n);
        for (uint64_t e = 0; e < n; ++e) {
            key[e] = part_of(in[3 * e], V, p) * p + part_of(in[3 * e + 2], V, p);
            ++cnt[key[e] + 1];
        }
        for (uint32_t b = 0; b < nbk; ++b) cnt[b + 1] += cnt[b];
        for (uint32_t b = 0; b <= nbk; ++b) offsets[b] = cnt[b];
        for (uint64_t e = 0; e < n; ++e) {
            const uint64_t at = cnt[key[e]]++;
            out[3 * at] = in[3 * e];
            out[3 * at + 1] = in[3 * e + 1];
            out[3 * at + 2] = in[3 * e + 2];
        }
        return;
    }
    if (n >= (1ULL << 31)) throw ConfigError("device bucketing supports < 2^31 edges per call");
    EMBER_CUDA(cudaSetDevice(device));
    uint32_t *keys, *keys2, *vals, *vals2;
    EMBER_CUDA(cudaMalloc(&keys, n * 4 + 4));
    EMBER_CUDA(cudaMalloc(&keys2, n * 4 + 4));
    EMBER_CUDA(cudaMalloc(&vals, n * 4 + 4));
    EMBER_CUDA(cudaMalloc(&vals2, n * 4 + 4));
    const unsigned blocks = (unsigned)((n + 255) / 256);
    k_bucket_keys<<<blocks, 256>>>(in, n, V, p, keys, vals);
    EMBER_CUDA(cudaGetLastError());
    uint32_t bits = 1;
    while ((1u << bits) < nbk) ++bits;
    size_t tmp_bytes = 0;
    EMBER_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2, vals, vals2, (int)n, 0, (int)bits));
    void* tmp;
    EMBER_CUDA(cudaMalloc(&tmp, tmp_bytes + 16));
    EMBER_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, vals, vals2, (int)n, 0, (int)bits));
    k_permute_edges<<<blocks, 256>>>(in, vals2, n, out);
    EMBER_CUDA(cudaGetLastError());
    uint64_t* doff;
    EMBER_CUDA(cudaMalloc(&doff, (nbk + 1) * sizeof(uint64_t)));
    k_bucket_offsets<<<(nbk + 1 + 255) / 256, 256>>>(keys2, n, nbk, doff);
    EMBER_CUDA(cudaGetLastError());
    EMBER_CUDA(cudaMemcpy(offsets, doff, (nbk + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    EMBER_CUDA(cudaDeviceSynchronize());
    cudaFree(keys);
    cudaFree(keys2);
    cudaFree(vals);
    cudaFree(vals2);
    cudaFree(tmp);
    cudaFree(doff);
}

// ---- graph-store preprocessing on the device (ingest, partition_nodes,
// bucket_edges) ----------------------------------------------------------------------------
// Pinned semantics (SPEC leaves orders open): dense node ids = rank of the token among the sorted
// unique src/dst tokens, dense relation ids likewise; the node permutation sorts dense ids by
// (mix_seed(mix_seed(seed, 0x9e47), v), v) and relabels v -> its position, so partition k (a
// contiguous row range) is a seeded random node subset; the edge shuffle sorts edge indices by
// (mix_seed(mix_seed(seed, 0x5917), e), e); the first floor(train*n) shuffled edges are train,
// the next floor(valid*n) valid, the rest test; train is bucketed stably (bucket_edges above).
// Restated on the CPU in oracle/ember_oracle.c (orc_preprocess) and compared bit for bit.
namespace {

__global__ void k_prep_tokens(const uint32_t* raw, uint64_t n, uint32_t* nodes, uint32_t* rels) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    nodes[e] = raw[3 * e];
    nodes[n + e] = raw[3 * e + 2];
    rels[e] = raw[3 * e + 1];
}

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a, uint32_t n, uint32_t x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void k_prep_keys(uint64_t seed, uint64_t n, uint64_t* keys, uint32_t* vals) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keys[i] = mix_seed(seed, i);
    vals[i] = (uint32_t)i;
}

__global__ void k_prep_gather(const uint32_t* src, const uint32_t* idx, uint64_t n, uint32_t* out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = src[idx[i]];
}

__global__ void k_prep_invert(const uint32_t* order, uint64_t n, uint32_t* new_id) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) new_id[order[i]] = (uint32_t)i;
}

// shuffled edge i = raw edge order[i], relabeled.
__global__ void k_prep_relabel(const uint32_t* raw, const uint32_t* order, uint64_t n, const uint32_t* U, uint32_t V,
                               const uint32_t* RU, uint32_t R, const uint32_t* new_id, uint32_t* out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t e = order[i];
    out[3 * i] = new_id[lower_bound_u32(U, V, raw[3 * e])];
    out[3 * i + 1] = lower_bound_u32(RU, R, raw[3 * e + 1]);
    out[3 * i + 2] = new_id[lower_bound_u32(U, V, raw[3 * e + 2])];
}

template <typename T>
T* dnew(size_t n) {
    T* p = nullptr;
    EMBER_CUDA(cudaMalloc(&p, (n ? n : 1) * sizeof(T)));
    return p;
}

// sorted unique values of in[0, n) -> out (capacity n), returns the count
uint32_t sort_unique(const uint32_t* in, uint64_t n, uint32_t* out) {
    uint32_t* sorted = dnew<uint32_t>(n);
    uint32_t* cnt = dnew<uint32_t>(1);
    size_t b1 = 0, b2 = 0;
    EMBER_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, b1, in, sorted, (int)n));
    EMBER_CUDA(cub::DeviceSelect::Unique(nullptr, b2, sorted, out, cnt, (int)n));
    void* tmp = dnew<char>(std::max(b1, b2));
    size_t b = std::max(b1, b2);
    EMBER_CUDA(cub::DeviceRadixSort::SortKeys(tmp, b, in, sorted, (int)n));
    b = std::max(b1, b2);
    EMBER_CUDA(cub::DeviceSelect::Unique(tmp, b, sorted, out, cnt, (int)n));
    uint32_t h = 0;
    EMBER_CUDA(cudaMemcpy(&h, cnt, 4, cudaMemcpyDeviceToHost));
    cudaFree(sorted);
    cudaFree(cnt);
    cudaFree(tmp);
    return h;
}

// order[i] = index of the i-th smallest (mix_seed(seed, index), index)
void seeded_order(uint64_t seed, uint64_t n, uint32_t* order) {
    uint64_t *k1 = dnew<uint64_t>(n), *k2 = dnew<uint64_t>(n);
    uint32_t* v1 = dnew<uint32_t>(n);
    const unsigned blocks = (unsigned)((n + 255) / 256);
    k_prep_keys<<<blocks, 256>>>(seed, n, k1, v1);
    EMBER_CUDA(cudaGetLastError());
    size_t b = 0;
    EMBER_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, b, k1, k2, v1, order, (int)n));  // stable: ties by index
    void* tmp = dnew<char>(b);
    EMBER_CUDA(cub::DeviceRadixSort::SortPairs(tmp, b, k1, k2, v1, order, (int)n));
    cudaFree(k1);
    cudaFree(k2);
    cudaFree(v1);
    cudaFree(tmp);
}

}  // namespace

void graph_preprocess(int device, const uint32_t* raw, uint64_t n, uint32_t p, uint64_t seed, float train_frac,
                      float valid_frac, uint32_t* train_out, uint64_t* offsets, uint32_t* valid_out, uint32_t* test_out,
                      uint64_t* counts, uint32_t* node_tokens, uint32_t* rel_tokens, uint64_t* num_nodes,
                      uint32_t* num_rel) {
    if (device < 0) throw ConfigError("graph preprocessing runs on a device (the CPU restatement is the oracle)");
    if (n == 0) throw ConfigError("empty edge list");
    if (n >= (1ULL << 31)) throw ConfigError("preprocessing supports < 2^31 edges per call");
    if (!(train_frac >= 0.f && valid_frac >= 0.f && train_frac + valid_frac <= 1.f))
        throw ConfigError("split fractions must be >= 0 and sum to <= 1");
    EMBER_CUDA(cudaSetDevice(device));
    const unsigned blocks = (unsigned)((n + 255) / 256);
    uint32_t* toks = dnew<uint32_t>(2 * n);
    uint32_t* rtoks = dnew<uint32_t>(n);
    k_prep_tokens<<<blocks, 256>>>(raw, n, toks, rtoks);
    EMBER_CUDA(cudaGetLastError());
    uint32_t* U = dnew<uint32_t>(2 * n);
    uint32_t* RU = dnew<uint32_t>(n);
    const uint32_t V = sort_unique(toks, 2 * n, U);
    const uint32_t R = sort_unique(rtoks, n, RU);
    if (p == 0 || p > V) throw ConfigError("need 1 <= p <= number of nodes");
    // partition_nodes: seeded permutation of the dense ids
    uint32_t* vorder = dnew<uint32_t>(V);
    uint32_t* new_id = dnew<uint32_t>(V);
    seeded_order(mix_seed(seed, 0x9e47ULL), V, vorder);
    k_prep_invert<<<(V + 255) / 256, 256>>>(vorder, V, new_id);
    EMBER_CUDA(cudaGetLastError());
    // ingest: seeded shuffle of the edges, relabeled
    uint32_t* eorder = dnew<uint32_t>(n);
    seeded_order(mix_seed(seed, 0x5917ULL), n, eorder);
    uint32_t* shuffled = dnew<uint32_t>(3 * n);
    k_prep_relabel<<<blocks, 256>>>(raw, eorder, n, U, V, RU, R, new_id, shuffled);
    EMBER_CUDA(cudaGetLastError());
    const uint64_t n_train = (uint64_t)((double)train_frac * (double)n);
    const uint64_t n_valid = std::min<uint64_t>(n - n_train, (uint64_t)((double)valid_frac * (double)n));
    const uint64_t n_test = n - n_train - n_valid;
    // bucket_edges of the train split (stable)
    if (n_train) graph_bucket(device, V, p, shuffled, n_train, train_out, offsets);
    else
        for (uint64_t b = 0; b <= (uint64_t)p * p; ++b) offsets[b] = 0;
    if (valid_out && n_valid)
        EMBER_CUDA(cudaMemcpy(valid_out, shuffled + 3 * n_train, n_valid * 12, cudaMemcpyDeviceToDevice));
    if (test_out && n_test)
        EMBER_CUDA(cudaMemcpy(test_out, shuffled + 3 * (n_train + n_valid), n_test * 12, cudaMemcpyDeviceToDevice));
    if (node_tokens) {  // token of relabeled node i: U[vorder[i]]
        k_prep_gather<<<(V + 255) / 256, 256>>>(U, vorder, V, node_tokens);
        EMBER_CUDA(cudaGetLastError());
    }
    if (rel_tokens) EMBER_CUDA(cudaMemcpy(rel_tokens, RU, (size_t)R * 4, cudaMemcpyDeviceToDevice));
    EMBER_CUDA(cudaDeviceSynchronize());
    counts[0] = n_train;
    counts[1] = n_valid;
    counts[2] = n_test;
    *num_nodes = V;
    *num_rel = R;
    for (void* q : {(void*)toks, (void*)rtoks, (void*)U, (void*)RU, (void*)vorder, (void*)new_id, (void*)eorder,
                    (void*)shuffled})
        cudaFree(q);
}

}  // namespace ember
