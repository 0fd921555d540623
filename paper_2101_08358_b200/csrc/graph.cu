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

}  // namespace ember
