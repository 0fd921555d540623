// SPDX-License-Identifier: Apache-2.0
//
// Link-prediction ranks on the device (unfiltered protocol PAPER.md:321):
// each block of `block` test edges shares n_eval sampled negatives per corruption side, drawn by
// the training sampler's stream keyed (eval_seed, 0, 0, block index) over all nodes with the
// alpha_eval degree part taken from train edges; rank = 1 + #{neg : score >= pos}.
#include <cuda_runtime.h>

#include <cmath>

#include "engine.h"

namespace ember {
namespace {

struct Tables {
    const PartView* parts;  // device array
    uint64_t V;
    uint32_t p;
};

__device__ __forceinline__ const float* row_any(const Tables& T, uint32_t id, uint32_t d) {
    const uint64_t q = T.V / T.p, r = T.V % T.p, big = r * (q + 1);
    const uint32_t k = id < big ? (uint32_t)(id / (q + 1)) : (uint32_t)(r + (id - big) / q);
    const PartView v = T.parts[k];
    return v.theta + (uint64_t)(id - v.first) * d;
}

__global__ void k_eval_sample(uint32_t* out, uint32_t nblk, uint32_t ne, uint32_t n_deg, uint64_t seed,
                              const uint32_t* train, uint64_t n_train, uint64_t V) {
    const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= (uint64_t)nblk * 2 * ne) return;
    const uint32_t q = (uint32_t)(t / (2 * ne));
    const uint32_t slot = (uint32_t)(t % (2 * ne));
    const uint32_t k = slot % ne, side = slot / ne;
    Rng g(mix_seed(mix_seed(mix_seed(seed, 0, 0), q), slot));
    uint32_t id;
    if (k < n_deg && n_train > 0) {
        const uint64_t e = g.uniform_below(n_train);
        id = train[3 * e + (side == 0 ? 2 : 0)];
    } else {
        id = (uint32_t)g.uniform_below(V);
    }
    out[t] = id;
}

__global__ void k_eval_rank(Tables T, const float* __restrict__ rel, int kind, uint32_t d,
                            const uint32_t* __restrict__ test, uint32_t n_test, const uint32_t* __restrict__ negs,
                            uint32_t ne, uint32_t block, uint32_t* ranks) {
    extern __shared__ float sm[];
    const uint32_t wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t w = blockIdx.x * (blockDim.x >> 5) + wib;
    if (w >= 2 * n_test) return;
    const uint32_t side = w / n_test, e = w % n_test;
    float* a = sm + wib * d;
    const uint32_t s = test[3 * e], r = test[3 * e + 1], t = test[3 * e + 2];
    const float* ts = row_any(T, s, d);
    const float* tt = row_any(T, t, d);
    const float* tr = kind == EMBER_DOT ? nullptr : rel + (uint64_t)r * d;
    const uint32_t h = d / 2;
    for (uint32_t k = lane; k < (kind == EMBER_COMPLEX ? h : d); k += 32) {
        if (kind == EMBER_DOT) {
            a[k] = side == 0 ? ts[k] : tt[k];
        } else if (kind == EMBER_DISTMULT) {
            a[k] = side == 0 ? ts[k] * tr[k] : tr[k] * tt[k];
        } else {
            const uint32_t re = hbm_pos(kind, d, k), im = re + 2;  // complex coordinate k (HBM layout)
            const float c = tr[re], ee = tr[im];
            if (side == 0) {
                a[re] = ts[re] * c - ts[im] * ee;
                a[im] = ts[re] * ee + ts[im] * c;
            } else {
                a[re] = c * tt[re] + ee * tt[im];
                a[im] = c * tt[im] - ee * tt[re];
            }
        }
    }
    __syncwarp();
    const float* other = side == 0 ? tt : ts;
    float pos = 0.f;
    for (uint32_t k = lane; k < d; k += 32) pos += a[k] * other[k];
    for (int o = 16; o; o >>= 1) pos += __shfl_xor_sync(0xffffffffu, pos, o);
    const uint32_t* ng = negs + ((uint64_t)(e / block) * 2 + side) * ne;
    uint32_t cnt = 0;
    for (uint32_t k = 0; k < ne; ++k) {
        const float* x = row_any(T, ng[k], d);
        float sc = 0.f;
        for (uint32_t c = lane; c < d; c += 32) sc += a[c] * x[c];
        for (int o = 16; o; o >>= 1) sc += __shfl_xor_sync(0xffffffffu, sc, o);
        cnt += sc >= pos ? 1u : 0u;
    }
    if (lane == 0) ranks[(uint64_t)side * n_test + e] = 1 + cnt;
}

// Filtered protocol: every node is a candidate for the corrupted slot, known
// true triples (sorted packed keys s<<40 | r<<24 | t) are skipped, ties count against the
// positive (rank = 1 + #{c != true : score(c) >= score(true), (c) not a known triple}).
// One CTA ranks QB query vectors (test edge x side) against all nodes, streaming candidate rows
// through shared memory in CB-row tiles; each thread owns a 4-query x 8-candidate register tile.
constexpr int FQ = 64, FC = 128, FT = 256;

__device__ __forceinline__ bool key_known(const uint64_t* __restrict__ keys, uint64_t n, uint64_t k) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (keys[mid] < k) lo = mid + 1; else hi = mid;
    }
    return lo < n && keys[lo] == k;
}

__global__ void __launch_bounds__(FT) k_eval_filtered(Tables T, const float* __restrict__ rel, int kind, uint32_t d,
                                                      const uint32_t* __restrict__ test, uint32_t n_test,
                                                      const uint64_t* __restrict__ keys, uint64_t n_keys,
                                                      uint32_t* ranks) {
    extern __shared__ float sm[];
    const uint32_t ld = d + 1;  // padded row stride: conflict-free candidate reads
    float* As = sm;                       // [FQ][ld]
    float* Cs = As + FQ * ld;             // [FC][ld]
    float* pos = Cs + FC * ld;            // [FQ]
    uint32_t* meta = reinterpret_cast<uint32_t*>(pos + FQ);  // [FQ][4]: s, r, t, side|valid
    const uint32_t tid = threadIdx.x, lane = tid & 31, wib = tid >> 5;
    const uint32_t nq = 2 * n_test, q0 = blockIdx.x * FQ;
    const uint32_t h = d / 2;
    for (uint32_t qq = wib; qq < FQ; qq += FT / 32) {
        const uint32_t q = q0 + qq;
        float* a = As + qq * ld;
        if (q >= nq) {
            for (uint32_t k = lane; k < d; k += 32) a[k] = 0.f;
            if (lane == 0) meta[4 * qq + 3] = 0;
            continue;
        }
        const uint32_t side = q / n_test, e = q % n_test;
        const uint32_t s = test[3 * e], r = test[3 * e + 1], t = test[3 * e + 2];
        const float* ts = row_any(T, s, d);
        const float* tt = row_any(T, t, d);
        const float* tr = kind == EMBER_DOT ? nullptr : rel + (uint64_t)r * d;
        for (uint32_t k = lane; k < (kind == EMBER_COMPLEX ? h : d); k += 32) {
            if (kind == EMBER_DOT) {
                a[k] = side == 0 ? ts[k] : tt[k];
            } else if (kind == EMBER_DISTMULT) {
                a[k] = side == 0 ? ts[k] * tr[k] : tr[k] * tt[k];
            } else {
                const uint32_t re = hbm_pos(kind, d, k), im = re + 2;  // complex coordinate k (HBM layout)
                const float c = tr[re], ee = tr[im];
                if (side == 0) {
                    a[re] = ts[re] * c - ts[im] * ee;
                    a[im] = ts[re] * ee + ts[im] * c;
                } else {
                    a[re] = c * tt[re] + ee * tt[im];
                    a[im] = c * tt[im] - ee * tt[re];
                }
            }
        }
        __syncwarp();
        const float* other = side == 0 ? tt : ts;
        float ps = 0.f;
        for (uint32_t k = lane; k < d; k += 32) ps += a[k] * other[k];
        for (int o = 16; o; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
        if (lane == 0) {
            pos[qq] = ps;
            meta[4 * qq] = s;
            meta[4 * qq + 1] = r;
            meta[4 * qq + 2] = t;
            meta[4 * qq + 3] = 2 | side;
        }
    }
    const uint32_t tq = tid >> 4, tc = tid & 15;  // queries tq*4 .. +3, candidates tc + 16*m
    uint32_t cnt[4] = {0, 0, 0, 0};
    for (uint64_t c0 = 0; c0 < T.V; c0 += FC) {
        __syncthreads();
        for (uint32_t x = tid; x < FC * d; x += FT) {
            const uint32_t cr = x / d, k = x % d;
            const uint64_t c = c0 + cr;
            Cs[cr * ld + k] = c < T.V ? row_any(T, (uint32_t)c, d)[k] : 0.f;
        }
        __syncthreads();
        float acc[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
        for (uint32_t k = 0; k < d; ++k) {
            float av[4], cv[8];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[(tq * 4 + i) * ld + k];
#pragma unroll
            for (int j = 0; j < 8; ++j) cv[j] = Cs[(tc + 16 * j) * ld + k];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], cv[j], acc[i][j]);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t qq = tq * 4 + i;
            const uint32_t mt = meta[4 * qq + 3];
            if (!(mt & 2)) continue;
            const uint32_t side = mt & 1, s = meta[4 * qq], r = meta[4 * qq + 1], t = meta[4 * qq + 2];
            const float ps = pos[qq];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint64_t c = c0 + tc + 16 * j;
                if (c >= T.V || acc[i][j] < ps) continue;
                if (c == (side == 0 ? t : s)) continue;
                const uint64_t key = side == 0 ? ((uint64_t)s << 40 | (uint64_t)r << 24 | c)
                                               : (c << 40 | (uint64_t)r << 24 | t);
                if (!key_known(keys, n_keys, key)) ++cnt[i];
            }
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        uint32_t v = cnt[i];
        for (int o = 8; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        const uint32_t q = q0 + tq * 4 + i;
        if (tc == 0 && q < nq) ranks[q] = 1 + v;  // q = side * n_test + e
    }
}

}  // namespace

void launch_eval_filtered(const Engine& E, const uint32_t* test, uint32_t n_test, const uint64_t* keys, uint64_t n_keys,
                          uint32_t* ranks) {
    if (!n_test) return;
    for (uint32_t k = 0; k < E.parts.size(); ++k) E.view(k);
    if (E.m.kind != EMBER_DOT && !E.rel_theta) throw ConfigError("relation table not bound");
    PartView* parts = nullptr;
    EMBER_CUDA(cudaMallocAsync(&parts, E.parts.size() * sizeof(PartView), E.stream));
    EMBER_CUDA(cudaMemcpyAsync(parts, E.parts.data(), E.parts.size() * sizeof(PartView), cudaMemcpyHostToDevice,
                               E.stream));
    Tables T{parts, E.g.num_nodes, E.g.num_partitions};
    const size_t smem = ((size_t)(FQ + FC) * (E.dim + 1) + FQ) * sizeof(float) + FQ * 4 * sizeof(uint32_t);
    EMBER_CUDA(cudaFuncSetAttribute(k_eval_filtered, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const uint32_t blocks = (2 * n_test + FQ - 1) / FQ;
    k_eval_filtered<<<blocks, FT, smem, E.stream>>>(T, E.rel_theta, E.m.kind, E.dim, test, n_test, keys, n_keys, ranks);
    EMBER_LAUNCHED(E);
    EMBER_CUDA(cudaFreeAsync(parts, E.stream));
}

void launch_eval(const Engine& E, const uint32_t* test, uint32_t n_test, const uint32_t* train, uint64_t n_train,
                 uint32_t n_eval, float alpha_eval, uint32_t block, uint64_t eval_seed, uint32_t* ranks) {
    if (!n_test) return;
    for (uint32_t k = 0; k < E.parts.size(); ++k) E.view(k);  // all partitions must be bound
    if (E.m.kind != EMBER_DOT && !E.rel_theta) throw ConfigError("relation table not bound");
    const uint32_t nblk = (n_test + block - 1) / block;
    const uint32_t n_deg = (uint32_t)ceil((double)alpha_eval * (double)n_eval);
    uint32_t* negs = nullptr;
    PartView* parts = nullptr;
    EMBER_CUDA(cudaMallocAsync(&negs, (size_t)nblk * 2 * (n_eval ? n_eval : 1) * 4, E.stream));
    EMBER_CUDA(cudaMallocAsync(&parts, E.parts.size() * sizeof(PartView), E.stream));
    EMBER_CUDA(cudaMemcpyAsync(parts, E.parts.data(), E.parts.size() * sizeof(PartView), cudaMemcpyHostToDevice,
                               E.stream));
    const uint64_t ns = (uint64_t)nblk * 2 * n_eval;
    if (ns) {
        k_eval_sample<<<(unsigned)((ns + 255) / 256), 256, 0, E.stream>>>(negs, nblk, n_eval, n_deg, eval_seed, train,
                                                                         n_train, E.g.num_nodes);
        EMBER_LAUNCHED(E);
    }
    Tables T{parts, E.g.num_nodes, E.g.num_partitions};
    const uint32_t warps = 8, w = 2 * n_test;
    k_eval_rank<<<(w + warps - 1) / warps, warps * 32, warps * E.dim * sizeof(float), E.stream>>>(
        T, E.rel_theta, E.m.kind, E.dim, test, n_test, negs, n_eval, block, ranks);
    EMBER_LAUNCHED(E);
    EMBER_CUDA(cudaFreeAsync(negs, E.stream));
    EMBER_CUDA(cudaFreeAsync(parts, E.stream));
}

}  // namespace ember
