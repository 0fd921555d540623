// SPDX-License-Identifier: Apache-2.0
//
// Memory-bound kernels of the training step (everything but the dense contraction):
//   k_sample          sample_negatives, SPEC.md:148-156 (counter-based, bit-exact with the oracle)
//   k_gather_adjust   formBatch gather + "adjust" to per-side dot-product operands
//   k_gather_negs     negative rows
//   k_chain_rule      chain rule back through adjust
//   k_batch_loss      deterministic loss reduction
//   k_adagrad_segs    segmented sum of sorted gradient rows + sparse Adagrad
// Rows are dim floats (dim % 4 == 0) and are moved warp-per-row with 128-bit accesses.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include "engine.h"

namespace ember {
namespace {

__device__ __forceinline__ const float* node_row(const PartView& v, uint32_t id, uint32_t d) {
    return v.theta + (uint64_t)(id - v.first) * d;
}

__device__ __forceinline__ float4 ldg4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }

// Loads a dim-float row into shared memory with float4 lanes.
__device__ __forceinline__ void warp_load_row(float* dst, const float* src, uint32_t d, uint32_t lane) {
    for (uint32_t v = lane; v < d / 4; v += 32) reinterpret_cast<float4*>(dst)[v] = ldg4(src + 4 * v);
}

__global__ void k_sample(uint32_t* out, uint32_t nt, uint32_t n_deg, uint32_t total, uint64_t base,
                         const uint32_t* __restrict__ bucket, uint64_t bucket_n, uint64_t src_first, uint64_t src_rows,
                         uint64_t dst_first, uint64_t dst_rows) {
    const uint32_t slot = blockIdx.x * blockDim.x + threadIdx.x;
    if (slot >= total) return;
    const uint32_t k = slot % nt;
    const uint32_t side = (slot / nt) & 1u;
    Rng g(mix_seed(base, (uint64_t)slot));
    uint32_t id;
    if (k < n_deg && bucket_n > 0) {
        const uint64_t e = g.uniform_below(bucket_n);
        id = bucket[3 * e + (side == 0 ? 2 : 0)];  // endpoint of a uniform bucket edge
    } else if (side == 0) {
        id = (uint32_t)(dst_first + g.uniform_below(dst_rows));
    } else {
        id = (uint32_t)(src_first + g.uniform_below(src_rows));
    }
    out[slot] = id;
}

// One warp per edge: A[0][e] = adj_dst(s, r), A[1][e] = adj_src(r, t), fpos[e] = adj_dst . t.
__global__ void k_gather_adjust(const uint32_t* __restrict__ edges, uint32_t nb, PartView pi, PartView pj,
                                const float* __restrict__ rel, int kind, uint32_t d, float* __restrict__ A,
                                float* __restrict__ fpos) {
    extern __shared__ float sm[];
    const uint32_t wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t e = blockIdx.x * (blockDim.x >> 5) + wib;
    if (e >= nb) return;
    float* ss = sm + wib * 3 * d;
    float* sr = ss + d;
    float* st = sr + d;
    const uint32_t s = edges[3 * e], r = edges[3 * e + 1], t = edges[3 * e + 2];
    warp_load_row(ss, node_row(pi, s, d), d, lane);
    warp_load_row(st, node_row(pj, t, d), d, lane);
    if (kind != EMBER_DOT) warp_load_row(sr, rel + (uint64_t)r * d, d, lane);
    __syncwarp();
    float* ad = A + (uint64_t)e * d;
    float* as = A + ((uint64_t)nb + e) * d;
    float part = 0.f;
    if (kind == EMBER_COMPLEX) {
        const uint32_t h = d / 2;
        for (uint32_t k = lane; k < h; k += 32) {
            const float a = ss[k], b = ss[h + k], c = sr[k], x = st[k], y = st[h + k];
            const float ee = sr[h + k];
            const float re = __fsub_rn(__fmul_rn(a, c), __fmul_rn(b, ee));
            const float im = __fadd_rn(__fmul_rn(a, ee), __fmul_rn(b, c));
            ad[k] = re;
            ad[h + k] = im;
            as[k] = __fadd_rn(__fmul_rn(c, x), __fmul_rn(ee, y));
            as[h + k] = __fsub_rn(__fmul_rn(c, y), __fmul_rn(ee, x));
            part += re * x + im * y;
        }
    } else {
        for (uint32_t k = lane; k < d; k += 32) {
            const float v = kind == EMBER_DOT ? ss[k] : __fmul_rn(ss[k], sr[k]);
            ad[k] = v;
            as[k] = kind == EMBER_DOT ? st[k] : __fmul_rn(sr[k], st[k]);
            part += v * st[k];
        }
    }
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) fpos[e] = part;
}

// Negative rows: slot -> N[slot] (side 0 rows come from partition j, side 1 from i).
__global__ void k_gather_negs(const uint32_t* __restrict__ negs, uint32_t n, uint32_t nt, PartView pi, PartView pj,
                              uint32_t d, float* __restrict__ N) {
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= n) return;
    const uint32_t side = (w / nt) & 1u;
    const float* src = node_row(side == 0 ? pj : pi, negs[w], d);
    float4* dst = reinterpret_cast<float4*>(N + (uint64_t)w * d);
    for (uint32_t v = lane; v < d / 4; v += 32) dst[v] = ldg4(src + 4 * v);
}

// Chain rule (one warp per edge). dA excludes the positive term, added here:
//   grad adj_dst = g0_dst * t + (P N)_dst,  grad adj_src = g0_src * s + (P N)_src
//   grad t += g0_dst * adj_dst (positive score = adj_dst . t), grad s += g0_src * adj_src.
__global__ void k_chain_rule(const uint32_t* __restrict__ edges, uint32_t nb, PartView pi, PartView pj,
                             const float* __restrict__ rel, int kind, uint32_t d, const float* __restrict__ A,
                             const float* __restrict__ dA, const float* __restrict__ g0, float* __restrict__ grows,
                             float* __restrict__ rrows) {
    extern __shared__ float sm[];
    const uint32_t wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t e = blockIdx.x * (blockDim.x >> 5) + wib;
    if (e >= nb) return;
    float* ss = sm + wib * 3 * d;
    float* sr = ss + d;
    float* st = sr + d;
    const uint32_t s = edges[3 * e], r = edges[3 * e + 1], t = edges[3 * e + 2];
    warp_load_row(ss, node_row(pi, s, d), d, lane);
    warp_load_row(st, node_row(pj, t, d), d, lane);
    if (kind != EMBER_DOT) warp_load_row(sr, rel + (uint64_t)r * d, d, lane);
    __syncwarp();
    const float gd = g0[e], gs = g0[(uint64_t)nb + e];
    const float* ad = A + (uint64_t)e * d;
    const float* as = A + ((uint64_t)nb + e) * d;
    const float* u = dA + (uint64_t)e * d;
    const float* w = dA + ((uint64_t)nb + e) * d;
    float* gS = grows + (uint64_t)e * d;
    float* gT = grows + ((uint64_t)nb + e) * d;
    float* gR = rrows + (uint64_t)e * d;
    if (kind == EMBER_COMPLEX) {
        const uint32_t h = d / 2;
        for (uint32_t k = lane; k < h; k += 32) {
            const float a = ss[k], b = ss[h + k], c = sr[k], ee = sr[h + k], x = st[k], y = st[h + k];
            const float u0 = u[k] + gd * x, u1 = u[h + k] + gd * y;
            const float w0 = w[k] + gs * a, w1 = w[h + k] + gs * b;
            gS[k] = gs * as[k] + (u0 * c + u1 * ee);
            gS[h + k] = gs * as[h + k] + (u1 * c - u0 * ee);
            gR[k] = (u0 * a + u1 * b) + (w0 * x + w1 * y);
            gR[h + k] = (u1 * a - u0 * b) + (w0 * y - w1 * x);
            gT[k] = gd * ad[k] + (w0 * c - w1 * ee);
            gT[h + k] = gd * ad[h + k] + (w0 * ee + w1 * c);
        }
    } else if (kind == EMBER_DISTMULT) {
        for (uint32_t k = lane; k < d; k += 32) {
            const float uk = u[k] + gd * st[k], wk = w[k] + gs * ss[k];
            gS[k] = gs * as[k] + uk * sr[k];
            gR[k] = uk * ss[k] + wk * st[k];
            gT[k] = gd * ad[k] + wk * sr[k];
        }
    } else {
        for (uint32_t k = lane; k < d; k += 32) {
            gS[k] = gs * as[k] + (u[k] + gd * st[k]);
            gT[k] = gd * ad[k] + (w[k] + gs * ss[k]);
        }
    }
}

// loss = (1/nb) sum_e (lse_dst - f) + (lse_src - f), one block, fixed order.
__global__ void k_batch_loss(const float* lse, const float* fpos, uint32_t nb, float* out) {
    __shared__ double red[1024];
    double acc = 0.0;
    for (uint32_t e = threadIdx.x; e < nb; e += blockDim.x)
        acc += (double)(lse[e] - fpos[e]) + (double)(lse[(uint64_t)nb + e] - fpos[e]);
    red[threadIdx.x] = acc;
    __syncthreads();
    for (uint32_t s = blockDim.x / 2; s; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = (float)(red[0] / (double)nb);
}

__global__ void k_node_keys(const uint32_t* __restrict__ edges, uint32_t nb, const uint32_t* __restrict__ negs,
                            uint32_t n_neg, uint32_t* keys, uint32_t* vals) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t n = 2 * nb + n_neg;
    if (i >= n) return;
    uint32_t k;
    if (i < nb) k = edges[3 * i];
    else if (i < 2 * nb) k = edges[3 * (i - nb) + 2];
    else k = negs[i - 2 * nb];
    keys[i] = k;
    vals[i] = i;
}

__global__ void k_rel_keys(const uint32_t* __restrict__ edges, uint32_t nb, uint32_t* keys, uint32_t* vals) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nb) return;
    keys[i] = edges[3 * i + 1];
    vals[i] = i;
}

__device__ __forceinline__ float adagrad_elem(float& th, float& ac, float g, float lr, float eps) {
    const float a = __fadd_rn(ac, __fmul_rn(g, g));
    ac = a;
    th = __fsub_rn(th, __fdiv_rn(__fmul_rn(lr, g), __fadd_rn(__fsqrt_rn(a), eps)));
    return th;
}

// Segmented sum in two deterministic passes so hot ids (Zipf relations, power-law nodes) are not
// serialised on one warp: every segment is cut into chunks of <= kChunk sorted rows.
constexpr uint32_t kChunk = 32;

__global__ void k_chunk_counts(const uint32_t* __restrict__ counts, const uint32_t* __restrict__ nunique, uint32_t n,
                               uint32_t* cc) {
    const uint32_t u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= n) return;
    cc[u] = u < *nunique ? (counts[u] + kChunk - 1) / kChunk : 0u;
}

// Pass 1: one warp per chunk sums its rows (ascending sorted position) into partial[chunk].
__global__ void k_chunk_sum(const uint32_t* __restrict__ coff, const uint32_t* __restrict__ offsets,
                            const uint32_t* __restrict__ counts, const uint32_t* __restrict__ nunique,
                            const uint32_t* __restrict__ vals, const float* __restrict__ rows, uint32_t d,
                            float* __restrict__ partial) {
    const uint32_t g = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const uint32_t nu = *nunique;
    if (nu == 0) return;
    const uint32_t total = coff[nu - 1] + (counts[nu - 1] + kChunk - 1) / kChunk;
    if (g >= total) return;
    uint32_t lo = 0, hi = nu - 1;  // last segment whose first chunk is <= g
    while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (coff[mid] <= g) lo = mid;
        else hi = mid - 1;
    }
    const uint32_t r0 = offsets[lo] + (g - coff[lo]) * kChunk;
    const uint32_t r1 = min(r0 + kChunk, offsets[lo] + counts[lo]);
    const uint32_t cnt = r1 - r0;
    const uint32_t my = lane < cnt ? vals[r0 + lane] : 0u;
    for (uint32_t base = 0; base < d / 4; base += 32) {  // all lanes stay converged for the shuffles
        const uint32_t c4 = base + lane;
        const bool live = c4 < d / 4;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
        for (uint32_t c = 0; c < cnt; ++c) {
            const uint32_t idx = __shfl_sync(0xffffffffu, my, c);
            if (live) {
                const float4 x = ldg4(rows + (uint64_t)idx * d + 4 * c4);
                acc.x += x.x; acc.y += x.y; acc.z += x.z; acc.w += x.w;
            }
        }
        if (live) reinterpret_cast<float4*>(partial + (uint64_t)g * d)[c4] = acc;
    }
}

// Pass 2: one warp per unique id sums its chunk partials in order, then Adagrad (or exports).
__global__ void k_adagrad_segs(const uint32_t* __restrict__ ukeys, const uint32_t* __restrict__ coff,
                               const uint32_t* __restrict__ counts, const uint32_t* __restrict__ nunique,
                               const float* __restrict__ partial, uint32_t d, PartView pi, PartView pj, int relations,
                               float* rel_theta, float* rel_acc, float lr, float eps, uint32_t* ids_out,
                               float* rows_out, int apply) {
    const uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (u >= *nunique) return;
    const uint32_t key = ukeys[u], beg = coff[u], cnt = (counts[u] + kChunk - 1) / kChunk;
    float* th;
    float* ac;
    if (relations) {
        th = rel_theta + (uint64_t)key * d;
        ac = rel_acc + (uint64_t)key * d;
    } else {
        const PartView& v = (key - pi.first < pi.rows) ? pi : pj;
        th = v.theta + (uint64_t)(key - v.first) * d;
        ac = v.acc + (uint64_t)(key - v.first) * d;
    }
    if (ids_out && lane == 0) ids_out[u] = key;
    for (uint32_t c4 = lane; c4 < d / 4; c4 += 32) {
        float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
        for (uint32_t c = 0; c < cnt; ++c) {
            const float4 x = ldg4(partial + (uint64_t)(beg + c) * d + 4 * c4);
            g.x += x.x; g.y += x.y; g.z += x.z; g.w += x.w;
        }
        if (rows_out) reinterpret_cast<float4*>(rows_out + (uint64_t)u * d)[c4] = g;
        if (!apply) continue;
        float4 t = reinterpret_cast<float4*>(th)[c4];
        float4 a = reinterpret_cast<float4*>(ac)[c4];
        adagrad_elem(t.x, a.x, g.x, lr, eps);
        adagrad_elem(t.y, a.y, g.y, lr, eps);
        adagrad_elem(t.z, a.z, g.z, lr, eps);
        adagrad_elem(t.w, a.w, g.w, lr, eps);
        reinterpret_cast<float4*>(th)[c4] = t;
        reinterpret_cast<float4*>(ac)[c4] = a;
    }
}

__global__ void k_adagrad_rows(const uint32_t* __restrict__ ids, const float* __restrict__ rows, uint32_t n,
                               uint32_t d, PartView pi, PartView pj, int relations, float* rel_theta, float* rel_acc,
                               float lr, float eps) {
    const uint32_t u = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (u >= n) return;
    const uint32_t key = ids[u];
    float* th;
    float* ac;
    if (relations) {
        th = rel_theta + (uint64_t)key * d;
        ac = rel_acc + (uint64_t)key * d;
    } else {
        const PartView& v = (key - pi.first < pi.rows) ? pi : pj;
        th = v.theta + (uint64_t)(key - v.first) * d;
        ac = v.acc + (uint64_t)(key - v.first) * d;
    }
    for (uint32_t k = lane; k < d; k += 32) adagrad_elem(th[k], ac[k], rows[(uint64_t)u * d + k], lr, eps);
}

// Warp per (row, negative): debug scores for parity tests.
__global__ void k_debug_scores(const float* A, const float* N, uint32_t rows, uint32_t nt, uint32_t d, float* out) {
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= rows * nt) return;
    const uint32_t r = w / nt, k = w % nt;
    float acc = 0.f;
    for (uint32_t c = lane; c < d; c += 32) acc += A[(uint64_t)r * d + c] * N[(uint64_t)k * d + c];
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) out[w] = acc;
}

__global__ void k_init_rows(float* theta, float* acc, uint64_t first, uint64_t rows, uint32_t d, uint64_t seed,
                            float a) {
    const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    Rng g(mix_seed(seed, first + r));
    float* out = theta + r * d;
    for (uint32_t k = 0; k < d; k += 4) {
        float4 v;
        v.x = g.uniform(-a, a);
        v.y = g.uniform(-a, a);
        v.z = g.uniform(-a, a);
        v.w = g.uniform(-a, a);
        reinterpret_cast<float4*>(out)[k / 4] = v;
        if (acc) reinterpret_cast<float4*>(acc + r * d)[k / 4] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
}

}  // namespace

void launch_sample(const Engine& E, uint32_t* out, uint64_t base, const uint32_t* bucket, uint64_t bucket_n,
                   const PartView& src, const PartView& dst) {
    const uint32_t n_deg = (uint32_t)ceil((double)E.m.alpha * (double)E.nt);
    const uint32_t total = E.n_neg;
    if (!total) return;
    k_sample<<<(total + 255) / 256, 256, 0, E.stream>>>(out, E.nt, n_deg, total, base, bucket, bucket_n, src.first,
                                                         src.rows, dst.first, dst.rows);
    EMBER_LAUNCHED(E);
}

void launch_gather_adjust(const Engine& E, const uint32_t* edges, uint32_t nb, const PartView& pi, const PartView& pj) {
    const uint32_t warps = 8;
    const size_t sm = (size_t)warps * 3 * E.dim * sizeof(float);
    k_gather_adjust<<<(nb + warps - 1) / warps, warps * 32, sm, E.stream>>>(edges, nb, pi, pj, E.rel_theta, E.m.kind,
                                                                             E.dim, E.s.A, E.s.fpos);
    EMBER_LAUNCHED(E);
}

void launch_gather_negatives(const Engine& E, const uint32_t* negs, const PartView& pi, const PartView& pj) {
    if (!E.n_neg) return;
    k_gather_negs<<<(E.n_neg * 32 + 255) / 256, 256, 0, E.stream>>>(negs, E.n_neg, E.nt, pi, pj, E.dim, E.s.N);
    EMBER_LAUNCHED(E);
}

void launch_chain_rule(const Engine& E, const uint32_t* edges, uint32_t nb, const PartView& pi, const PartView& pj) {
    const uint32_t warps = 8;
    const size_t sm = (size_t)warps * 3 * E.dim * sizeof(float);
    k_chain_rule<<<(nb + warps - 1) / warps, warps * 32, sm, E.stream>>>(edges, nb, pi, pj, E.rel_theta, E.m.kind,
                                                                          E.dim, E.s.A, E.s.dA, E.s.g0, E.s.grows,
                                                                          E.s.rrows);
    EMBER_LAUNCHED(E);
}

void launch_loss(const Engine& E, uint32_t nb, float* loss_out) {
    k_batch_loss<<<1, 1024, 0, E.stream>>>(E.s.lse, E.s.fpos, nb, loss_out);
    EMBER_LAUNCHED(E);
}

void launch_node_keys(const Engine& E, const uint32_t* edges, uint32_t nb, const uint32_t* negs) {
    const uint32_t n = 2 * nb + E.n_neg;
    k_node_keys<<<(n + 255) / 256, 256, 0, E.stream>>>(edges, nb, negs, E.n_neg, E.s.keys, E.s.vals);
    EMBER_LAUNCHED(E);
}

void launch_rel_keys(const Engine& E, const uint32_t* edges, uint32_t nb) {
    k_rel_keys<<<(nb + 255) / 256, 256, 0, E.stream>>>(edges, nb, E.s.keys, E.s.vals);
    EMBER_LAUNCHED(E);
}

void launch_adagrad_segments(const Engine& E, const uint32_t* ukeys, const uint32_t* offsets, const uint32_t* counts,
                             const uint32_t* nunique, const uint32_t* vals_sorted, const float* rows, uint32_t max_u,
                             const PartView& pi, const PartView& pj, bool relations, uint32_t* ids_out,
                             float* rows_out, bool apply) {
    if (!max_u) return;
    const unsigned wblocks = (max_u * 32 + 255) / 256;
    k_chunk_counts<<<(max_u + 255) / 256, 256, 0, E.stream>>>(counts, nunique, max_u, E.s.cc);
    EMBER_LAUNCHED(E);
    size_t bytes = E.s.cub_bytes;
    EMBER_CUDA(cub::DeviceScan::ExclusiveSum(E.s.cub_tmp, bytes, E.s.cc, E.s.coff, (int)max_u, E.stream));
    ++E.lib_calls;
    k_chunk_sum<<<wblocks, 256, 0, E.stream>>>(E.s.coff, offsets, counts, nunique, vals_sorted, rows, E.dim,
                                               E.s.partial);
    EMBER_LAUNCHED(E);
    k_adagrad_segs<<<wblocks, 256, 0, E.stream>>>(ukeys, E.s.coff, counts, nunique, E.s.partial, E.dim, pi, pj,
                                                  relations ? 1 : 0, E.rel_theta, E.rel_acc, E.m.lr, E.m.eps, ids_out,
                                                  rows_out, apply ? 1 : 0);
    EMBER_LAUNCHED(E);
}

void launch_adagrad_rows(const Engine& E, const uint32_t* ids, const float* rows, uint32_t n, const PartView& pi,
                         const PartView& pj, bool relations) {
    if (!n) return;
    k_adagrad_rows<<<(n * 32 + 255) / 256, 256, 0, E.stream>>>(ids, rows, n, E.dim, pi, pj, relations ? 1 : 0,
                                                                E.rel_theta, E.rel_acc, E.m.lr, E.m.eps);
    EMBER_LAUNCHED(E);
}

void launch_init_rows(cudaStream_t st, float* theta, float* acc, uint64_t first, uint64_t rows, uint32_t dim,
                      uint64_t seed) {
    if (!rows) return;
    const float a = (float)(1.0 / sqrt((double)dim));
    k_init_rows<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(theta, acc, first, rows, dim, seed, a);
    EMBER_CUDA(cudaGetLastError());
}

void launch_debug_scores(const Engine& E, const uint32_t* edges, uint32_t nb, const uint32_t* negs, int side,
                         uint32_t rows, float* out, const PartView& pi, const PartView& pj) {
    launch_gather_adjust(E, edges, nb, pi, pj);
    launch_gather_negatives(E, negs, pi, pj);
    const float* A = E.s.A + (uint64_t)side * nb * E.dim;
    const float* N = E.s.N + (uint64_t)side * E.nt * E.dim;
    const uint32_t w = rows * E.nt;
    k_debug_scores<<<(w * 32 + 255) / 256, 256, 0, E.stream>>>(A, N, rows, E.nt, E.dim, out);
    EMBER_LAUNCHED(E);
}

}  // namespace ember
